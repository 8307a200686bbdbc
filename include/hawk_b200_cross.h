/* hawk_b200_cross.h — CROSS_JOIN materialisation.
 *
 * Replaces the nested loop of the reference's CROSS_JOIN op
 * (proj/src/planner_pipelines.cpp:337-352; oracle semantics
 * proj/src/planner_reference.cpp:188-203: every probe-side row paired with
 * every auxiliary row). The engine lowers a terminal pipeline
 * LOOP(driver) ... CROSS_JOIN(aux) ... into LOOP over the driver-major pair
 * space of n_driver x n_aux rows; this call writes one column of that space.
 */
#ifndef HAWK_B200_CROSS_H
#define HAWK_B200_CROSS_H

#include <stdint.h>

#include "hawk_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* d_out[i] = side == 0 ? d_src[i / n_aux] : d_src[i % n_aux] for
 * i < n_driver * n_aux; rows up to the next multiple of 64 (at least 64) are
 * zeroed
 * (the column padding every device column carries). Asynchronous on the
 * context stream. HAWK_ERR_ARGUMENT on null pointers, negative sizes or a
 * side other than 0 / 1. */
int32_t hawk_b200_cross_expand(hawk_ctx* ctx, const int64_t* d_src, int64_t n_driver,
                               int64_t n_aux, int32_t side, int64_t* d_out);

#ifdef __cplusplus
}
#endif

#endif
