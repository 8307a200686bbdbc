/* hawk_b200_engine.h — C ABI of the engine library (libhawk_engine.so), the
 * entry point a host without the reference's C++ types binds (Python ctypes in
 * this repo). It mirrors the reference CLI's `run`,
 * `explore` and `learn` commands over SQL text,
 * and returns result tables as plain columns.
 *
 * Every call returns a hawk_status (include/hawk_b200.h); on failure
 * hawk_engine_last_error() holds the message and hawk_engine_last_error_class()
 * the reference exception class (hawk/error.hpp:9-54). Config strings use the
 * reference's VariantConfiguration::to_string() format
 * (/root/reference/proj/src/ir_program.cpp:84-96): "<projection>;<aggregation>",
 * e.g. "multi_pass/coalesced/branched/tm=1024;local_hash/coalesced/branched/
 * cuckoo/murmur/wg=256/ht=1". A '|'-separated list gives one configuration per
 * pipeline instead.
 */
#ifndef HAWK_B200_ENGINE_H
#define HAWK_B200_ENGINE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hawk_engine hawk_engine;
typedef struct hawk_result hawk_result;
typedef struct hawk_partial hawk_partial;

const char* hawk_engine_last_error(void);
int32_t hawk_engine_last_error_class(void);

/* device < 0 creates a planning-only engine (catalog, passes, lowering; no GPU) */
int32_t hawk_engine_create(int32_t device, hawk_engine** out);
void hawk_engine_destroy(hawk_engine* e);
int32_t hawk_engine_sm_count(hawk_engine* e);
void* hawk_engine_ctx(hawk_engine* e); /* the underlying hawk_ctx* */

/* ---- device column store ------------------------------------------------------ */
/* kinds: 0 int64, 1 float64, 2 string (int64 codes into the column's lexicon).
 * data[c] are HOST pointers (copied H2D). distinct may be NULL. */
int32_t hawk_engine_put_columns(hawk_engine* e, const char* name, int32_t ncols,
                                const char* const* names, const int32_t* kinds, int64_t rows,
                                const void* const* data, const char* const* const* lexicons,
                                const int64_t* lexicon_sizes, const int64_t* distinct,
                                int64_t row_offset);
/* synthetic table generated in HBM (include/hawk_gen.h); rows < 0 = all */
int32_t hawk_engine_generate(hawk_engine* e, int32_t table, double sf, uint64_t seed,
                             int64_t row_begin, int64_t rows);
/* CSV file -> device columns (include/hawk_b200_csv.h; the reference's
 * load_csv rules, storage_csv.cpp:111-155); kinds as above */
int32_t hawk_engine_load_csv(hawk_engine* e, const char* path, const char* name, int32_t ncols,
                             const char* const* names, const int32_t* kinds, char delimiter,
                             int32_t header);
int32_t hawk_engine_drop(hawk_engine* e, const char* name);
int64_t hawk_engine_table_rows(hawk_engine* e, const char* name);
/* device pointer of a stored column (for direct kernel tests) */
const int64_t* hawk_engine_column(hawk_engine* e, const char* table, const char* column);
int32_t hawk_engine_flush_l2(hawk_engine* e);

/* ---- execution ----------------------------------------------------------------- */
int32_t hawk_engine_run(hawk_engine* e, const char* sql, const char* config, hawk_result** out);
/* shard execution: partial aggregates / projections before the cross-GPU merge */
int32_t hawk_engine_run_partial(hawk_engine* e, const char* sql, const char* config,
                                hawk_partial** out);
/* multi-GPU: this rank's shard, NCCL gather of the partials to `root`, device
 * merge there (hawk::b200::Engine::execute_sharded); comm from
 * hawk_nccl_comm_create (include/hawk_b200_comm.h). Non-root ranks get an
 * empty result with the query's columns. */
struct hawk_comm;
int32_t hawk_engine_run_sharded(hawk_engine* e, const char* sql, const char* config,
                                struct hawk_comm* comm, int32_t root, hawk_result** out);
int64_t hawk_partial_rows(const hawk_partial* p);
int32_t hawk_partial_width(const hawk_partial* p);
int32_t hawk_partial_sink(const hawk_partial* p);
const int64_t* hawk_partial_data(const hawk_partial* p);
double hawk_partial_kernel_ms(const hawk_partial* p);
int32_t hawk_partial_launches(const hawk_partial* p); /* kernels the shard run launched */
void hawk_partial_free(hawk_partial* p);
/* merges partial row blocks (each rows[i] x width int64 words) and finalises */
int32_t hawk_engine_finalize(hawk_engine* e, const char* sql, const char* config, int32_t nparts,
                             const int64_t* const* data, const int64_t* rows, hawk_result** out);

int64_t hawk_result_rows(const hawk_result* r);
int32_t hawk_result_ncols(const hawk_result* r);
const char* hawk_result_col_name(const hawk_result* r, int32_t c);
int32_t hawk_result_col_kind(const hawk_result* r, int32_t c);
const void* hawk_result_col_data(const hawk_result* r, int32_t c);
int64_t hawk_result_col_lexicon_size(const hawk_result* r, int32_t c);
const char* hawk_result_col_lexicon(const hawk_result* r, int32_t c, int64_t i);
double hawk_result_kernel_ms(const hawk_result* r);
double hawk_result_wall_ms(const hawk_result* r);
int64_t hawk_result_input_tuples(const hawk_result* r);
int32_t hawk_result_launches(const hawk_result* r);
/* one line per pipeline: "variant kernel_ms launches rows_in rows_out grid block retries" */
const char* hawk_result_metrics_text(const hawk_result* r);
void hawk_result_free(hawk_result* r);

/* ---- pipeline IR introspection -------------------------------------------------- */
int32_t hawk_engine_pipeline_count(hawk_engine* e, const char* sql, int32_t* n);
/* size of enumerate_variant_space for pipeline i, and how many are single-pass */
int32_t hawk_engine_space_size(hawk_engine* e, const char* sql, int32_t pipeline, int32_t* n,
                               int32_t* single_pass);
/* writes the i-th configuration of pipeline p's space (to_string format) */
int32_t hawk_engine_space_config(hawk_engine* e, const char* sql, int32_t pipeline, int32_t i,
                                 char* buf, int32_t len);
/* validate_program diagnostics after apply_variant ("" when clean) */
int32_t hawk_engine_validate(hawk_engine* e, const char* sql, const char* config, char* buf,
                             int32_t len);

/* generates and NVRTC-compiles every pipeline's program (no GPU needed) */
int32_t hawk_engine_compile_check(hawk_engine* e, const char* sql, const char* config, char* buf,
                                  int32_t len);
/* lowered device programs of every pipeline, one op per line */
int32_t hawk_engine_explain(hawk_engine* e, const char* sql, const char* config, char* buf,
                            int32_t len);

/* ---- optimizer ------------------------------------------------------------------------ */
int32_t hawk_engine_measure(hawk_engine* e, const char* const* sqls, int32_t n, const char* config,
                            double prune_ms, int32_t reps, double* ms);
int32_t hawk_engine_learn(hawk_engine* e, const char* const* sqls, int32_t n, int32_t q,
                          double prune_ms, int32_t reps, char* best, int32_t len, double* best_ms,
                          int32_t* evaluations, int32_t* sweeps);

/* Learned-configuration files: key=value, one dimension per
 * line ("projection.strategy=single_pass", ...). load writes the
 * configuration in to_string() form ("<proj>;<agg>") into buf. */
int32_t hawk_config_save(const char* config, const char* path);
int32_t hawk_config_load(const char* path, char* buf, int32_t len);

/* full_exploration of one pipeline kind's variant space
 * (kind 0: the 32 projection variants, 1: the 896 aggregation variants), the
 * other kind fixed by `fixed` ("<proj>;<agg>", "" = default). Writes the
 * ranking-order trace as CSV to csv_path (NULL = none): index, projection,
 * aggregation, ms, status (ok / pruned / error), detail. */
int32_t hawk_engine_explore(hawk_engine* e, const char* const* sqls, int32_t n, int32_t kind,
                            const char* fixed, double prune_ms, int32_t reps, const char* csv_path,
                            char* best, int32_t len, double* best_ms, int32_t* evaluations);
/* learn_variant_configuration with every option: early termination, an
 * unroll pass after the descent, '|'-separated start configurations (NULL =
 * the reference default), the measurement trace as CSV and the learned
 * configuration as a key-value file (NULL paths = not written). */
int32_t hawk_engine_learn_ex(hawk_engine* e, const char* const* sqls, int32_t n, int32_t q,
                             int32_t early_termination, double prune_ms, int32_t reps,
                             int32_t unroll_pass, const char* starts, const char* trace_csv_path,
                             const char* config_path, char* best, int32_t len, double* best_ms,
                             int32_t* evaluations, int32_t* sweeps);

/* Algorithm 1 over an abstract space: dimension d has sizes[d] values;
 * cost(index vector) may return INFINITY. Measurements are cached by index
 * vector; best receives ndims indices. */
typedef double (*hawk_index_cost_fn)(const int32_t* index, int32_t ndims, void* user);
int32_t hawk_coordinate_descent(int32_t ndims, const int32_t* sizes, hawk_index_cost_fn cost, void* user,
                                int32_t q, int32_t early_termination, int32_t* best, double* best_ms,
                                int32_t* evaluations, int32_t* sweeps, int32_t* sweep1_evaluations);

/* Algorithm 1 over a caller-supplied cost: cost(config)
 * returns the time of a workload configuration in to_string() format
 * (INFINITY = failed/pruned). No engine or GPU involved. */
typedef double (*hawk_cost_fn)(const char* config, void* user);
int32_t hawk_learn_with_cost(hawk_cost_fn cost, void* user, int32_t q, int32_t early_termination,
                             const char* starts, char* best, int32_t len, double* best_ms,
                             int32_t* evaluations, int32_t* sweeps);
/* starts: NULL = the reference default configuration; else '|'-separated
 * workload configurations, one descent from each (shared cache, best kept) */

#ifdef __cplusplus
}
#endif

#endif /* HAWK_B200_ENGINE_H */
