/* hawk_b200_comm.h — the multi-GPU exchange of the executor: NCCL collectives
 * over device buffers on the context's stream (SURVEY.md §8e, §8b
 * "hawk_nccl_{bcast,allreduce,allgather,alltoall} wrappers").
 *
 * The reference is single-process (no collective anywhere,
 * /root/reference/proj/CMakeLists.txt:44-45: Threads only); Hawk's data-
 * parallel path shards the fact table's rows over one process per GPU and
 * has exactly one exchange step per query: the partial aggregates (or
 * projected rows) of every shard are gathered and merged on the device.
 * libnccl.so.2 is opened at first use (the one torch already mapped, if any),
 * so the library loads on hosts without NCCL and these calls then return
 * HAWK_ERR_UNSUPPORTED.
 *
 * Element types use the executor's value types (HAWK_I64 / HAWK_F64) and
 * reductions its aggregate functions (HAWK_SUM / HAWK_MIN / HAWK_MAX);
 * int64 SUM wraps like the reference's wrap_add (planner_reference.cpp:25-33).
 */
#ifndef HAWK_B200_COMM_H
#define HAWK_B200_COMM_H

#include <stddef.h>
#include <stdint.h>

#include "hawk_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hawk_comm hawk_comm;

#define HAWK_COMM_ID_BYTES 128

/* 1 when libnccl.so.2 could be opened */
int32_t hawk_nccl_available(void);
/* ncclGetUniqueId: rank 0 creates it and ships the bytes to every rank */
int32_t hawk_nccl_unique_id(uint8_t id[HAWK_COMM_ID_BYTES]);
/* ncclCommInitRank on the context's device; collectives run on its stream */
int32_t hawk_nccl_comm_create(hawk_ctx* ctx, int32_t nranks, int32_t rank,
                              const uint8_t id[HAWK_COMM_ID_BYTES], hawk_comm** out);
int32_t hawk_nccl_comm_destroy(hawk_comm* comm);
int32_t hawk_nccl_comm_rank(const hawk_comm* comm);
int32_t hawk_nccl_comm_size(const hawk_comm* comm);
hawk_ctx* hawk_nccl_comm_ctx(const hawk_comm* comm);

/* d_recv[i] = op over ranks of d_send[i], count elements of `type` */
int32_t hawk_nccl_allreduce(hawk_comm* comm, const void* d_send, void* d_recv, size_t count,
                            int32_t type, int32_t op);
/* d_recv = concatenation in rank order of every rank's `bytes` bytes */
int32_t hawk_nccl_allgather(hawk_comm* comm, const void* d_send, void* d_recv, size_t bytes);
/* root's `bytes` bytes of d_buf to every rank */
int32_t hawk_nccl_bcast(hawk_comm* comm, void* d_buf, size_t bytes, int32_t root);
/* personalised exchange (grouped ncclSend / ncclRecv): send_bytes[p] bytes
 * at d_send + send_off[p] go to rank p; what rank p sends to this rank
 * (recv_bytes[p] bytes) lands at d_recv + recv_off[p] */
int32_t hawk_nccl_alltoall(hawk_comm* comm, const void* d_send, const size_t* send_bytes,
                           const size_t* send_off, void* d_recv, const size_t* recv_bytes,
                           const size_t* recv_off);

/* In-process loopback group (tests): N ranks of one process, one host thread
 * each, on one GPU. The hawk_nccl_* calls of a loopback communicator are
 * device-to-device copies between the ranks' buffers sequenced by host
 * barriers, so the multi-rank exchange logic runs where only one GPU is
 * present; no kernel ever waits on another rank. */
typedef struct hawk_loopback hawk_loopback;
int32_t hawk_loopback_group_create(int32_t nranks, hawk_loopback** out);
int32_t hawk_loopback_group_destroy(hawk_loopback* group);
int32_t hawk_loopback_comm_create(hawk_ctx* ctx, hawk_loopback* group, int32_t rank, hawk_comm** out);

#ifdef __cplusplus
}
#endif

#endif /* HAWK_B200_COMM_H */
