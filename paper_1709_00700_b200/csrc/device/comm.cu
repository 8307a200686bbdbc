// comm.cu — NCCL collectives over device buffers (include/hawk_b200_comm.h).
// libnccl.so.2 is opened with dlopen at first use; if torch already mapped
// its bundled NCCL into the process, that same library is reused.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "hawk_b200.h"
#include "hawk_b200_comm.h"

struct hawk_comm {
  hawk_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, size = 1, device = 0;
};

namespace {

struct Nccl {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"})
      if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return;
#define HK_NCCL(field, sym)                                   \
  *reinterpret_cast<void**>(&n.field) = dlsym(h, sym);        \
  if (!n.field) return;
    HK_NCCL(GetUniqueId, "ncclGetUniqueId")
    HK_NCCL(CommInitRank, "ncclCommInitRank")
    HK_NCCL(CommDestroy, "ncclCommDestroy")
    HK_NCCL(AllReduce, "ncclAllReduce")
    HK_NCCL(AllGather, "ncclAllGather")
    HK_NCCL(Broadcast, "ncclBroadcast")
    HK_NCCL(Send, "ncclSend")
    HK_NCCL(Recv, "ncclRecv")
    HK_NCCL(GroupStart, "ncclGroupStart")
    HK_NCCL(GroupEnd, "ncclGroupEnd")
    HK_NCCL(GetErrorString, "ncclGetErrorString")
#undef HK_NCCL
    n.ok = true;
  });
  return n;
}

int32_t status(ncclResult_t r) {
  if (r == ncclSuccess) return HAWK_OK;
  std::fprintf(stderr, "hawk_b200: NCCL error %s\n", nccl().GetErrorString(r));
  return HAWK_ERR_NCCL;
}

cudaStream_t stream_of(const hawk_comm* c) {
  return static_cast<cudaStream_t>(hawk_b200_ctx_stream(c->ctx));
}

}  // namespace

extern "C" {

int32_t hawk_nccl_available(void) { return nccl().ok ? 1 : 0; }

int32_t hawk_nccl_unique_id(uint8_t id[HAWK_COMM_ID_BYTES]) {
  if (!id) return HAWK_ERR_ARGUMENT;
  if (!nccl().ok) return HAWK_ERR_UNSUPPORTED;
  static_assert(sizeof(ncclUniqueId) == HAWK_COMM_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId u;
  const int32_t st = status(nccl().GetUniqueId(&u));
  if (st == HAWK_OK) std::memcpy(id, &u, HAWK_COMM_ID_BYTES);
  return st;
}

int32_t hawk_nccl_comm_create(hawk_ctx* ctx, int32_t nranks, int32_t rank,
                              const uint8_t id[HAWK_COMM_ID_BYTES], hawk_comm** out) {
  if (!ctx || !id || !out || nranks < 1 || rank < 0 || rank >= nranks) return HAWK_ERR_ARGUMENT;
  if (!nccl().ok) return HAWK_ERR_UNSUPPORTED;
  auto* c = new hawk_comm;
  c->ctx = ctx;
  c->rank = rank;
  c->size = nranks;
  c->device = hawk_b200_ctx_device(ctx);
  cudaSetDevice(c->device);
  ncclUniqueId u;
  std::memcpy(&u, id, HAWK_COMM_ID_BYTES);
  const int32_t st = status(nccl().CommInitRank(&c->comm, nranks, u, rank));
  if (st != HAWK_OK) {
    delete c;
    return st;
  }
  *out = c;
  return HAWK_OK;
}

int32_t hawk_nccl_comm_destroy(hawk_comm* c) {
  if (!c) return HAWK_OK;
  if (c->comm) nccl().CommDestroy(c->comm);
  delete c;
  return HAWK_OK;
}

int32_t hawk_nccl_comm_rank(const hawk_comm* c) { return c ? c->rank : -1; }
int32_t hawk_nccl_comm_size(const hawk_comm* c) { return c ? c->size : 0; }
hawk_ctx* hawk_nccl_comm_ctx(const hawk_comm* c) { return c ? c->ctx : nullptr; }

int32_t hawk_nccl_allreduce(hawk_comm* c, const void* d_send, void* d_recv, size_t count,
                            int32_t type, int32_t op) {
  if (!c || (!d_send && count) || (!d_recv && count)) return HAWK_ERR_ARGUMENT;
  const ncclDataType_t t = type == HAWK_F64 ? ncclFloat64 : ncclInt64;
  // int64 sums wrap in two's complement: add them as uint64 (same bits)
  const ncclDataType_t tt = (type == HAWK_I64 && op == HAWK_SUM) ? ncclUint64 : t;
  ncclRedOp_t o;
  switch (op) {
    case HAWK_SUM: o = ncclSum; break;
    case HAWK_MIN: o = ncclMin; break;
    case HAWK_MAX: o = ncclMax; break;
    default: return HAWK_ERR_ARGUMENT;
  }
  cudaSetDevice(c->device);
  return status(nccl().AllReduce(d_send, d_recv, count, tt, o, c->comm, stream_of(c)));
}

int32_t hawk_nccl_allgather(hawk_comm* c, const void* d_send, void* d_recv, size_t bytes) {
  if (!c || (!d_recv && bytes)) return HAWK_ERR_ARGUMENT;
  cudaSetDevice(c->device);
  return status(nccl().AllGather(d_send, d_recv, bytes, ncclUint8, c->comm, stream_of(c)));
}

int32_t hawk_nccl_bcast(hawk_comm* c, void* d_buf, size_t bytes, int32_t root) {
  if (!c || (!d_buf && bytes) || root < 0 || root >= c->size) return HAWK_ERR_ARGUMENT;
  cudaSetDevice(c->device);
  return status(nccl().Broadcast(d_buf, d_buf, bytes, ncclUint8, root, c->comm, stream_of(c)));
}

int32_t hawk_nccl_alltoall(hawk_comm* c, const void* d_send, const size_t* send_bytes,
                           const size_t* send_off, void* d_recv, const size_t* recv_bytes,
                           const size_t* recv_off) {
  if (!c || !send_bytes || !send_off || !recv_bytes || !recv_off) return HAWK_ERR_ARGUMENT;
  cudaSetDevice(c->device);
  Nccl& n = nccl();
  int32_t st = status(n.GroupStart());
  if (st != HAWK_OK) return st;
  for (int p = 0; p < c->size; ++p) {
    if (send_bytes[p])
      st = st != HAWK_OK ? st
                         : status(n.Send(static_cast<const char*>(d_send) + send_off[p], send_bytes[p],
                                         ncclUint8, p, c->comm, stream_of(c)));
    if (recv_bytes[p])
      st = st != HAWK_OK ? st
                         : status(n.Recv(static_cast<char*>(d_recv) + recv_off[p], recv_bytes[p],
                                         ncclUint8, p, c->comm, stream_of(c)));
  }
  const int32_t end = status(n.GroupEnd());
  return st != HAWK_OK ? st : end;
}

}  // extern "C"
