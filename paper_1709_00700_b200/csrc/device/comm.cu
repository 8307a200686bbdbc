// comm.cu — NCCL collectives over device buffers (include/hawk_b200_comm.h).
// libnccl.so.2 is opened with dlopen at first use; if torch already mapped
// its bundled NCCL into the process, that same library is reused.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <algorithm>
#include <cstring>
#include <condition_variable>
#include <mutex>
#include <vector>
#include <string>

#include "hawk_b200.h"
#include "hawk_b200_comm.h"

// In-process loopback group: N ranks of one process (host threads) whose
// collectives are device-to-device copies between the ranks' buffers,
// sequenced by host barriers. It stands in for NCCL where only one GPU is
// present, to exercise the multi-rank exchange logic (counts, offsets,
// gather-to-root, merge) — no kernel waits on another rank's kernel.
struct hawk_loopback {
  int n = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t phase = 0;
  std::vector<const void*> send;
  std::vector<size_t> bytes;
  std::vector<void*> recv;
  std::vector<const size_t*> send_b, send_o, recv_b, recv_o;
  void barrier() {
    std::unique_lock<std::mutex> l(mu);
    const uint64_t my = phase;
    if (++arrived == n) {
      arrived = 0;
      ++phase;
      cv.notify_all();
    } else {
      cv.wait(l, [&] { return phase != my; });
    }
  }
};

struct hawk_comm {
  hawk_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  hawk_loopback* loop = nullptr;
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

int32_t hawk_loopback_group_create(int32_t nranks, hawk_loopback** out) {
  if (nranks < 1 || !out) return HAWK_ERR_ARGUMENT;
  auto* g = new hawk_loopback;
  g->n = nranks;
  g->send.assign((size_t)nranks, nullptr);
  g->bytes.assign((size_t)nranks, 0);
  g->recv.assign((size_t)nranks, nullptr);
  g->send_b.assign((size_t)nranks, nullptr);
  g->send_o.assign((size_t)nranks, nullptr);
  g->recv_b.assign((size_t)nranks, nullptr);
  g->recv_o.assign((size_t)nranks, nullptr);
  *out = g;
  return HAWK_OK;
}

int32_t hawk_loopback_group_destroy(hawk_loopback* g) {
  delete g;
  return HAWK_OK;
}

int32_t hawk_loopback_comm_create(hawk_ctx* ctx, hawk_loopback* g, int32_t rank, hawk_comm** out) {
  if (!ctx || !g || !out || rank < 0 || rank >= g->n) return HAWK_ERR_ARGUMENT;
  auto* c = new hawk_comm;
  c->ctx = ctx;
  c->loop = g;
  c->rank = rank;
  c->size = g->n;
  c->device = hawk_b200_ctx_device(ctx);
  *out = c;
  return HAWK_OK;
}

int32_t hawk_nccl_comm_rank(const hawk_comm* c) { return c ? c->rank : -1; }
int32_t hawk_nccl_comm_size(const hawk_comm* c) { return c ? c->size : 0; }
hawk_ctx* hawk_nccl_comm_ctx(const hawk_comm* c) { return c ? c->ctx : nullptr; }

namespace {
int32_t sync_stream(hawk_comm* c) {
  return cudaStreamSynchronize(stream_of(c)) == cudaSuccess ? HAWK_OK : HAWK_ERR_CUDA;
}
}  // namespace

int32_t hawk_nccl_allreduce(hawk_comm* c, const void* d_send, void* d_recv, size_t count,
                            int32_t type, int32_t op) {
  if (!c || (!d_send && count) || (!d_recv && count)) return HAWK_ERR_ARGUMENT;
  if (c->loop) {  // host reduction of every rank's values (small counts)
    hawk_loopback& g = *c->loop;
    if (sync_stream(c) != HAWK_OK) return HAWK_ERR_CUDA;
    g.send[(size_t)c->rank] = d_send;
    g.barrier();
    std::vector<int64_t> acc(count), tmp(count);
    for (int r = 0; r < g.n; ++r) {
      if (cudaMemcpy(tmp.data(), g.send[(size_t)r], count * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
        return HAWK_ERR_CUDA;
      for (size_t i = 0; i < count; ++i) {
        if (r == 0) {
          acc[i] = tmp[i];
          continue;
        }
        if (type == HAWK_F64) {
          double x, y;
          std::memcpy(&x, &acc[i], 8);
          std::memcpy(&y, &tmp[i], 8);
          const double z = op == HAWK_SUM ? x + y : op == HAWK_MIN ? std::min(x, y) : std::max(x, y);
          std::memcpy(&acc[i], &z, 8);
        } else {
          acc[i] = op == HAWK_SUM ? (int64_t)((uint64_t)acc[i] + (uint64_t)tmp[i])
                   : op == HAWK_MIN ? std::min(acc[i], tmp[i]) : std::max(acc[i], tmp[i]);
        }
      }
    }
    g.barrier();
    return cudaMemcpy(d_recv, acc.data(), count * 8, cudaMemcpyHostToDevice) == cudaSuccess ? HAWK_OK
                                                                                             : HAWK_ERR_CUDA;
  }
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
  if (c->loop) {
    hawk_loopback& g = *c->loop;
    if (sync_stream(c) != HAWK_OK) return HAWK_ERR_CUDA;
    g.send[(size_t)c->rank] = d_send;
    g.barrier();
    for (int r = 0; r < g.n; ++r)
      if (bytes && cudaMemcpy(static_cast<char*>(d_recv) + (size_t)r * bytes, g.send[(size_t)r], bytes,
                              cudaMemcpyDeviceToDevice) != cudaSuccess)
        return HAWK_ERR_CUDA;
    g.barrier();
    return HAWK_OK;
  }
  cudaSetDevice(c->device);
  return status(nccl().AllGather(d_send, d_recv, bytes, ncclUint8, c->comm, stream_of(c)));
}

int32_t hawk_nccl_bcast(hawk_comm* c, void* d_buf, size_t bytes, int32_t root) {
  if (!c || (!d_buf && bytes) || root < 0 || root >= c->size) return HAWK_ERR_ARGUMENT;
  if (c->loop) {
    hawk_loopback& g = *c->loop;
    if (sync_stream(c) != HAWK_OK) return HAWK_ERR_CUDA;
    g.recv[(size_t)c->rank] = d_buf;
    g.barrier();
    if (c->rank != root && bytes &&
        cudaMemcpy(d_buf, g.recv[(size_t)root], bytes, cudaMemcpyDeviceToDevice) != cudaSuccess)
      return HAWK_ERR_CUDA;
    g.barrier();
    return HAWK_OK;
  }
  cudaSetDevice(c->device);
  return status(nccl().Broadcast(d_buf, d_buf, bytes, ncclUint8, root, c->comm, stream_of(c)));
}

int32_t hawk_nccl_alltoall(hawk_comm* c, const void* d_send, const size_t* send_bytes,
                           const size_t* send_off, void* d_recv, const size_t* recv_bytes,
                           const size_t* recv_off) {
  if (!c || !send_bytes || !send_off || !recv_bytes || !recv_off) return HAWK_ERR_ARGUMENT;
  if (c->loop) {  // every rank pulls what each peer sends it
    hawk_loopback& g = *c->loop;
    if (sync_stream(c) != HAWK_OK) return HAWK_ERR_CUDA;
    const size_t me = (size_t)c->rank;
    g.send[me] = d_send;
    g.send_b[me] = send_bytes;
    g.send_o[me] = send_off;
    g.barrier();
    for (int p = 0; p < g.n; ++p) {
      const size_t b = g.send_b[(size_t)p][me];
      if (b != recv_bytes[p]) return HAWK_ERR_ARGUMENT;  // the peers disagree on a size
      if (b && cudaMemcpy(static_cast<char*>(d_recv) + recv_off[p],
                          static_cast<const char*>(g.send[(size_t)p]) + g.send_o[(size_t)p][me], b,
                          cudaMemcpyDeviceToDevice) != cudaSuccess)
        return HAWK_ERR_CUDA;
    }
    g.barrier();
    return HAWK_OK;
  }
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
