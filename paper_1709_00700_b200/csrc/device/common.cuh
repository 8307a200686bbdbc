// common.cuh — device-side building blocks shared by every kernel family:
// hash functions, 64-bit atomics, TMA bulk copies
// and mbarriers (sm_90+/sm_100a), warp helpers.
#pragma once

#ifndef __CUDACC_RTC__
#include <cstdint>
#endif

#include "hawk_b200.h"

namespace hk {

using u64 = unsigned long long;
using i64 = long long;

constexpr u64 kEmpty = 0x8000000000000000ull;  // HAWK_EMPTY_KEY
constexpr u64 kBusy = 2ull;                    // aggregation slot being claimed

// ---- hashing ---------------------------------------

__host__ __device__ __forceinline__ u64 fmix64(u64 k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

// Per-seed odd multiplier of multiply-shift. The reference's descriptor seeds
// are small integers (planner_pipelines.cpp:123), so they are spread over all
// 64 bits first; a small multiplier would leave the high bits (the slot) empty.
__host__ __device__ __forceinline__ u64 ms_multiplier(u64 seed) {
  return (seed * 0x9e3779b97f4a7c15ull) | 1ull;
}

// slot in [0, 2^log2cap). Murmur: fmix64(x ^ seed) masked; multiply-shift:
// (a*x mod 2^64) >> (64 - b) with a = ms_multiplier(seed) (odd), b = log2cap >= 1.
template <int HFN>
__host__ __device__ __forceinline__ u64 hash_slot(u64 x, u64 seed, int log2cap) {
  if (HFN == HAWK_MURMUR) return fmix64(x ^ seed) & ((1ull << log2cap) - 1ull);
  return (ms_multiplier(seed) * x) >> (64 - log2cap);
}

__host__ __device__ __forceinline__ u64 hash_dispatch(int fn, u64 x, u64 seed, int log2cap) {
  return fn == HAWK_MURMUR ? hash_slot<HAWK_MURMUR>(x, seed, log2cap)
                           : hash_slot<HAWK_MULTIPLY_SHIFT>(x, seed, log2cap);
}

// Combines a composite group key into one 64-bit word before hashing.
__host__ __device__ __forceinline__ u64 combine_key(u64 h, u64 k) {
  return fmix64(h + 0x9e3779b97f4a7c15ull) ^ k;
}

// ---- bit casts ---------------------------------------------------------------

__device__ __forceinline__ double as_f64(u64 b) { return __longlong_as_double((i64)b); }
__device__ __forceinline__ u64 as_bits(double d) { return (u64)__double_as_longlong(d); }

// ---- loads ---------------------------------------------------------------------

__device__ __forceinline__ u64 ldg64(const void* p) {
  return (u64)__ldg(reinterpret_cast<const i64*>(p));
}
// streaming column reads: no L1 allocation, so L1 keeps the small
// dimension structures (key bitmaps, join tables) the probes hit.
// (asm volatile: these sit under validity predicates and must not be hoisted
// speculatively past them)
// They also carry an L2 evict_first cache hint: a fact column is read once,
// and without the hint the scan evicts the dimension indexes and bitmaps the
// probes need from L2 (HK_STREAM_L2_NORMAL: plain L2 policy, for A/B).
__device__ __forceinline__ u64 l2_evict_first() {
  u64 pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ u64 ldg64_stream(const void* p) {
  u64 v;
#ifdef HK_STREAM_L2_NORMAL
  asm volatile("ld.global.nc.L1::no_allocate.b64 %0, [%1];" : "=l"(v) : "l"(p));
#else
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b64 %0, [%1], %2;"
               : "=l"(v) : "l"(p), "l"(l2_evict_first()));
#endif
  return v;
}
__device__ __forceinline__ void ldg128_stream(const void* p, u64& a, u64& b) {
#ifdef HK_STREAM_L2_NORMAL
  asm volatile("ld.global.nc.L1::no_allocate.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
#else
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.b64 {%0, %1}, [%2], %3;"
               : "=l"(a), "=l"(b) : "l"(p), "l"(l2_evict_first()));
#endif
}
// probe-side reads of small, hot structures: keep in L1
__device__ __forceinline__ u64 ldg64_keep(const void* p) {
  u64 v;
  asm volatile("ld.global.nc.L1::evict_last.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void ldg128_keep(const void* p, u64& a, u64& b) {
  asm volatile("ld.global.nc.L1::evict_last.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}
__device__ __forceinline__ void ldg128(const void* p, u64& a, u64& b) {
  longlong2 v = __ldg(reinterpret_cast<const longlong2*>(p));
  a = (u64)v.x;
  b = (u64)v.y;
}
__device__ __forceinline__ u64 ld_volatile(const u64* p) {
  return *reinterpret_cast<const volatile u64*>(p);
}
// acquire loads: a published slot tag orders the claimer's key/accumulator
// writes before our subsequent reads (generic addresses: smem or HBM)
__device__ __forceinline__ u64 ld_acquire_cta(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.cta.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 ld_acquire_gpu(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int ld_acquire_cta_i32(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta_i32(int* p, int v) {
  asm volatile("st.release.cta.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- atomics on generic addresses (smem or HBM) -------------------------------

__device__ __forceinline__ u64 atomic_cas(u64* p, u64 cmp, u64 val) { return atomicCAS(p, cmp, val); }
__device__ __forceinline__ void atomic_add_i(u64* p, u64 v) { atomicAdd(p, v); }
__device__ __forceinline__ void atomic_add_f(u64* p, double v) {
  atomicAdd(reinterpret_cast<double*>(p), v);
}
__device__ __forceinline__ void atomic_min_i(u64* p, u64 v) {
  atomicMin(reinterpret_cast<i64*>(p), (i64)v);
}
__device__ __forceinline__ void atomic_max_i(u64* p, u64 v) {
  atomicMax(reinterpret_cast<i64*>(p), (i64)v);
}
__device__ __forceinline__ void atomic_min_f(u64* p, double v) {
  u64 old = ld_volatile(p);
  while (v < as_f64(old)) {
    u64 prev = atomicCAS(p, old, as_bits(v));
    if (prev == old) break;
    old = prev;
  }
}
__device__ __forceinline__ void atomic_max_f(u64* p, double v) {
  u64 old = ld_volatile(p);
  while (v > as_f64(old)) {
    u64 prev = atomicCAS(p, old, as_bits(v));
    if (prev == old) break;
    old = prev;
  }
}

// 128-bit atomic exchange of a {key, payload} join slot (cuckoo eviction).
__device__ __forceinline__ void atomic_exch128(u64* p, u64& key, u64& payload) {
  asm volatile(
      "{\n\t.reg .b128 d, s;\n\t"
      "mov.b128 s, {%2, %3};\n\t"
      "atom.global.exch.b128 d, [%4], s;\n\t"
      "mov.b128 {%0, %1}, d;\n\t}"
      : "=l"(key), "=l"(payload)
      : "l"(key), "l"(payload), "l"(p)
      : "memory");
}

// ---- TMA bulk copies + mbarriers (cp.async.bulk, sm_90+) ------------------

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk prefetch of a global range into L2 (bytes % 16 == 0, 16B aligned)
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// global -> shared bulk copy completing on `bar` (bytes % 16 == 0, 16B aligned)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// ---- warp helpers ------------------------------------------------------------

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Member mask of the calling thread's warp: blocks may be smaller than a
// warp (work_group_size 16, thread_multiplier 1), so the last warp can be
// partial. Members are always lanes 0..n-1.
__device__ __forceinline__ unsigned warp_mask() {
  const int rem = (int)blockDim.x - (int)(threadIdx.x & ~31u);
  return rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
}
__device__ __forceinline__ int warp_size_here() {
  const int rem = (int)blockDim.x - (int)(threadIdx.x & ~31u);
  return rem >= 32 ? 32 : rem;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v, unsigned mask) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(mask, v, o);
    if (lane_id() >= o) v += n;
  }
  return v;
}

}  // namespace hk
