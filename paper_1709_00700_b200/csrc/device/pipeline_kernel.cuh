// pipeline_kernel.cuh — the kernel template: LOOP driver (coalesced with L2
// bulk prefetch, or per-thread sequential), the per-row op chain, and the
// eight sink roles.
#pragma once

#include "tables.cuh"

namespace hk {

// FILTER -> HASH_PROBE -> FILTER -> ARITHMETIC over one batch of R rows.
template <int ACCESS, int PRED, int IMPL, int HFN, int R>
__device__ __forceinline__ void evaluate(const KParams& kp, const Batch<R, ACCESS>& b,
                                         State<R>& s) {
  const hawk_pipeline& p = kp.p;
  s.alive = b.valid;
  // driver FILTER conjuncts (planner_reference.cpp:97-104)
  for (int i = 0; i < kp.npre; ++i) {
    if (PRED == HAWK_BRANCHED && s.alive == 0u) return;
    const KFilter& f = kp.pre[i];
    u64 x[R], y[R];
    fetch<PRED, R, ACCESS>(kp, f.lhs, f.type, b, s, x);
    if (f.op != kRange) fetch<PRED, R, ACCESS>(kp, f.rhs, f.type, b, s, y);
    s.alive &= compare_rows<R>(f, x, y);
  }
  // HASH_PROBE chain: branched opens a found-scope, predicated
  // folds the match bit into result_increment.
  for (int i = 0; i < p.nprobe; ++i) {
    if (PRED == HAWK_BRANCHED && s.alive == 0u) return;
    const hawk_probe& pr = p.probe[i];
    u64 k[R];
    fetch<PRED, R, ACCESS>(kp, pr.key, HAWK_I64, b, s, k);
    const hawk_table& t = p.tables[pr.table];
    int32_t r[R];
    table_find_rows<IMPL, HFN, R>(t, k, PRED == HAWK_PREDICATED ? b.valid : s.alive, r);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if (r[j] < 0) s.alive &= ~(1u << j);
      s.rid(i, j) = (u64)(r[j] < 0 ? 0 : r[j]);
    }
  }
  // post-probe FILTER conjuncts (operands may be build payloads)
  for (int i = 0; i < kp.npost; ++i) {
    if (PRED == HAWK_BRANCHED && s.alive == 0u) return;
    const KFilter& f = kp.post[i];
    u64 x[R], y[R];
    fetch<PRED, R, ACCESS>(kp, f.lhs, f.type, b, s, x);
    if (f.op != kRange) fetch<PRED, R, ACCESS>(kp, f.rhs, f.type, b, s, y);
    s.alive &= compare_rows<R>(f, x, y);
  }
  // ARITHMETIC into registers 0..narith-1
  for (int a = 0; a < p.narith; ++a) {
    if (PRED == HAWK_BRANCHED && s.alive == 0u) return;
    const hawk_arith& ar = p.arith[a];
    u64 x[R], y[R], z[R];
    fetch<PRED, R, ACCESS>(kp, ar.lhs, ar.type, b, s, x);
    fetch<PRED, R, ACCESS>(kp, ar.rhs, ar.type, b, s, y);
    arith_rows<R>(ar.op, ar.type, x, y, z);
#pragma unroll
    for (int j = 0; j < R; ++j) s.reg(a, j) = z[j];
  }
}

// A program policy gives the kernel skeleton the per-row op chain and the
// sink inputs. InterpProg interprets the lowered program from the kernel
// parameters (the AOT instantiations in libhawk_b200.so); a compiled policy
// (jit.cpp) is generated per pipeline with the same interface, constants
// inlined and per-row values in registers.
struct InterpProg {
  static constexpr bool kStatic = false;  // program shape known only at run time
  static constexpr bool kSplit = false;   // no live-row compaction after the first probe
  static constexpr int kDrain = 1;        // (queued rows per lane per drain)
  static constexpr int kBlock = 0;        // block size known only at run time
  template <int R>
  struct Vals {};
  template <int ACCESS, int PRED, int IMPL, int HFN, int R>
  __device__ static __forceinline__ void eval(const KParams& kp, const Batch<R, ACCESS>& b,
                                              State<R>& s, Vals<R>&) {
    evaluate<ACCESS, PRED, IMPL, HFN, R>(kp, b, s);
  }
  template <int ACCESS, int PRED, int R>
  __device__ static __forceinline__ void agg_input(const KParams& kp, int a,
                                                   const Batch<R, ACCESS>& b, const State<R>& s,
                                                   const Vals<R>&, u64 (&v)[R]) {
    fetch<PRED, R, ACCESS>(kp, kp.p.aggs[a].input, kp.p.aggs[a].type, b, s, v);
  }
  template <int ACCESS, int PRED, int R>
  __device__ static __forceinline__ void key_input(const KParams& kp, int i,
                                                   const Batch<R, ACCESS>& b, const State<R>& s,
                                                   const Vals<R>&, u64 (&v)[R]) {
    fetch<PRED, R, ACCESS>(kp, kp.p.keys[i], HAWK_I64, b, s, v);
  }
  template <int ACCESS, int PRED, int R>
  __device__ static __forceinline__ void proj_input(const KParams& kp, int i,
                                                    const Batch<R, ACCESS>& b, const State<R>& s,
                                                    const Vals<R>&, u64 (&v)[R]) {
    fetch<PRED, R, ACCESS>(kp, kp.p.project[i], kp.p.project[i].type, b, s, v);
  }
};

// ---- sinks of compiled programs: the shape (keys, aggregates, functions) is
// static, so keys stay in registers and every aggregate update is specialised

template <int V>
struct IntC {
  static constexpr int value = V;
};
template <int I, int N>
struct StaticFor {
  template <class F>
  __device__ __forceinline__ static void run(F&& f) {
    if constexpr (I < N) {
      f(IntC<I>{});
      StaticFor<I + 1, N>::run(f);
    }
  }
};

// agg_find_or_insert with K keys held in registers
template <int IMPL, int HFN, bool SHARED, int K>
__device__ __forceinline__ u64* agg_find_static(const KParams& kp, u64* slots, int log2cap,
                                               const uint64_t* seeds, const u64 (&key)[K],
                                               u64* fresh_counter, int* out_pos) {
  const hawk_pipeline& p = kp.p;
  const int words = 1 + K + p.naggs;
  u64 x = key[0];
#pragma unroll
  for (int i = 1; i < K; ++i) x = combine_key(x, key[i]);
  const u64 h = HFN == HAWK_MURMUR ? fmix64(x ^ seeds[0]) : ms_multiplier(seeds[0]) * x;
  const u64 tag = h | 1ull;
  const u64 cap = 1ull << log2cap;
  // cuckoo aggregation tables are bucketised: each of the two candidate
  // positions opens a run of kAggBucket slots (groups are never moved, since
  // other threads update their accumulators in place)
  const int max_tries = IMPL == HAWK_LINEAR_PROBING ? (int)(cap < 4096 ? cap : 4096) : 2 * kAggBucket;
  const u64 home = HFN == HAWK_MURMUR ? (h & (cap - 1ull)) : (h >> (64 - log2cap));
  u64 pos = home;
  for (int t = 0; t < max_tries; ++t) {
    if (IMPL == HAWK_CUCKOO)
      pos = t < kAggBucket ? ((home + (u64)t) & (cap - 1ull))
                           : cap + ((hash_slot<HFN>(x, seeds[1], log2cap) + (u64)(t - kAggBucket)) & (cap - 1ull));
    u64* sl = slots + pos * (u64)words;
    u64 st = SHARED ? ld_acquire_cta(sl) : ld_acquire_gpu(sl);
    if (st == 0ull) {
      const u64 prev = atomicCAS(sl, 0ull, kBusy);
      if (prev == 0ull) {
#pragma unroll
        for (int i = 0; i < K; ++i) sl[1 + i] = key[i];
        for (int a = 0; a < p.naggs; ++a) sl[1 + K + a] = agg_identity(p.aggs[a].fn, p.aggs[a].type);
        if (SHARED) __threadfence_block(); else __threadfence();
        atomicExch(sl, tag);
        if (fresh_counter) atomicAdd(fresh_counter, 1ull);
        if (out_pos) *out_pos = (int)pos;
        return sl;
      }
      st = prev;
    }
    while (st == kBusy) st = SHARED ? ld_acquire_cta(sl) : ld_acquire_gpu(sl);
    if (st == tag) {
      bool eq = true;
#pragma unroll
      for (int i = 0; i < K; ++i) eq &= ld_volatile(sl + 1 + i) == key[i];
      if (eq) {
        if (out_pos) *out_pos = (int)pos;
        return sl;
      }
    }
    if (IMPL == HAWK_LINEAR_PROBING) pos = (pos + 1) & (cap - 1ull);
  }
  return nullptr;
}

// Dense group ordinal of a CTA-table slot: exactly one thread per group (the
// one that moves the slot from -1 to -2) draws the next ordinal.
__device__ __forceinline__ int claim_ordinal(int* ordinal, int si, int* ord_slot, int* nord, int GP) {
  volatile int* ov = reinterpret_cast<volatile int*>(ordinal + si);
  int o = *ov;
  if (o < 0) {
    if (o == -1 && atomicCAS(ordinal + si, -1, -2) == -1) {
      const int mine = atomicAdd(nord, 1);
      o = mine < GP ? mine : GP;
      if (o < GP) ord_slot[o] = si;
      __threadfence_block();
      *ov = o;
    } else {
      while ((o = *ov) < 0) {
      }
    }
  }
  return o;
}

template <class P, int ROLE, int ACCESS, int PRED, int IMPL, int HFN, int R>
__device__ __forceinline__ void hagg_static(const KParams& kp, const Batch<R, ACCESS>& b,
                                            const State<R>& s,
                                            const typename P::template Vals<R>& vals,
                                            u64* local_table, int* ordinal, int* ord_slot,
                                            int* nord, u64* priv, int GP, int* dense_ord,
                                            u64 (&last_key)[HAWK_MAX_KEYS], u64& last_target) {
  constexpr int K = P::kKeys, A = P::kAggs;
  const int B = P::kBlock > 0 ? P::kBlock : (int)blockDim.x;
  const uint32_t alive = s.alive;
  const hawk_table& gt = kp.p.sink_table;
  u64 key[K][R];
  StaticFor<0, K>::run([&](auto ic) {
    constexpr int i = decltype(ic)::value;
    P::template key_value<i, ACCESS, PRED, R>(kp, b, s, vals, key[i]);
  });
  // target per row: private word offset ((ord*A*B + t) << 1 | 1), slot, or 0
  u64 tw[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    u64 target = 0;
    if ((alive >> j) & 1u) {
      u64 kj[K];
#pragma unroll
      for (int i = 0; i < K; ++i) kj[i] = key[i][j];
      bool same = last_target != 0;
#pragma unroll
      for (int i = 0; i < K; ++i) same &= kj[i] == last_key[i];
      if (same) {
        target = last_target;
      } else {
        // small key domains: the dense index of the key tuple caches its
        // group ordinal (a CTA-wide lookaside in front of the hash table)
        int d = -1;
        if constexpr (ROLE == K_HAGG_LOCAL) {
          if (dense_ord != nullptr) {
            u64 idx = 0;
            bool in = true;
#pragma unroll
            for (int i = 0; i < K; ++i) {
              const u64 r = kj[i] - (u64)kp.p.key_lo[i];
              in &= r < (u64)kp.p.key_span[i];
              idx += r * (u64)kp.p.key_stride[i];
            }
            if (in) {
              d = (int)idx;
              HK_CHECK(kp, d < kp.p.dense_groups);
              // GP > 0: private accumulators are thread-owned and need no
              // ordering; GP == 0: the CTA slot's contents must be visible
              const int o = GP > 0 ? *reinterpret_cast<volatile int*>(dense_ord + d)
                                   : ld_acquire_cta_i32(dense_ord + d);
              // GP > 0: o is the group's ordinal (thread-private accumulators);
              // GP == 0: o is its slot in the CTA table (shared-memory atomics)
              if (o >= 0)
                target = GP > 0 ? ((((u64)o * A * B) + threadIdx.x) << 1) | 1ull
                                : ((u64)o << 2) | 2ull;
            }
          }
        }
        u64* slot = nullptr;
        if constexpr (ROLE == K_HAGG_LOCAL) {
          if (target == 0) {
            int si = 0;
            slot = agg_find_static<IMPL, HFN, true, K>(kp, local_table, kp.local_log2, gt.seed, kj,
                                                       nullptr, &si);
            if (slot != nullptr && GP > 0) {
              const int o = claim_ordinal(ordinal, si, ord_slot, nord, GP);
              if (o < GP) {
                target = ((((u64)o * A * B) + threadIdx.x) << 1) | 1ull;
                if (d >= 0) st_release_cta_i32(dense_ord + d, o);  // every writer stores the same ordinal
              }
            } else if (slot != nullptr && d >= 0) {
              st_release_cta_i32(dense_ord + d, si);  // every writer stores the same slot
            }
            // GP == 0: a CTA-table slot (shared-memory atomics); GP > 0 keeps
            // its rare ordinal-overflow rows on the generic path below
            if (slot != nullptr && target == 0 && GP == 0) target = ((u64)si << 2) | 2ull;
          }
        }
        if (target == 0) {
          if (slot == nullptr)
            slot = agg_find_static<IMPL, HFN, false, K>(kp, reinterpret_cast<u64*>(gt.d_slots),
                                                        gt.log2_capacity, gt.seed, kj,
                                                        kp.d_cursor, nullptr);
          if (slot == nullptr) atomicOr(kp.d_flags, HAWK_FLAG_TABLE_FULL);
          target = reinterpret_cast<u64>(slot);
        }
#pragma unroll
        for (int i = 0; i < K; ++i) last_key[i] = kj[i];
        last_target = target;
      }
    }
    tw[j] = target;
  }
  // target encoding: (offset << 1) | 1 = private accumulators (plain
  // shared-memory read-modify-write, predicated, no branches); (slot << 2) |
  // 2 = a CTA-table slot (shared-memory atomics); else a global-table slot
  // pointer (HBM atomics); 0 = no row
  uint32_t pmask = 0, smask = 0, gmask = 0;
  u64 off[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    pmask |= (uint32_t)(tw[j] & 1ull) << j;
    if (GP == 0) smask |= (uint32_t)((tw[j] & 3ull) == 2ull) << j;
    gmask |= (uint32_t)(tw[j] != 0ull && (tw[j] & 3ull) == 0ull) << j;
    off[j] = tw[j] >> 1;
  }
  const uint32_t local_base = smem_addr(local_table);
#ifdef HK_CHECKED
#pragma unroll
  for (int j = 0; j < R; ++j) {  // private words and CTA-table slots inside their arrays
    HK_CHECK(kp, !((pmask >> j) & 1u) || off[j] < (u64)GP * A * B);
    HK_CHECK(kp, !((smask >> j) & 1u) || (tw[j] >> 2) < (u64)(1 << kp.local_log2) * (IMPL == HAWK_CUCKOO ? 2 : 1));
  }
#endif
  if constexpr (ROLE == K_HAGG_LOCAL) {
    // Fast path: every live row of the batch has thread-private accumulators
    // (TPC-H Q1 after each CTA's first rows). Branch-free: rows that are not
    // live add the aggregate's identity to a live row's accumulators, and the
    // loop runs rows outermost, so each row reads all of its A accumulators
    // before writing any: the shared-memory read-modify-writes of one row
    // overlap instead of forming one chain through every (aggregate, row).
    uint32_t live = 0;
#pragma unroll
    for (int j = 0; j < R; ++j) live |= (uint32_t)(tw[j] != 0ull) << j;
    if (GP > 0 && live != 0u && pmask == live) {
      const int first = __ffs(live) - 1;
      u64 any_off = off[0];
#pragma unroll
      for (int j = R - 1; j >= 0; --j)
        if (j == first) any_off = off[j];
      u64 av[A][R];
      StaticFor<0, A>::run([&](auto ac) {
        constexpr int a = decltype(ac)::value;
        constexpr int fn = P::kAggFn[a], ty = P::kAggType[a];
        if constexpr (fn == HAWK_COUNT) {
#pragma unroll
          for (int j = 0; j < R; ++j) av[a][j] = (live >> j) & 1u;
        } else {
          P::template agg_value<a, ACCESS, PRED, R>(kp, b, s, vals, av[a]);
          const u64 id = agg_identity(fn, ty);
#pragma unroll
          for (int j = 0; j < R; ++j) av[a][j] = ((live >> j) & 1u) ? av[a][j] : id;
        }
      });
#pragma unroll
      for (int j = 0; j < R; ++j) {
        u64* base = priv + (((live >> j) & 1u) ? off[j] : any_off);
        u64 acc[A];
#pragma unroll
        for (int a = 0; a < A; ++a) acc[a] = base[(size_t)a * B];
        StaticFor<0, A>::run([&](auto ac) {
          constexpr int a = decltype(ac)::value;
          constexpr int fn = P::kAggFn[a], ty = P::kAggType[a];
          if constexpr (fn == HAWK_COUNT || (fn == HAWK_SUM && ty == HAWK_I64)) acc[a] += av[a][j];
          else acc[a] = agg_combine(fn, ty, acc[a], av[a][j]);
        });
#pragma unroll
        for (int a = 0; a < A; ++a) base[(size_t)a * B] = acc[a];
      }
      return;
    }
  }
  StaticFor<0, A>::run([&](auto ac) {
    constexpr int a = decltype(ac)::value;
    constexpr int fn = P::kAggFn[a], ty = P::kAggType[a];
    u64 v[R];
    if constexpr (fn == HAWK_COUNT) {
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = 1ull;
    } else {
      P::template agg_value<a, ACCESS, PRED, R>(kp, b, s, vals, v);
    }
    u64* pa = priv + (size_t)a * B;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if ((pmask >> j) & 1u) {
        u64& acc = pa[off[j]];
        if constexpr (fn == HAWK_COUNT || (fn == HAWK_SUM && ty == HAWK_I64)) acc += v[j];
        else acc = agg_combine(fn, ty, acc, v[j]);
      }
    }
    if (smask) {
#pragma unroll
      for (int j = 0; j < R; ++j)
        if ((smask >> j) & 1u)
          agg_update_smem<fn, ty>(local_base + (uint32_t)(((tw[j] >> 2) * (1 + K + A) + 1 + K + a) * 8), v[j]);
    }
    if (gmask) {
#pragma unroll
      for (int j = 0; j < R; ++j)
        if ((gmask >> j) & 1u) agg_update(reinterpret_cast<u64*>(tw[j]) + 1 + K + a, fn, ty, v[j]);
    }
  });
}

template <class P, int ACCESS, int PRED, int R>
__device__ __forceinline__ void agg_static(const KParams& kp, const Batch<R, ACCESS>& b,
                                           State<R>& s, const typename P::template Vals<R>& vals) {
  const uint32_t alive = s.alive;
  StaticFor<0, P::kAggs>::run([&](auto ac) {
    constexpr int a = decltype(ac)::value;
    constexpr int fn = P::kAggFn[a], ty = P::kAggType[a];
    u64& acc = s.acc(a);
    if constexpr (fn == HAWK_COUNT) {
      acc += (u64)__popc(alive);
    } else {
      u64 v[R];
      P::template agg_value<a, ACCESS, PRED, R>(kp, b, s, vals, v);
      if constexpr (fn == HAWK_SUM && ty == HAWK_I64) {
        u64 sum = 0;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          if (PRED == HAWK_PREDICATED) sum += v[j] * (u64)((alive >> j) & 1u);
          else if ((alive >> j) & 1u) sum += v[j];
        }
        acc += sum;
      } else {
        u64 x = acc;
#pragma unroll
        for (int j = 0; j < R; ++j)
          if ((alive >> j) & 1u) x = agg_combine(fn, ty, x, v[j]);
        acc = x;
      }
    }
  });
}

// block-wide exclusive scan of one 64-bit value per thread; returns the
// exclusive prefix and writes the block total. Uses `scratch` (>= 33 words).
__device__ __forceinline__ u64 block_exclusive_scan(u64 v, u64* scratch, u64& total) {
  const int lane = lane_id(), warp = threadIdx.x >> 5;
  const int nwarps = (blockDim.x + 31) >> 5;
  const unsigned mask = warp_mask();
  u64 incl = warp_incl_scan<u64>(v, mask);
  if (lane == warp_size_here() - 1) scratch[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    u64 w = lane < nwarps ? scratch[lane] : 0ull;
    u64 wi = warp_incl_scan<u64>(w, mask);
    if (lane < nwarps) scratch[lane] = wi - w;
    if (lane == warp_size_here() - 1) scratch[32] = wi;
  }
  __syncthreads();
  const u64 excl = scratch[warp] + incl - v;
  total = scratch[32];
  __syncthreads();
  return excl;
}


template <class T>
struct Plain {
  using type = T;
};
template <class T>
struct Plain<T&> {
  using type = T;
};
template <class T>
struct Plain<const T> {
  using type = T;
};
template <class T>
struct Plain<const T&> {
  using type = T;
};

// PROJECT, single pass (compiled programs): warp-aggregated atomic cursor
template <class P, int ACCESS, int PRED, int R>
__device__ __forceinline__ void project_static(const KParams& kp, const Batch<R, ACCESS>& b,
                                               const State<R>& s,
                                               const typename P::template Vals<R>& vals) {
  const uint32_t alive = s.alive;
  const unsigned mask = warp_mask();
  const int last = warp_size_here() - 1;
  const uint32_t cnt = (uint32_t)__popc(alive);
  const uint32_t incl = warp_incl_scan<uint32_t>(cnt, mask);
  const uint32_t tot = __shfl_sync(mask, incl, last);
  u64 base = 0;
  if (lane_id() == last && tot) base = atomicAdd(kp.d_cursor, (u64)tot);
  base = __shfl_sync(mask, base, last);
  if (cnt) {
    const u64 pos = base + incl - cnt;
    for (int i = 0; i < kp.p.nproject; ++i) {
      u64 v[R];
      P::template proj_input<ACCESS, PRED, R>(kp, i, b, s, vals, v);
      int64_t* out = kp.d_out + (size_t)i * kp.out_stride + pos;
      int k = 0;
#pragma unroll
      for (int j = 0; j < R; ++j)
        if ((alive >> j) & 1u) out[k++] = (int64_t)v[j];
    }
  }
}

// Live-row compaction (compiled, branched): the filters and the first (most
// selective) probe run on the pass's R rows per thread; the surviving rows of
// the warp are appended to a per-warp queue (row, probe-0 row id) in shared
// memory. Once the queue holds D rows per lane it is drained: the rest of the
// chain + the sink run on D queued rows per lane (P::kDrain), so every
// dependent step of the remaining probe chain (gather the key, look it up,
// gather the payload) has D independent loads in flight per lane instead of
// one, and later probes issue instructions for live rows only (SSB Q4.1: 20%
// of the rows survive the first probe). The tail drains after the LOOP.
template <class P, int ROLE, int PRED, int IMPL, int HFN, int D, class Sink, class St>
__device__ __forceinline__ void drain_rows(const KParams& kp, const St& s, uint2* q, uint32_t first,
                                           uint32_t n, int64_t cb, int B, Sink& sink) {
  Batch<D, kGather> g;
  g.base = cb;
  g.B = B;
  g.stage = nullptr;
  g.valid = 0;
  typename P::template Vals<D> v;
  const uint32_t lanes = (uint32_t)warp_size_here();
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const uint32_t idx = first + (uint32_t)j * lanes + (uint32_t)lane_id();
    const bool ok = idx < first + n;
    const uint2 e = ok ? q[idx] : make_uint2(0u, 0u);
    g.valid |= (uint32_t)ok << j;
    g.rows_[j] = cb + (int64_t)e.x;
    v.p0[j] = (int32_t)e.y;
  }
  State<D> s1;
  s1.ts = s.ts;
  s1.B = s.B;
  s1.tid = s.tid;
  s1.rid_base = s.rid_base;
  s1.key_base = s.key_base;
  s1.acc_base = s.acc_base;
  s1.alive = g.valid;  // (lanes without rows still reach the sink's warp collectives)
  P::template eval2<kGather, PRED, IMPL, HFN, D>(kp, g, s1, v);
  sink(g, s1, v);
}

template <class P, int ROLE, int ACCESS, int PRED, int IMPL, int HFN, int R, class Sink>
__device__ __forceinline__ void split_rows(const KParams& kp, const Batch<R, ACCESS>& b,
                                           State<R>& s, typename P::template Vals<R>& vals,
                                           int64_t cb, int B, uint2* q, uint32_t& qn, Sink& sink) {
  constexpr int D = P::kDrain;
  P::template eval1<ACCESS, PRED, IMPL, HFN, R>(kp, b, s, vals);
  const uint32_t alive = s.alive;
  const unsigned mask = warp_mask();
  const int last = warp_size_here() - 1;
  const uint32_t c = (uint32_t)__popc(alive);
  const uint32_t incl = warp_incl_scan<uint32_t>(c, mask);
  const uint32_t total = __shfl_sync(mask, incl, last);
  if (total == 0u) return;
  uint32_t pos = qn + incl - c;
  HK_CHECK(kp, qn + total <= (uint32_t)(32 * (R + D)));  // the warp's queue capacity
#pragma unroll
  for (int j = 0; j < R; ++j)
    if ((alive >> j) & 1u) q[pos++] = make_uint2((uint32_t)(b.row(j) - cb), (uint32_t)vals.p0[j]);
  qn += total;
  __syncwarp(mask);
  const uint32_t batch = (uint32_t)D * (uint32_t)(last + 1);
  if (qn < batch) return;
  uint32_t first = 0;
  while (qn - first >= batch) {
    drain_rows<P, ROLE, PRED, IMPL, HFN, D>(kp, s, q, first, batch, cb, B, sink);
    first += batch;
  }
  // move the remainder (< one batch) to the front of the queue
  const uint32_t rest = qn - first;
  __syncwarp(mask);
  uint2 tmp[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const uint32_t idx = (uint32_t)j * (uint32_t)(last + 1) + (uint32_t)lane_id();
    if (idx < rest) tmp[j] = q[first + idx];
  }
  __syncwarp(mask);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const uint32_t idx = (uint32_t)j * (uint32_t)(last + 1) + (uint32_t)lane_id();
    if (idx < rest) q[idx] = tmp[j];
  }
  __syncwarp(mask);
  qn = rest;
}

template <class P, int ROLE, int ACCESS, int PRED, int IMPL, int HFN, int U>
__device__ __forceinline__ void pipeline_body(const KParams& kp) {
  constexpr int R = 4 * U;
  typename P::template Vals<R> vals;
  extern __shared__ __align__(128) unsigned char smem[];
  const hawk_pipeline& p = kp.p;
  const int B = P::kBlock > 0 ? P::kBlock : (int)blockDim.x;  // static for compiled programs
  const int64_t cb = min(p.nrows, (int64_t)blockIdx.x * kp.chunk_rows);
  const int64_t ce = min(p.nrows, cb + kp.chunk_rows);
  u64* scratch = reinterpret_cast<u64*>(smem + kp.smem_scratch_off);

  State<R> s;
  s.ts = reinterpret_cast<u64*>(smem + kp.smem_state_off);
  s.B = B;
  s.tid = threadIdx.x;
  s.rid_base = kp.rid_base;
  s.key_base = kp.key_base;
  s.acc_base = kp.acc_base;
  s.alive = 0;

  // ---- sink state ----
  if constexpr (ROLE == K_AGG_LOCAL || ROLE == K_AGG_GLOBAL) {
    for (int a = 0; a < p.naggs; ++a) s.acc(a) = agg_identity(p.aggs[a].fn, p.aggs[a].type);
  }
  u64 count = 0;    // COUNT role
  u64 running = 0;  // SCATTER role: rows written by this CTA so far
  u64* local_table = reinterpret_cast<u64*>(smem + kp.smem_table_off);
  const int K = p.nkeys;
  const int words = 1 + p.nkeys + p.naggs;
  // HAGG_LOCAL: the first priv_groups groups a CTA meets get dense ordinals
  // and thread-private accumulators (plain shared-memory read-modify-write,
  // no atomics); the CTA folds them into its table at the end. Low-cardinality
  // group-bys (TPC-H Q1: 4 groups) otherwise serialise on a few atomics.
  const int GP = ROLE == K_HAGG_LOCAL ? kp.priv_groups : 0;
  const int A = p.naggs;
  const int local_slots = (1 << kp.local_log2) * (IMPL == HAWK_CUCKOO ? 2 : 1);
  int* ordinal = reinterpret_cast<int*>(smem + kp.smem_ord_off);  // [local_slots]
  int* ord_slot = ordinal + local_slots;                           // [GP]
  int* nord = ord_slot + GP;                                       // [1]
  u64* priv = reinterpret_cast<u64*>(smem + kp.smem_priv_off);
  int* dense_ord = kp.smem_dense_off > 0 ? reinterpret_cast<int*>(smem + kp.smem_dense_off) : nullptr;
  if constexpr (ROLE == K_HAGG_LOCAL) {
    if (dense_ord != nullptr)
      for (int i = threadIdx.x; i < p.dense_groups; i += B) dense_ord[i] = -1;
    for (int i = threadIdx.x; i < local_slots; i += B) local_table[(size_t)i * words] = 0ull;
    if (GP > 0) {
      for (int i = threadIdx.x; i < local_slots; i += B) ordinal[i] = -1;
      for (int i = threadIdx.x; i < GP; i += B) ord_slot[i] = -1;
      if (threadIdx.x == 0) *nord = 0;
      for (int w = 0; w < GP * A; ++w)
        priv[(size_t)w * B + threadIdx.x] = agg_identity(p.aggs[w % A].fn, p.aggs[w % A].type);
    }
    __syncthreads();
  }
  u64 scatter_base = 0;
  if constexpr (ROLE == K_PROJECT_SCATTER) scatter_base = (u64)kp.d_offsets[blockIdx.x];
  u64 last_key[HAWK_MAX_KEYS] = {0, 0, 0, 0};  // HAGG: the thread's last group
  u64 last_target = 0;

  // sinks of compiled programs for any batch shape (R rows / compacted rows)
  auto sink_static = [&](const auto& bb, auto& ss, auto& vv) {
    using BT = typename Plain<decltype(bb)>::type;
    constexpr int RR = BT::kR, AA = BT::kAccess;
    if constexpr (ROLE == K_AGG_LOCAL || ROLE == K_AGG_GLOBAL) {
      if (ss.alive == 0u) return;
      agg_static<P, AA, PRED, RR>(kp, bb, ss, vv);
    } else if constexpr (ROLE == K_HAGG_LOCAL || ROLE == K_HAGG_GLOBAL) {
      if (ss.alive == 0u) return;
      hagg_static<P, ROLE, AA, PRED, IMPL, HFN, RR>(kp, bb, ss, vv, local_table, ordinal, ord_slot,
                                                    nord, priv, GP, dense_ord, last_key,
                                                    last_target);
    } else if constexpr (ROLE == K_PROJECT_SINGLE) {
      project_static<P, AA, PRED, RR>(kp, bb, ss, vv);
    }
  };
  // live-row compaction queue of this warp (compiled, branched programs)
  constexpr bool kSplitRows = P::kSplit && PRED == HAWK_BRANCHED &&
                              (ROLE <= K_HAGG_GLOBAL || ROLE == K_PROJECT_SINGLE);
  uint2* split_q = reinterpret_cast<uint2*>(smem + kp.smem_queue_off) +
                   (threadIdx.x >> 5) * (32 * (R + P::kDrain));
  uint32_t split_n = 0;
  auto process = [&](const Batch<R, ACCESS>& b) {
    if constexpr (kSplitRows) {
      split_rows<P, ROLE, ACCESS, PRED, IMPL, HFN, R>(kp, b, s, vals, cb, B, split_q, split_n,
                                                      sink_static);
      return;
    }
    P::template eval<ACCESS, PRED, IMPL, HFN, R>(kp, b, s, vals);
    const uint32_t alive = s.alive;
    if constexpr (ROLE == K_AGG_LOCAL || ROLE == K_AGG_GLOBAL) {
      // AGGREGATE: predicated SUM/COUNT multiply by the
      // 0/1 result_increment, MIN/MAX select.
      if (PRED == HAWK_BRANCHED && alive == 0u) return;
      if constexpr (P::kStatic) {
        agg_static<P, ACCESS, PRED, R>(kp, b, s, vals);
        return;
      }
      for (int a = 0; a < p.naggs; ++a) {
        const hawk_agg& g = p.aggs[a];
        u64& acc = s.acc(a);
        if (g.fn == HAWK_COUNT) {
          acc += (u64)__popc(alive);
          continue;
        }
        u64 v[R];
        P::template agg_input<ACCESS, PRED, R>(kp, a, b, s, vals, v);
        if (g.fn == HAWK_SUM && g.type == HAWK_I64) {
          u64 sum = 0;
#pragma unroll
          for (int j = 0; j < R; ++j) {
            if (PRED == HAWK_PREDICATED) sum += v[j] * (u64)((alive >> j) & 1u);
            else if ((alive >> j) & 1u) sum += v[j];
          }
          acc += sum;
        } else {
          u64 x = acc;
#pragma unroll
          for (int j = 0; j < R; ++j)
            if ((alive >> j) & 1u) x = agg_combine(g.fn, g.type, x, v[j]);
          acc = x;
        }
      }
    } else if constexpr (ROLE == K_HAGG_LOCAL || ROLE == K_HAGG_GLOBAL) {
      if (PRED == HAWK_BRANCHED && alive == 0u) return;
      if constexpr (P::kStatic) {
        hagg_static<P, ROLE, ACCESS, PRED, IMPL, HFN, R>(kp, b, s, vals, local_table, ordinal,
                                                         ord_slot, nord, priv, GP, dense_ord,
                                                         last_key, last_target);
        return;
      }
      for (int i = 0; i < K; ++i) {
        u64 v[R];
        P::template key_input<ACCESS, PRED, R>(kp, i, b, s, vals, v);
#pragma unroll
        for (int j = 0; j < R; ++j) s.key(i, j) = v[j];
      }
      // find or claim each alive row's group; slot pointers go to the
      // per-thread state (rows are not unrolled here: the probe sequence is
      // data dependent and inlining it R times would only add registers)
      const hawk_table& gt = p.sink_table;
      const int kstride = R * B;
#pragma unroll 1
      for (int j = 0; j < R; ++j) {
        u64 target = 0;  // slot pointer (even), (ordinal << 1) | 1 (private), 0 (none)
        if ((alive >> j) & 1u) {
          const u64* kj = &s.key(0, j);
          // consecutive rows of one group skip the table lookup
          bool same = last_target != 0;
#pragma unroll
          for (int i = 0; i < HAWK_MAX_KEYS; ++i)
            if (i < K) same &= kj[(size_t)i * kstride] == last_key[i];
          if (same) {
            s.rid(p.nprobe, j) = last_target;
            continue;
          }
          u64* slot = nullptr;
          if constexpr (ROLE == K_HAGG_LOCAL) {
            int si = 0;
            slot = agg_find_or_insert<IMPL, HFN, true>(kp, local_table, kp.local_log2, gt.seed,
                                                      kj, kstride, nullptr, &si);
            if (slot != nullptr && GP > 0) {
              // dense ordinals: exactly one thread per group (the one that
              // moves the slot from -1 to -2) draws the next ordinal
              volatile int* ov = reinterpret_cast<volatile int*>(ordinal + si);
              int o = *ov;
              if (o < 0) {
                if (o == -1 && atomicCAS(ordinal + si, -1, -2) == -1) {
                  const int mine = atomicAdd(nord, 1);
                  o = mine < GP ? mine : GP;
                  if (o < GP) ord_slot[o] = si;
                  __threadfence_block();
                  *ov = o;
                } else {
                  while ((o = *ov) < 0) {
                  }
                }
              }
              if (o < GP) target = ((u64)o << 1) | 1ull;
            }
          }
          if (target == 0 && slot == nullptr)
            slot = agg_find_or_insert<IMPL, HFN, false>(
                kp, reinterpret_cast<u64*>(gt.d_slots), gt.log2_capacity, gt.seed, kj, kstride,
                kp.d_cursor);
          if (target == 0) {
            if (slot == nullptr) atomicOr(kp.d_flags, HAWK_FLAG_TABLE_FULL);
            target = reinterpret_cast<u64>(slot);
          }
#pragma unroll
          for (int i = 0; i < HAWK_MAX_KEYS; ++i)
            if (i < K) last_key[i] = kj[(size_t)i * kstride];
          last_target = target;
        }
        s.rid(p.nprobe, j) = target;  // the row after the probe ids
      }
      // targets of the R rows: private word offset ((ord*A*B + t) << 1 | 1),
      // a slot pointer, or 0; loaded once for all aggregates
      u64 tw[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const u64 t = s.rid(p.nprobe, j);
        tw[j] = (t & 1ull) ? ((((t >> 1) * (u64)A * (u64)B + threadIdx.x) << 1) | 1ull) : t;
      }
      for (int a = 0; a < A; ++a) {
        const hawk_agg& g = p.aggs[a];
        u64* pa = priv + (size_t)a * B;
        const int agg_word = 1 + K + a;
        if (g.fn == HAWK_COUNT || (g.fn == HAWK_SUM && g.type == HAWK_I64)) {
          // the hot case (TPC-H Q1: 5 SUMs + 1 COUNT): add, no dispatch per row
          u64 v[R];
          if (g.fn == HAWK_COUNT) {
#pragma unroll
            for (int j = 0; j < R; ++j) v[j] = 1ull;
          } else {
            P::template agg_input<ACCESS, PRED, R>(kp, a, b, s, vals, v);
          }
#pragma unroll
          for (int j = 0; j < R; ++j) {
            if (tw[j] & 1ull) pa[tw[j] >> 1] += v[j];
            else if (tw[j]) atomic_add_i(reinterpret_cast<u64*>(tw[j]) + agg_word, v[j]);
          }
        } else {
          u64 v[R];
          P::template agg_input<ACCESS, PRED, R>(kp, a, b, s, vals, v);
#pragma unroll
          for (int j = 0; j < R; ++j) {
            if (tw[j] & 1ull) {
              u64& acc = pa[tw[j] >> 1];
              acc = agg_combine(g.fn, g.type, acc, v[j]);
            } else if (tw[j]) {
              agg_update(reinterpret_cast<u64*>(tw[j]) + agg_word, g.fn, g.type, v[j]);
            }
          }
        }
      }
    } else if constexpr (ROLE == K_PROJECT_SINGLE) {
      // single pass: warp-aggregated atomic output cursor
      const unsigned mask = warp_mask();
      const int last = warp_size_here() - 1;
      const uint32_t cnt = (uint32_t)__popc(alive);
      const uint32_t incl = warp_incl_scan<uint32_t>(cnt, mask);
      const uint32_t tot = __shfl_sync(mask, incl, last);
      u64 base = 0;
      if (lane_id() == last && tot) base = atomicAdd(kp.d_cursor, (u64)tot);
      base = __shfl_sync(mask, base, last);
      if (cnt) {
        const u64 pos = base + incl - cnt;
        for (int i = 0; i < p.nproject; ++i) {
          u64 v[R];
          P::template proj_input<ACCESS, PRED, R>(kp, i, b, s, vals, v);
          int64_t* out = kp.d_out + (size_t)i * kp.out_stride + pos;
          int k = 0;
#pragma unroll
          for (int j = 0; j < R; ++j)
            if ((alive >> j) & 1u) out[k++] = (int64_t)v[j];
        }
      }
    } else if constexpr (ROLE == K_COUNT) {
      count += (u64)__popc(alive);
    } else if constexpr (ROLE == K_PROJECT_SCATTER) {
      const u64 cnt = (u64)__popc(alive);
      u64 total;
      const u64 excl = block_exclusive_scan(cnt, scratch, total);
      if (cnt) {
        const u64 pos = scatter_base + running + excl;
        for (int i = 0; i < p.nproject; ++i) {
          u64 v[R];
          P::template proj_input<ACCESS, PRED, R>(kp, i, b, s, vals, v);
          int64_t* out = kp.d_out + (size_t)i * kp.out_stride + pos;
          int k = 0;
#pragma unroll
          for (int j = 0; j < R; ++j)
            if ((alive >> j) & 1u) out[k++] = (int64_t)v[j];
        }
      }
      running += total;
    } else if constexpr (ROLE == K_PUT_SINGLE) {
      {  // inserted-row count (the engine orders probes by build selectivity)
        const unsigned mask = warp_mask();
        const unsigned n = __reduce_add_sync(mask, (unsigned)__popc(alive));
        if (lane_id() == 0 && n) atomicAdd(kp.d_cursor, (u64)n);
      }
      if (PRED == HAWK_BRANCHED && alive == 0u) return;
      u64 key[R], rid[R];
      P::template key_input<ACCESS, PRED, R>(kp, 0, b, s, vals, key);
#pragma unroll
      for (int j = 0; j < R; ++j) rid[j] = (u64)(b.row(j) + p.row_offset);
      table_insert_rows<IMPL, HFN, R>(p.sink_table, key, rid, alive, kp.d_flags);
      if (p.sink_table.d_bits != nullptr) {  // exact key bitmap for filter-only probes
        unsigned long long* bits = reinterpret_cast<unsigned long long*>(p.sink_table.d_bits);
        const u64 words = ((u64)p.sink_table.bits_span + 63ull) >> 6;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const u64 r = key[j] - (u64)p.sink_table.bits_lo;
          if (((alive >> j) & 1u) && r < (u64)p.sink_table.bits_span)
            for (int c = 0; c < p.sink_table.bits_copies; ++c)
              atomicOr(bits + c * words + (r >> 6), 1ull << (r & 63));
        }
      }
    }
  };

  // ---- LOOP ----
  const int64_t len = ce - cb;
  if constexpr (ACCESS == HAWK_COALESCED) {
    // Pass tiles of B*R rows: every referenced driver column of a tile is
    // staged into shared memory by one TMA bulk copy (cp.async.bulk), S tiles
    // in flight; thread t consumes tile rows t + jB.
    const int64_t pass_rows = (int64_t)B * R;
    const int64_t npasses = (len + pass_rows - 1) / pass_rows;
    // C stays a runtime value even in programs that never stage: folding it
    // to a constant 0 (HK_NO_STAGE) let the compiler reshape the pass loop
    // and TPC-H Q1 SF10's terminal went 0.61 -> 1.36 ms (profiles/ab_r02_stage_count.txt)
    const int S = kp.prefetch_passes, C = kp.nprefetch;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kp.smem_stage_off);
    int64_t* stages = reinterpret_cast<int64_t*>(smem + kp.smem_stage_off + 128);
    if (threadIdx.x == 0 && C > 0) {
      for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
      fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t ps) {
      const int st = (int)(ps % S);
      const int64_t b0 = cb + ps * pass_rows;
      const int64_t rows = min(pass_rows, ce - b0);
      const uint32_t bytes = (uint32_t)(((rows + 1) & ~1ll) * 8);
      mbar_arrive_expect_tx(&bars[st], bytes * (uint32_t)C);
      for (int c = 0; c < C; ++c)
        tma_load_1d(stages + ((size_t)st * C + c) * pass_rows,
                    reinterpret_cast<const int64_t*>(p.d_columns[kp.prefetch_col[c]]) + b0, bytes,
                    &bars[st]);
    };
    // unstaged tiles: one thread per column bulk-prefetches the tile
    // l2_distance passes ahead into L2 (no shared memory), so the coalesced
    // loads of a pass hit L2 instead of waiting on HBM
    const int L2C = C > 0 ? 0 : kp.l2_cols, D = kp.l2_distance;
    auto prefetch = [&](int64_t ps) {
      const int64_t b0 = cb + ps * pass_rows;
      const uint32_t bytes = (uint32_t)(((min(pass_rows, ce - b0) + 1) & ~1ll) * 8);
      for (int c = threadIdx.x; c < L2C; c += B)
        prefetch_l2_bulk(reinterpret_cast<const int64_t*>(p.d_columns[kp.prefetch_col[c]]) + b0, bytes);
    };
    if (threadIdx.x == 0 && C > 0)
      for (int64_t ps = 0; ps < min((int64_t)S, npasses); ++ps) issue(ps);
    if ((int)threadIdx.x < L2C)
      for (int64_t ps = 0; ps < min((int64_t)D, npasses); ++ps) prefetch(ps);
    for (int64_t ps = 0; ps < npasses; ++ps) {
      const int st = (int)(ps % S);
      if (C > 0) mbar_wait(&bars[st], (uint32_t)((ps / S) & 1));
      Batch<R, ACCESS> b;
      b.base = cb + ps * pass_rows;
      b.B = B;
      b.stage = C > 0 ? stages + (size_t)st * C * pass_rows : nullptr;
      if ((int)threadIdx.x < L2C && ps + D < npasses) prefetch(ps + D);
      if (b.base + pass_rows <= ce) {
        // full tile: a separate inlined copy with every row valid, so the
        // per-row validity predicates fold away
        b.valid = (1u << R) - 1u;
        process(b);
      } else {
        b.valid = 0;
#pragma unroll
        for (int j = 0; j < R; ++j) b.valid |= (uint32_t)(b.row(j) < ce) << j;
        process(b);
      }
      if (C > 0) {
        __syncthreads();  // every thread is done with stage st
        if (threadIdx.x == 0 && ps + S < npasses) {
          fence_proxy_async();
          issue(ps + S);
        }
      } else if (kp.pass_sync) {
        __syncthreads();  // keeps the CTA's warps on one tile (DRAM page locality)
      }
    }
  } else {
    // each thread scans its own contiguous sub-chunk with 128-bit loads
    const int64_t per = ((((len + B - 1) / B) + R - 1) / R) * R;
    const int64_t ts = cb + (int64_t)threadIdx.x * per;
    const int64_t te = min(ce, ts + per);
    for (int64_t k = 0; k < per; k += R) {
      Batch<R, ACCESS> b;
      b.base = ts + k;
      b.B = B;
      b.stage = nullptr;
      if (ts + k + R <= te) {
        b.valid = (1u << R) - 1u;
      } else {
        b.valid = 0;
#pragma unroll
        for (int j = 0; j < R; ++j) b.valid |= (uint32_t)(ts + k + j < te) << j;
      }
      process(b);
    }
  }

  if constexpr (kSplitRows) {  // rows still queued at the end of the chunk
    if (split_n > 0u)
      drain_rows<P, ROLE, PRED, IMPL, HFN, P::kDrain>(kp, s, split_q, 0u, split_n, cb, B, sink_static);
    __syncwarp(warp_mask());
  }

  // ---- sink epilogues ----
  if constexpr (ROLE == K_AGG_LOCAL || ROLE == K_AGG_GLOBAL) {
    const int lane = lane_id(), warp = threadIdx.x >> 5, nwarps = (B + 31) >> 5;
    const unsigned mask = warp_mask();
    const int wsize = warp_size_here();
    for (int a = 0; a < p.naggs; ++a) {
      const int fn = p.aggs[a].fn, ty = p.aggs[a].type;
      u64 v = s.acc(a);
      for (int o = 16; o > 0; o >>= 1) {
        u64 w = __shfl_down_sync(mask, v, o);
        if (lane + o < wsize) v = agg_combine(fn, ty, v, w);
      }
      if constexpr (ROLE == K_AGG_GLOBAL) {
        if (lane == 0) agg_merge(kp.d_final + a, fn, ty, v);  // direct global atomics
      } else {
        if (lane == 0) scratch[warp * HAWK_MAX_AGGS + a] = v;
      }
    }
    if constexpr (ROLE == K_AGG_LOCAL) {
      __syncthreads();
      __shared__ bool is_last;
      if (threadIdx.x == 0) {
        for (int a = 0; a < p.naggs; ++a) {
          u64 v = scratch[a];
          for (int w = 1; w < nwarps; ++w)
            v = agg_combine(p.aggs[a].fn, p.aggs[a].type, v, scratch[w * HAWK_MAX_AGGS + a]);
          kp.d_partials[(size_t)blockIdx.x * p.naggs + a] = v;
        }
        __threadfence();
        is_last = atomicAdd(kp.d_counter, 1u) == gridDim.x - 1;
      }
      __syncthreads();
      if (is_last) {
        __threadfence();
        // deterministic final reduction over per-CTA partials, fixed order
        for (int a = warp; a < p.naggs; a += nwarps) {
          const int fn = p.aggs[a].fn, ty = p.aggs[a].type;
          u64 v = agg_identity(fn, ty);
          for (unsigned i = lane; i < gridDim.x; i += wsize)
            v = agg_combine(fn, ty, v, ld_volatile(kp.d_partials + (size_t)i * p.naggs + a));
          for (int o = 16; o > 0; o >>= 1) {
            u64 w = __shfl_down_sync(mask, v, o);
            if (lane + o < wsize) v = agg_combine(fn, ty, v, w);
          }
          if (lane == 0) kp.d_final[a] = v;
        }
        if (threadIdx.x == 0) *kp.d_counter = 0u;
      }
    }
  } else if constexpr (ROLE == K_HAGG_LOCAL) {
    // HostMergeHashTables on the device: fold the CTA's smem partials into
    // the global table with atomics.
    __syncthreads();
    if (GP > 0) {
      // fold the thread-private accumulators of every ordinal group into its
      // slot: one warp per (group, aggregate) pair, fixed order
      const int n = min(*nord, GP);
      const int lane = lane_id(), warp = threadIdx.x >> 5, nwarps = (B + 31) >> 5;
      const unsigned mask = warp_mask();
      const int wsize = warp_size_here();
      for (int pa = warp; pa < n * A; pa += nwarps) {
        const int o = pa / A, a = pa % A;
        if (ord_slot[o] < 0) continue;  // ordinal lost a claim race: never used
        const int fn = p.aggs[a].fn == HAWK_COUNT ? HAWK_SUM : p.aggs[a].fn;
        const int ty = p.aggs[a].type;
        u64 v = agg_identity(fn, ty);
        for (int t = lane; t < B; t += 32) v = agg_combine(fn, ty, v, priv[(size_t)pa * B + t]);
        for (int off = 16; off > 0; off >>= 1) {
          u64 w = __shfl_down_sync(mask, v, off);
          if (lane + off < wsize) v = agg_combine(fn, ty, v, w);
        }
        if (lane == 0) {
          u64* acc = local_table + (size_t)ord_slot[o] * words + 1 + K + a;
          *acc = agg_combine(fn, ty, *acc, v);
        }
      }
      __syncthreads();
    }
    const hawk_table& gt = p.sink_table;
    const int slots = local_slots;
    for (int i = threadIdx.x; i < slots; i += B) {
      const u64* sl = local_table + (size_t)i * words;
      if (sl[0] == 0ull) continue;
      u64* g = agg_find_or_insert<IMPL, HFN, false>(kp, reinterpret_cast<u64*>(gt.d_slots),
                                                   gt.log2_capacity, gt.seed, sl + 1, 1,
                                                   kp.d_cursor);
      if (!g) {
        atomicOr(kp.d_flags, HAWK_FLAG_TABLE_FULL);
        continue;
      }
      for (int a = 0; a < p.naggs; ++a)
        agg_merge(g + 1 + K + a, p.aggs[a].fn, p.aggs[a].type, sl[1 + K + a]);
    }
  } else if constexpr (ROLE == K_COUNT) {
    u64 total;
    block_exclusive_scan(count, scratch, total);
    if (threadIdx.x == 0) kp.d_offsets[blockIdx.x] = (int64_t)total;
  }
}

template <int ROLE, int ACCESS, int PRED, int IMPL, int HFN, int U>
__global__ void __launch_bounds__(kMaxBlock, U == 1 ? 3 : (U == 2 ? 2 : 1))
    pipeline_kernel(const __grid_constant__ KParams kp) {
  pipeline_body<InterpProg, ROLE, ACCESS, PRED, IMPL, HFN, U>(kp);
}

}  // namespace hk
