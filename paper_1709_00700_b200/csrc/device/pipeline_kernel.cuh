// pipeline_kernel.cuh — the kernel template: LOOP driver (TMA-staged or
// per-thread sequential), the per-row op chain, and the eight sink roles.
#pragma once

#include "pipeline.cuh"

namespace hk {

// FILTER -> HASH_PROBE -> FILTER -> ARITHMETIC over one row batch.
template <int ACCESS, int PRED, int IMPL, int HFN, int R>
__device__ __forceinline__ void evaluate(const KParams& kp, const Batch<R>& b,
                                         const int64_t* stage, State<R>& s) {
  const hawk_pipeline& p = kp.p;
  s.alive = b.valid;
  // driver FILTER conjuncts (planner_reference.cpp:97-104)
  for (int i = 0; i < p.nfilter; ++i) {
    if (PRED == HAWK_BRANCHED && s.alive == 0u) return;
    const hawk_compare& c = p.filter[i];
    u64 x[R], y[R];
    fetch<ACCESS, PRED, R>(kp, c.lhs, c.type, b, s, stage, x);
    fetch<ACCESS, PRED, R>(kp, c.rhs, c.type, b, s, stage, y);
    s.alive &= compare_rows<R>(c.op, c.type, x, y);
  }
  // HASH_PROBE chain: branched opens a found-scope, predicated
  // folds the match bit into result_increment.
  for (int i = 0; i < p.nprobe; ++i) {
    if (PRED == HAWK_BRANCHED && s.alive == 0u) return;
    const hawk_probe& pr = p.probe[i];
    u64 k[R];
    fetch<ACCESS, PRED, R>(kp, pr.key, HAWK_I64, b, s, stage, k);
    const hawk_table& t = p.tables[pr.table];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const bool act = PRED == HAWK_PREDICATED ? ((b.valid >> j) & 1u) : ((s.alive >> j) & 1u);
      const int32_t r = act ? table_find<IMPL, HFN>(t, k[j]) : -1;
      if (r < 0) s.alive &= ~(1u << j);
      s.rid(i, j) = (u64)(r < 0 ? 0 : r);
    }
  }
  // post-probe FILTER conjuncts (operands may be build payloads)
  for (int i = 0; i < p.npost; ++i) {
    if (PRED == HAWK_BRANCHED && s.alive == 0u) return;
    const hawk_compare& c = p.post[i];
    u64 x[R], y[R];
    fetch<ACCESS, PRED, R>(kp, c.lhs, c.type, b, s, stage, x);
    fetch<ACCESS, PRED, R>(kp, c.rhs, c.type, b, s, stage, y);
    s.alive &= compare_rows<R>(c.op, c.type, x, y);
  }
  // ARITHMETIC into registers 0..narith-1
  for (int a = 0; a < p.narith; ++a) {
    if (PRED == HAWK_BRANCHED && s.alive == 0u) return;
    const hawk_arith& ar = p.arith[a];
    u64 x[R], y[R], z[R];
    fetch<ACCESS, PRED, R>(kp, ar.lhs, ar.type, b, s, stage, x);
    fetch<ACCESS, PRED, R>(kp, ar.rhs, ar.type, b, s, stage, y);
    arith_rows<R>(ar.op, ar.type, x, y, z);
#pragma unroll
    for (int j = 0; j < R; ++j) s.reg(a, j) = z[j];
  }
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

template <int ROLE, int ACCESS, int PRED, int IMPL, int HFN, int U>
__global__ void __launch_bounds__(1024)
    pipeline_kernel(const __grid_constant__ KParams kp) {
  constexpr int R = ACCESS == HAWK_COALESCED ? U : 2 * U;
  extern __shared__ __align__(128) unsigned char smem[];
  const hawk_pipeline& p = kp.p;
  const int B = blockDim.x;
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
  u64 count = 0;       // COUNT role
  u64 running = 0;     // SCATTER role: rows written by this CTA so far
  u64* local_table = reinterpret_cast<u64*>(smem + kp.smem_table_off);
  const int K = p.nkeys;
  const int words = 1 + p.nkeys + p.naggs;
  if constexpr (ROLE == K_HAGG_LOCAL) {
    const int slots = (1 << kp.local_log2) * (IMPL == HAWK_CUCKOO ? 2 : 1);
    for (int i = threadIdx.x; i < slots; i += B) local_table[(size_t)i * words] = 0ull;
    __syncthreads();
  }
  u64 scatter_base = 0;
  if constexpr (ROLE == K_PROJECT_SCATTER) scatter_base = (u64)kp.d_offsets[blockIdx.x];

  auto process = [&](const Batch<R>& b, const int64_t* stage) {
    evaluate<ACCESS, PRED, IMPL, HFN, R>(kp, b, stage, s);
    const uint32_t alive = s.alive;
    if constexpr (ROLE == K_AGG_LOCAL || ROLE == K_AGG_GLOBAL) {
      // AGGREGATE: predicated SUM/COUNT multiply by the
      // 0/1 result_increment, MIN/MAX select.
      if (PRED == HAWK_BRANCHED && alive == 0u) return;
      for (int a = 0; a < p.naggs; ++a) {
        const hawk_agg& g = p.aggs[a];
        u64& acc = s.acc(a);
        if (g.fn == HAWK_COUNT) {
          acc += (u64)__popc(alive);
          continue;
        }
        u64 v[R];
        fetch<ACCESS, PRED, R>(kp, g.input, g.type, b, s, stage, v);
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
      for (int i = 0; i < K; ++i) {
        u64 v[R];
        fetch<ACCESS, PRED, R>(kp, p.keys[i], HAWK_I64, b, s, stage, v);
#pragma unroll
        for (int j = 0; j < R; ++j) s.key(i, j) = v[j];
      }
      u64* slot[R];
      const hawk_table& gt = p.sink_table;
      const int kstride = R * B;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        slot[j] = nullptr;
        if (!((alive >> j) & 1u)) continue;
        const u64* kj = &s.key(0, j);
        if constexpr (ROLE == K_HAGG_LOCAL)
          slot[j] = agg_find_or_insert<IMPL, HFN, true>(kp, local_table, kp.local_log2, gt.seed,
                                                       kj, kstride, nullptr);
        if (slot[j] == nullptr)
          slot[j] = agg_find_or_insert<IMPL, HFN, false>(
              kp, reinterpret_cast<u64*>(gt.d_slots), gt.log2_capacity, gt.seed, kj, kstride,
              kp.d_cursor);
        if (slot[j] == nullptr) atomicOr(kp.d_flags, HAWK_FLAG_TABLE_FULL);
      }
      for (int a = 0; a < p.naggs; ++a) {
        const hawk_agg& g = p.aggs[a];
        u64 v[R];
        if (g.fn != HAWK_COUNT) fetch<ACCESS, PRED, R>(kp, g.input, g.type, b, s, stage, v);
#pragma unroll
        for (int j = 0; j < R; ++j)
          if (slot[j]) agg_update(slot[j] + 1 + K + a, g.fn, g.type, g.fn == HAWK_COUNT ? 1ull : v[j]);
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
          fetch<ACCESS, PRED, R>(kp, p.project[i], p.project[i].type, b, s, stage, v);
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
          fetch<ACCESS, PRED, R>(kp, p.project[i], p.project[i].type, b, s, stage, v);
          int64_t* out = kp.d_out + (size_t)i * kp.out_stride + pos;
          int k = 0;
#pragma unroll
          for (int j = 0; j < R; ++j)
            if ((alive >> j) & 1u) out[k++] = (int64_t)v[j];
        }
      }
      running += total;
    } else if constexpr (ROLE == K_PUT_SINGLE) {
      if (PRED == HAWK_BRANCHED && alive == 0u) return;
      u64 key[R];
      fetch<ACCESS, PRED, R>(kp, p.keys[0], HAWK_I64, b, s, stage, key);
#pragma unroll
      for (int j = 0; j < R; ++j)
        if ((alive >> j) & 1u)
          table_insert<IMPL, HFN>(p.sink_table, key[j], (u64)(b.row[j] + p.row_offset),
                                  kp.d_flags);
    }
  };

  // ---- LOOP ----
  if constexpr (ACCESS == HAWK_COALESCED) {
    // CTA-contiguous tiles; every referenced driver column of a tile is staged
    // into shared memory with one TMA bulk copy, nstages deep.
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    int64_t* stages = reinterpret_cast<int64_t*>(smem + kp.smem_stage_off);
    const int T = kp.tile_rows, S = kp.nstages, C = kp.nstaged;
    const int64_t ntiles = ce > cb ? (ce - cb + T - 1) / T : 0;
    if (threadIdx.x == 0) {
      for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
      fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t tile) {
      const int st = (int)(tile % S);
      const int64_t tb = cb + tile * T;
      const int64_t rows = min((int64_t)T, ce - tb);
      const uint32_t bytes = (uint32_t)(((rows + 1) & ~1ll) * 8);
      mbar_arrive_expect_tx(&bars[st], bytes * (uint32_t)C);
      for (int c = 0; c < C; ++c)
        tma_load_1d(stages + ((size_t)st * C + c) * T,
                    reinterpret_cast<const int64_t*>(p.d_columns[kp.staged_col[c]]) + tb, bytes,
                    &bars[st]);
    };
    if (threadIdx.x == 0 && C > 0)
      for (int64_t t = 0; t < min((int64_t)S, ntiles); ++t) issue(t);
    const int per_thread = (T + B - 1) / B;
    for (int64_t tile = 0; tile < ntiles; ++tile) {
      const int st = (int)(tile % S);
      if (C > 0) mbar_wait(&bars[st], (uint32_t)((tile / S) & 1));
      const int64_t* stage = stages + (size_t)st * C * T;
      const int64_t tb = cb + tile * T;
      const int rows = (int)min((int64_t)T, ce - tb);
      for (int k = 0; k < per_thread; k += U) {
        Batch<R> b;
        b.valid = 0;
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int r = threadIdx.x + (k + j) * B;
          const bool ok = (k + j) < per_thread && r < rows;
          b.valid |= (uint32_t)ok << j;
          b.sidx[j] = ok ? r : 0;
          b.row[j] = tb + (ok ? r : 0);
        }
        process(b, stage);
      }
      __syncthreads();
      if (threadIdx.x == 0 && C > 0 && tile + S < ntiles) {
        fence_proxy_async();
        issue(tile + S);
      }
    }
  } else {
    // each thread scans its own contiguous sub-chunk with 128-bit loads
    const int64_t len = ce - cb;
    const int64_t per = (((len + B - 1) / B) + 1) & ~1ll;
    const int64_t ts = cb + (int64_t)threadIdx.x * per;
    const int64_t te = min(ce, ts + per);
    for (int64_t k = 0; k < per; k += R) {
      Batch<R> b;
      b.valid = 0;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int64_t r = ts + k + j;
        b.valid |= (uint32_t)(r < te) << j;
        b.row[j] = r < te ? r : 0;
        b.sidx[j] = 0;
      }
      process(b, nullptr);
    }
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
    const hawk_table& gt = p.sink_table;
    const int slots = (1 << kp.local_log2) * (IMPL == HAWK_CUCKOO ? 2 : 1);
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

}  // namespace hk
