// kernels_misc.cuh — small kernels around the pipeline kernels: exclusive
// scans, standalone table build/probe, cuckoo
// duplicate check, aggregation-table extract/merge (HostMergeHashTables,
// SPEC.md:287), data generation (include/hawk_gen.h).
#pragma once

#include "hawk_gen.h"
#include "pipeline_kernel.cuh"

namespace hk {

// ---- exclusive prefix sum (3 phases: block scan, scan of block sums, add) -----

constexpr int kScanBlock = 512;
constexpr int kScanItems = 8;  // elements per thread per block pass

__global__ void __launch_bounds__(kScanBlock)
    scan_blocks_kernel(const int64_t* in, int64_t n, int64_t* out, int64_t* block_sums) {
  __shared__ u64 scratch[40];
  const int64_t base = (int64_t)blockIdx.x * kScanBlock * kScanItems;
  u64 v[kScanItems];
  u64 local = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t idx = base + (int64_t)threadIdx.x * kScanItems + i;
    v[i] = idx < n ? (u64)in[idx] : 0ull;
    local += v[i];
  }
  u64 total;
  u64 excl = block_exclusive_scan(local, scratch, total);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t idx = base + (int64_t)threadIdx.x * kScanItems + i;
    if (idx < n) out[idx] = (int64_t)excl;
    excl += v[i];
  }
  if (threadIdx.x == 0) block_sums[blockIdx.x] = (int64_t)total;
}

// single-CTA exclusive scan of up to any length (loops); writes the total.
__global__ void __launch_bounds__(1024)
    scan_single_kernel(int64_t* data, int64_t n, int64_t* total_out) {
  __shared__ u64 scratch[40];
  u64 carry = 0;
  for (int64_t base = 0; base < n; base += blockDim.x) {
    const int64_t idx = base + threadIdx.x;
    const u64 v = idx < n ? (u64)data[idx] : 0ull;
    u64 total;
    const u64 excl = block_exclusive_scan(v, scratch, total);
    if (idx < n) data[idx] = (int64_t)(carry + excl);
    carry += total;
  }
  if (threadIdx.x == 0 && total_out) *total_out = (int64_t)carry;
}

__global__ void scan_add_kernel(int64_t* out, int64_t n, const int64_t* block_offsets) {
  const int64_t base = (int64_t)blockIdx.x * kScanBlock * kScanItems;
  const int64_t add = block_offsets[blockIdx.x];
  for (int i = threadIdx.x; i < kScanBlock * kScanItems; i += blockDim.x) {
    const int64_t idx = base + i;
    if (idx < n) out[idx] += add;
  }
}

// ---- join tables ----------------------------------------------------------------

// min / max of an int64 column: grid-stride 128-bit loads, warp reduce,
// one pair of 64-bit atomics per warp. out = {min, max}, preset by the host.
__global__ void column_range_kernel(const int64_t* __restrict__ col, int64_t n, long long* out) {
  long long lo = 0x7fffffffffffffffll, hi = (long long)0x8000000000000000ull;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t pairs = n / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += stride) {
    u64 a, b;
    ldg128(reinterpret_cast<const u64*>(col) + 2 * i, a, b);
    lo = min(lo, (long long)min((int64_t)a, (int64_t)b));
    hi = max(hi, (long long)max((int64_t)a, (int64_t)b));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    lo = min(lo, (long long)col[n - 1]);
    hi = max(hi, (long long)col[n - 1]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_down_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_down_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, lo);
    atomicMax(out + 1, hi);
  }
}

// a deferred build's verdict: flags, inserted rows, dense-index fill count
// and whether there is an index (hawk_b200_deferred_collect)
__global__ void build_verdict_kernel(const u64* __restrict__ ctrl, int has_index, u64* __restrict__ out) {
  out[0] = ctrl[0] & 0xffffffffull;
  out[1] = ctrl[2];
  out[2] = ctrl[7];
  out[3] = (u64)has_index;
}

// ---- narrowed result read-back (hawk_b200_rows_pack*) ---------------------------

// per-column min / max of a row-major (n x w) block. Threads walk the flat
// word index with a stride that is a multiple of w, so each thread stays on
// one column; CTA partials meet in shared memory, one global atomic pair per
// column per CTA. out[2c] = min, out[2c + 1] = max, preset by the host.
__global__ void rows_range_kernel(const int64_t* __restrict__ rows, int64_t n, int w, long long* out) {
  extern __shared__ long long sh[];  // 2w
  for (int c = threadIdx.x; c < w; c += blockDim.x) {
    sh[2 * c] = 0x7fffffffffffffffll;
    sh[2 * c + 1] = (long long)0x8000000000000000ull;
  }
  __syncthreads();
  const int64_t threads = (int64_t)gridDim.x * blockDim.x / w * w;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < threads) {
    const int c = (int)(t % w);
    long long lo = 0x7fffffffffffffffll, hi = (long long)0x8000000000000000ull;
    for (int64_t i = t; i < n * w; i += threads) {
      const long long v = (long long)__ldg(rows + i);
      lo = min(lo, v);
      hi = max(hi, v);
    }
    atomicMin(&sh[2 * c], lo);
    atomicMax(&sh[2 * c + 1], hi);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < w; c += blockDim.x) {
    atomicMin(out + 2 * c, sh[2 * c]);
    atomicMax(out + 2 * c + 1, sh[2 * c + 1]);
  }
}

struct PackParams {
  int32_t width;
  int32_t bytes[HAWK_MAX_WIDTH];
  int64_t base[HAWK_MAX_WIDTH];
  int64_t offset[HAWK_MAX_WIDTH];
};

// one thread per row: reads the row's words, writes each column's narrowed
// value (coalesced across the warp per column)
__global__ void rows_pack_kernel(const int64_t* __restrict__ rows, int64_t n, const __grid_constant__ PackParams pp,
                                 unsigned char* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    const int64_t* row = rows + r * pp.width;
    for (int c = 0; c < pp.width; ++c) {
      const int b = pp.bytes[c];
      if (b == 0) continue;
      const u64 v = (u64)__ldg(row + c) - (u64)pp.base[c];
      unsigned char* d = out + pp.offset[c];
      if (b == 1) d[r] = (unsigned char)v;
      else if (b == 2) reinterpret_cast<uint16_t*>(d)[r] = (uint16_t)v;
      else if (b == 4) reinterpret_cast<uint32_t*>(d)[r] = (uint32_t)v;
      else reinterpret_cast<u64*>(d)[r] = v;
    }
  }
}

// L2 flush by reading a buffer twice the L2 size: evicts the working set
// while leaving only clean lines behind (a memset flush leaves dirty lines
// whose write-back would land in the next timed kernel).
__global__ void flush_read_kernel(const u64* __restrict__ p, int64_t pairs, u64* sink) {
  u64 acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += stride) {
    u64 a, b;
    ldg128(p + 2 * i, a, b);
    acc ^= a ^ b;
  }
  if (acc == 0x9e3779b97f4a7c15ull) *sink = acc;  // never true for a zeroed buffer; keeps the loads
}

__global__ void fill_kernel(u64* p, u64 value, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = value;
}

template <int IMPL, int HFN>
__global__ void table_insert_kernel(hawk_table t, const int64_t* keys, const int64_t* payloads,
                                    int64_t n, int* flags) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    table_insert<IMPL, HFN>(t, (u64)keys[i], payloads ? (u64)payloads[i] : (u64)i, flags);
}

template <int IMPL, int HFN>
__global__ void table_probe_kernel(hawk_table t, const int64_t* keys, int64_t n, int64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = table_find<IMPL, HFN>(t, (u64)keys[i]);
}

// A cuckoo key can only live at T1[h1(k)] or T2[h2(k)]; a duplicate build
// key therefore shows up as the same key in both candidate slots.
template <int HFN>
__global__ void cuckoo_duplicate_kernel(hawk_table t, int* flags) {
  const u64* s = reinterpret_cast<const u64*>(t.d_slots);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < t.capacity;
       i += (int64_t)gridDim.x * blockDim.x) {
    const u64 k = s[2 * i];
    if (k == kEmpty) continue;
    const u64 j = hash_slot<HFN>(k, t.seed[1], t.log2_capacity);
    if (s[2 * ((u64)t.capacity + j)] == k) atomicOr(flags, HAWK_FLAG_DUPLICATE);
  }
}

// Filled entries (!= -1) of a dense join index; fewer than the rows the
// build inserted means a duplicate build key.
__global__ void index_fill_count_kernel(const int32_t* __restrict__ idx, int64_t span, u64* out) {
  u64 n = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t quads = span / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < quads; i += stride) {
    const int4 v = __ldg(reinterpret_cast<const int4*>(idx) + i);
    n += (v.x != -1) + (v.y != -1) + (v.z != -1) + (v.w != -1);
  }
  if (blockIdx.x == 0 && threadIdx.x < span - quads * 4) n += idx[quads * 4 + threadIdx.x] != -1;
  n = __reduce_add_sync(0xffffffffu, (unsigned)n);
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(out, n);
}

// ---- aggregation tables -------------------------------------------------------------

// Compacts occupied slots into rows of (keys..., accs...).
__global__ void agg_extract_kernel(const u64* slots, int64_t nslots, int K, int A, int64_t* out,
                                   u64* cursor) {
  const int words = 1 + K + A;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nslots;
       i += (int64_t)gridDim.x * blockDim.x) {
    const u64* sl = slots + i * words;
    if ((sl[0] & 1ull) == 0ull) continue;  // EMPTY (0) / never BUSY after the kernel
    const u64 pos = atomicAdd(cursor, 1ull);
    for (int w = 0; w < K + A; ++w) out[pos * (K + A) + w] = (int64_t)sl[1 + w];
  }
}

// Merges partial group rows (keys..., accs...) into a table (multi-GPU merge).
template <int IMPL, int HFN>
__global__ void agg_merge_rows_kernel(const __grid_constant__ KParams kp, const int64_t* rows,
                                      int64_t n) {
  const hawk_pipeline& p = kp.p;
  const int K = p.nkeys, A = p.naggs;
  const hawk_table& gt = p.sink_table;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const u64* r = reinterpret_cast<const u64*>(rows + i * (K + A));
    u64* g = agg_find_or_insert<IMPL, HFN, false>(kp, reinterpret_cast<u64*>(gt.d_slots),
                                                 gt.log2_capacity, gt.seed, r, 1, kp.d_cursor);
    if (!g) {
      atomicOr(kp.d_flags, HAWK_FLAG_TABLE_FULL);
      continue;
    }
    for (int a = 0; a < A; ++a) agg_merge(g + 1 + K + a, p.aggs[a].fn, p.aggs[a].type, r[K + a]);
  }
}

// Combines n partial AGGREGATE rows (naggs accumulators each) into one row:
// the multi-GPU merge of non-grouped aggregates (COUNT partials add).
__global__ void agg_rows_combine_kernel(const __grid_constant__ KParams kp, const u64* rows,
                                        int64_t n, u64* out) {
  const hawk_pipeline& p = kp.p;
  for (int a = threadIdx.x; a < p.naggs; a += blockDim.x) {
    const int fn = p.aggs[a].fn == HAWK_COUNT ? HAWK_SUM : p.aggs[a].fn;
    u64 v = agg_identity(fn, p.aggs[a].type);
    for (int64_t i = 0; i < n; ++i) v = agg_combine(fn, p.aggs[a].type, v, rows[i * p.naggs + a]);
    out[a] = v;
  }
}

// ---- synthetic data ---------------------------------------------------------------

__global__ void gen_column_kernel(int table, int col, double sf, uint64_t seed, int64_t row_begin,
                                  int64_t n, int64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = hg_value(table, col, row_begin + i, sf, seed);
}

}  // namespace hk
