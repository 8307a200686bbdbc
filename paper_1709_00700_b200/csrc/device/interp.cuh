// interp.cuh — the vectorised pipeline-program interpreter shared by every
// kernel role.
//
// A lowered pipeline (hawk_pipeline, op order LOOP -> FILTER* -> HASH_PROBE*
// -> FILTER* -> ARITHMETIC* -> sink, as emitted by
// /root/reference/proj/src/planner_pipelines.cpp:319-397) is executed one op
// at a time over a batch of R = 4*U rows per thread: every op dispatches once
// (warp-uniform, parameters from the constant bank) and then runs a fully
// unrolled loop over its R rows, so the dispatch cost is amortised R-fold.
// Per-row values that live across ops (ARITHMETIC registers, probe row ids,
// group keys, AGGREGATE accumulators) are kept in shared memory, one word
// per thread per slot (bank-conflict free), which keeps register pressure
// independent of the program shape.
//
// The variant modes are template parameters (one instantiation per point):
//   ACCESS  COALESCED  — a warp reads 512 contiguous bytes per column load as
//                        128-bit vectors (thread t owns rows 2t, 2t+1 of each
//                        2B-row group, paper Listing 3 coalesced loop)
//           SEQUENTIAL — each thread scans its own contiguous sub-chunk
//                        (paper "sequential" partitioning)
//           both read 128-bit vectors (two int64 rows per load)
//   PRED    BRANCHED (scopes, early exit) / PREDICATED (branch-free
//           result_increment)
//   IMPL, HFN  hash table / hash function of every hash op of the pipeline
//   U       unroll factor: rows per op pass = 4*U
#pragma once

#include "common.cuh"

namespace hk {

// kernel roles: (sink, strategy) pairs
enum : int {
  K_AGG_LOCAL = 0,       // AGGREGATE, local: per-CTA partials + last-CTA reduce
  K_AGG_GLOBAL = 1,      // AGGREGATE, global: warp-reduced direct global atomics
  K_HAGG_LOCAL = 2,      // HASH_AGGREGATE, local: smem table per CTA + merge
  K_HAGG_GLOBAL = 3,     // HASH_AGGREGATE, global: one HBM table, direct atomics
  K_PROJECT_SINGLE = 4,  // PROJECT, single pass: warp-aggregated output cursor
  K_COUNT = 5,           // multi-pass pass 1: per-CTA match counts
  K_PROJECT_SCATTER = 6, // multi-pass pass 3: block scan + scatter
  K_PUT_SINGLE = 7,      // HASH_PUT inline
  K_NUM_ROLES = 8
};

constexpr int kMaxBlock = 256;   // threads per CTA (work groups > 256 span CTAs)
constexpr int kOpndRowId = 7;    // internal operand kind: the driver row id
constexpr int kRange = 6;        // internal compare op: lo <= x <= hi (int64)

// A FILTER conjunct after host-side compilation: int64 comparisons against
// literals become closed ranges, and conjuncts on the same operand merge
// (Q6: five conjuncts -> three ranges).
struct KFilter {
  hawk_operand lhs, rhs;
  int32_t op;    // HAWK_LT..HAWK_NE or kRange
  int32_t type;  // comparison domain
  int64_t lo, hi;
};

struct KParams {
  hawk_pipeline p;
  KFilter pre[HAWK_MAX_FILTERS];
  KFilter post[HAWK_MAX_FILTERS];
  int32_t npre, npost;
  int32_t nprefetch;                  // driver columns staged per pass (COALESCED)
  int8_t prefetch_col[HAWK_MAX_COLUMNS];   // staged index -> column slot
  int8_t stage_of[HAWK_MAX_COLUMNS];       // column slot -> staged index
  int32_t prefetch_passes;            // COALESCED: pipeline depth in pass tiles (>= 1)
  int32_t l2_cols;                    // COALESCED, unstaged: columns bulk-prefetched into L2
  int32_t l2_distance;                //   ... this many pass tiles ahead
  int32_t pass_sync;                  // COALESCED, unstaged: CTA barrier after every pass
  int32_t smem_stage_off;             // COALESCED: [mbarriers][stages x columns x B*R rows]
  int32_t local_log2;                 // HAGG_LOCAL: log2 smem table slots
  int64_t chunk_rows;                 // rows per CTA chunk (multiple of 64)
  u64* d_partials;                    // AGG_LOCAL: gridDim x naggs
  u64* d_final;                       // AGG: naggs
  unsigned* d_counter;                // AGG_LOCAL: last-CTA ticket
  int* d_flags;                       // HAWK_FLAG_*
  int64_t* d_out;                     // PROJECT: nproject columns
  int64_t out_stride;
  u64* d_cursor;                      // PROJECT_SINGLE cursor / HAGG group counter
  int64_t* d_offsets;                 // COUNT: per-CTA counts; SCATTER: exclusive offsets
  int64_t group_limit;                // HAGG: TABLE_FULL above this many groups
  int32_t smem_table_off;             // dynamic smem: [table][scratch][state][ord][priv]
  int32_t smem_scratch_off;
  int32_t priv_groups;                // HAGG_LOCAL: groups with thread-private accumulators
  int32_t smem_ord_off;               // HAGG_LOCAL: slot -> ordinal, ordinal -> slot, count
  int32_t smem_priv_off;              // HAGG_LOCAL: priv[(ord * naggs + a) * B + t]
  int32_t smem_dense_off;             // HAGG_LOCAL, compiled: dense key index -> ordinal (0: off)
  int32_t split;                      // compiled, branched: compact live rows after the first probe
  int32_t min_ctas;                   // compiled: __launch_bounds__ min CTAs per SM (0 = by unroll)
  int32_t smem_queue_off;             //   ... per-warp queues of (row, probe-0 row id)
  int32_t split_drain;                //   ... queued rows per lane per drain
  int32_t split_bits;                 //   ... key bitmaps for semi-join probes: 1 first, 2 all
  int32_t checked;                    // compiled: device bounds checks (HK_CHECKED)
  int32_t index_atomic;               // compiled single-pass builds: dense-index inserts by
                                      //   atomic exchange, duplicates flagged in place (HK_INDEX_ATOMIC)
  int32_t smem_state_off;
  int32_t state_words;                // state words per thread
  int32_t rid_base, key_base, acc_base;
};

// Device-side bounds checks of the compiled programs' indexed accesses
// (option "checked", -DHK_CHECKED): a failure raises HAWK_FLAG_CHECK and the
// access is skipped. compute-sanitizer is unavailable on this pool; this is
// the instrumented build that stands in for its memcheck.
#ifdef HK_CHECKED
#define HK_CHECK(kp, cond) \
  do {                     \
    if (!(cond)) atomicOr((kp).d_flags, HAWK_FLAG_CHECK); \
  } while (0)
#define HK_CHECKED_OK(kp, cond) ((cond) ? true : (atomicOr((kp).d_flags, HAWK_FLAG_CHECK), false))
#else
#define HK_CHECK(kp, cond) ((void)0)
#define HK_CHECKED_OK(kp, cond) true
#endif

// R rows of one op pass.
// COALESCED: the pass tile [base, base + B*R): thread t owns tile rows
//   2t + 2pB and 2t + 2pB + 1 for p < R/2, read with 128-bit loads from HBM
//   (or from the tile staged in shared memory by TMA bulk copies).
// SEQUENTIAL: thread t owns rows base + j of its own sub-chunk, read from
//   HBM with 128-bit loads (rows come in aligned pairs).
// kGather: R explicit rows (the compacted rows of a warp after the first
// probe; compiled programs only).
constexpr int kGather = 7;
template <int R, int ACCESS>
struct Batch {
  static constexpr int kR = R, kAccess = ACCESS;
  int64_t base;
  int B;
  uint32_t valid;          // rows inside the CTA chunk
  const int64_t* stage;    // COALESCED: this pass's staged tile
  int64_t rows_[ACCESS == kGather ? R : 1];
  // COALESCED: row pair p = j/2 of thread t is tile rows 2t + 2pB, +1, so
  // every column load of a warp reads 512 contiguous bytes as 128-bit vectors
  __device__ __forceinline__ int sidx(int j) const {
    return 2 * (int)threadIdx.x + (j >> 1) * 2 * B + (j & 1);
  }
  __device__ __forceinline__ int64_t row(int j) const {
    if constexpr (ACCESS == kGather) return rows_[j];
    if (ACCESS == HAWK_COALESCED) return base + sidx(j);
    return base + j;
  }
};

// Per-thread interpreter state in shared memory: word w of thread t at
// ts[w * B + t].
template <int R>
struct State {
  u64* ts;
  int B, tid;
  int rid_base, key_base, acc_base;
  uint32_t alive;
  __device__ __forceinline__ u64& w(int word) const { return ts[(size_t)word * B + tid]; }
  __device__ __forceinline__ u64& reg(int a, int j) const { return w(a * R + j); }
  __device__ __forceinline__ u64& rid(int i, int j) const { return w(rid_base + i * R + j); }
  __device__ __forceinline__ u64& key(int i, int j) const { return w(key_base + i * R + j); }
  __device__ __forceinline__ u64& acc(int a) const { return w(acc_base + a); }
};

// ---- operand fetch: one dispatch, R rows -------------------------------------------

template <int R, int ACCESS>
__device__ __forceinline__ void load_column(const KParams& kp, int slot, const Batch<R, ACCESS>& b,
                                            u64 (&v)[R]) {
  const int64_t* __restrict__ c = reinterpret_cast<const int64_t*>(kp.p.d_columns[slot]);
#ifdef HK_CHECKED
#pragma unroll
  for (int j = 0; j < R; ++j)  // rows inside the driver's padded extent
    HK_CHECK(kp, !((b.valid >> j) & 1u) || (b.row(j) >= 0 && b.row(j) < kp.p.nrows + 64));
#endif
  if constexpr (ACCESS == kGather) {  // compacted rows: gathers
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = ((b.valid >> j) & 1u) ? ldg64_stream(c + b.row(j)) : 0ull;
  } else if constexpr (ACCESS == HAWK_COALESCED) {
#ifdef HK_NO_STAGE  // compiled programs that never stage: no shared-memory tile path
    if (false) {
#else
    if (b.stage) {  // staged tile in shared memory (128-bit LDS per row pair)
#endif
      const int64_t* t = b.stage + (size_t)kp.stage_of[slot] * b.B * R;
#pragma unroll
      for (int j = 0; j < R; j += 2) {
        const longlong2 w = *reinterpret_cast<const longlong2*>(t + b.sidx(j));
        v[j] = (u64)w.x;
        v[j + 1] = (u64)w.y;
      }
    } else if (b.valid == (1u << R) - 1u) {  // full tile: warp-coalesced 128-bit loads
#pragma unroll
      for (int j = 0; j < R; j += 2) ldg128_stream(c + b.row(j), v[j], v[j + 1]);
    } else {
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = ((b.valid >> j) & 1u) ? ldg64_stream(c + b.row(j)) : 0ull;
    }
  } else if (b.valid == (1u << R) - 1u) {
#pragma unroll
    for (int j = 0; j < R; j += 2) ldg128(c + b.row(j), v[j], v[j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = ((b.valid >> j) & 1u) ? ldg64(c + b.row(j)) : 0ull;
  }
}

template <int PRED, int R, int ACCESS>
__device__ __forceinline__ void fetch(const KParams& kp, const hawk_operand& o, int want,
                                      const Batch<R, ACCESS>& b, const State<R>& s,
                                      u64 (&v)[R]) {
  switch (o.kind) {
    case HAWK_OPND_COLUMN:
      load_column<R, ACCESS>(kp, o.index, b, v);
      break;
    case HAWK_OPND_PAYLOAD: {
      const int64_t* c = reinterpret_cast<const int64_t*>(kp.p.d_columns[o.index]);
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const bool act = PRED == HAWK_PREDICATED ? ((b.valid >> j) & 1u) : ((s.alive >> j) & 1u);
        v[j] = act ? ldg64(c + s.rid(o.probe, j)) : 0ull;
      }
      break;
    }
    case HAWK_OPND_REG:
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = s.reg(o.index, j);
      break;
    case kOpndRowId:
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = (u64)(b.row(j) + kp.p.row_offset);
      break;
    default:  // INT / FLOAT literal
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = (u64)o.bits;
      break;
  }
  // int -> double promotion (planner_reference.cpp:114-128; sql_parser.cpp:527-528)
  if (want == HAWK_F64 && o.type == HAWK_I64) {
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = as_bits((double)(i64)v[j]);
  }
}

// ---- comparisons (planner_reference.cpp:76-95) -------------------------------------

template <int R>
__device__ __forceinline__ uint32_t compare_rows(const KFilter& f, const u64 (&a)[R],
                                                 const u64 (&b)[R]) {
  uint32_t m = 0;
  if (f.op == kRange) {
    const u64 lo = (u64)f.lo, span = (u64)f.hi - (u64)f.lo;
#pragma unroll
    for (int j = 0; j < R; ++j) m |= (uint32_t)(a[j] - lo <= span) << j;
    return m;
  }
  if (f.type == HAWK_I64) {
#define HK_CMP(EXPR)                                  \
  _Pragma("unroll") for (int j = 0; j < R; ++j) {     \
    const i64 x = (i64)a[j], y = (i64)b[j];           \
    m |= (uint32_t)(EXPR) << j;                       \
  }
    switch (f.op) {
      case HAWK_LT: HK_CMP(x < y) break;
      case HAWK_LE: HK_CMP(x <= y) break;
      case HAWK_EQ: HK_CMP(x == y) break;
      case HAWK_GE: HK_CMP(x >= y) break;
      case HAWK_GT: HK_CMP(x > y) break;
      default: HK_CMP(x != y) break;
    }
#undef HK_CMP
  } else {
#define HK_CMP(EXPR)                                  \
  _Pragma("unroll") for (int j = 0; j < R; ++j) {     \
    const double x = as_f64(a[j]), y = as_f64(b[j]);  \
    m |= (uint32_t)(EXPR) << j;                       \
  }
    switch (f.op) {
      case HAWK_LT: HK_CMP(x < y) break;
      case HAWK_LE: HK_CMP(x <= y) break;
      case HAWK_EQ: HK_CMP(x == y) break;
      case HAWK_GE: HK_CMP(x >= y) break;
      case HAWK_GT: HK_CMP(x > y) break;
      default: HK_CMP(x != y) break;
    }
#undef HK_CMP
  }
  return m;
}

// ---- arithmetic (planner_reference.cpp:106-141): int64 wraps, x/0 = 0 -----------------

template <int R>
__device__ __forceinline__ void arith_rows(int op, int type, const u64 (&a)[R], const u64 (&b)[R],
                                           u64 (&out)[R]) {
  if (type == HAWK_I64) {
    switch (op) {
      case HAWK_ADD:
#pragma unroll
        for (int j = 0; j < R; ++j) out[j] = a[j] + b[j];
        break;
      case HAWK_SUB:
#pragma unroll
        for (int j = 0; j < R; ++j) out[j] = a[j] - b[j];
        break;
      case HAWK_MUL:
#pragma unroll
        for (int j = 0; j < R; ++j) out[j] = a[j] * b[j];
        break;
      default:
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const i64 x = (i64)a[j], y = (i64)b[j];
          out[j] = y == 0 ? 0ull : (y == -1 ? (u64)0 - (u64)x : (u64)(x / y));
        }
        break;
    }
  } else {
    switch (op) {
      case HAWK_ADD:
#pragma unroll
        for (int j = 0; j < R; ++j) out[j] = as_bits(__dadd_rn(as_f64(a[j]), as_f64(b[j])));
        break;
      case HAWK_SUB:
#pragma unroll
        for (int j = 0; j < R; ++j) out[j] = as_bits(__dsub_rn(as_f64(a[j]), as_f64(b[j])));
        break;
      case HAWK_MUL:
#pragma unroll
        for (int j = 0; j < R; ++j) out[j] = as_bits(__dmul_rn(as_f64(a[j]), as_f64(b[j])));
        break;
      default:
#pragma unroll
        for (int j = 0; j < R; ++j) out[j] = as_bits(__ddiv_rn(as_f64(a[j]), as_f64(b[j])));
        break;
    }
  }
}

}  // namespace hk
