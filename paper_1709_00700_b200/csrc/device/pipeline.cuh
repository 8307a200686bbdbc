// pipeline.cuh — the templated pipeline-program kernel family.
//
// One kernel template executes a lowered pipeline program (hawk_pipeline):
//   LOOP -> FILTER* -> HASH_PROBE* -> FILTER* -> ARITHMETIC* -> sink
// which is the op order the reference lowering emits
// (/root/reference/proj/src/planner_pipelines.cpp:319-397). The variant modes
// are template parameters, one instantiation per variant point:
//   ACCESS  MemoryAccess     COALESCED: CTA-contiguous tiles staged into shared
//                            memory by TMA bulk copies (cp.async.bulk), threads
//                            read rows t, t+B, ... (paper Listing 3 coalesced);
//                            SEQUENTIAL: each thread scans its own contiguous
//                            chunk with 128-bit loads (paper "sequential").
//   PRED    PredicationMode  BRANCHED: per-row scopes / early exit;
//                            PREDICATED: branch-free result_increment
//                            (PAPER.md:1077-1111).
//   IMPL    HashTableImpl    linear probing / cuckoo
//   HFN     HashFunctionKind murmur / multiply-shift
//   U       unroll factor    rows evaluated per interpreter pass
// and (SINK, MODE) pick the pipeline's last op and the execution strategy.
// The per-query structure (predicates, probes, expressions, aggregates) is
// read from the kernel parameter block with warp-uniform control flow.
#pragma once

#include "common.cuh"

namespace hk {

// (SINK, MODE) kernel roles
enum : int {
  K_AGG_LOCAL = 0,      // AGGREGATE, local: per-CTA partials + last-CTA reduce
  K_AGG_GLOBAL = 1,     // AGGREGATE, global: warp-reduced direct global atomics
  K_HAGG_LOCAL = 2,     // HASH_AGGREGATE, local: smem table per CTA + merge
  K_HAGG_GLOBAL = 3,    // HASH_AGGREGATE, global: one HBM table, direct atomics
  K_PROJECT_SINGLE = 4, // PROJECT, single pass: warp-aggregated output cursor
  K_COUNT = 5,          // multi-pass pass 1: per-CTA match counts
  K_PROJECT_SCATTER = 6,// multi-pass pass 3: block scan + scatter
  K_PUT_SINGLE = 7,     // HASH_PUT inline
  K_NUM_ROLES = 8
};

// operand kind used only internally: the driver row id (multi-pass HASH_PUT
// compacts row ids through the PROJECT scatter)
constexpr int kOpndRowId = 7;

struct KParams {
  hawk_pipeline p;
  int8_t stage_of[HAWK_MAX_COLUMNS];    // column slot -> staged slot (-1: not staged)
  int8_t staged_col[HAWK_MAX_COLUMNS];  // staged slot -> column slot
  int32_t nstaged;
  int32_t tile_rows;   // rows per TMA tile (multiple of 16)
  int32_t nstages;     // TMA pipeline depth
  int32_t local_log2;  // HAGG_LOCAL: log2 smem table slots
  int64_t chunk_rows;  // rows per CTA chunk (multiple of 16)
  u64* d_partials;     // AGG_LOCAL: gridDim x naggs
  u64* d_final;        // AGG: naggs
  unsigned* d_counter; // AGG_LOCAL: last-CTA ticket
  int* d_flags;        // HAWK_FLAG_*
  int64_t* d_out;      // PROJECT: nproject columns
  int64_t out_stride;
  u64* d_cursor;       // PROJECT_SINGLE cursor / HAGG group counter
  int64_t* d_offsets;  // COUNT: per-CTA counts; SCATTER: per-CTA exclusive offsets
  int64_t group_limit; // HAGG: flag TABLE_FULL above this many groups
  int32_t smem_stage_off;   // dynamic smem layout: [mbarriers][stages][table][scratch]
  int32_t smem_table_off;
  int32_t smem_scratch_off;
  int32_t smem_state_off;   // per-thread interpreter state (see State)
  int32_t state_words;      // words per thread
  int32_t rid_base, key_base, acc_base;
};

template <int R>
struct Batch {
  int64_t row[R];  // shard-local row index
  int32_t sidx[R]; // row within the staged tile
  uint32_t valid;  // rows inside the CTA chunk
};

// Per-thread interpreter state lives in shared memory, word w of thread t at
// ts[w * B + t] (bank-conflict free): ARITHMETIC registers, probe row ids,
// group keys and AGGREGATE accumulators. Keeping it out of registers lets
// one kernel body serve every program shape at full occupancy.
template <int R>
struct State {
  u64* ts;        // this CTA's state area
  int B, tid;
  int rid_base;   // word of rid(0, 0)
  int key_base;   // word of key(0, 0)
  int acc_base;   // word of acc(0)
  uint32_t alive;
  __device__ __forceinline__ u64& w(int word) const { return ts[(size_t)word * B + tid]; }
  __device__ __forceinline__ u64& reg(int a, int j) const { return w(a * R + j); }
  __device__ __forceinline__ u64& rid(int i, int j) const { return w(rid_base + i * R + j); }
  __device__ __forceinline__ u64& key(int i, int j) const { return w(key_base + i * R + j); }
  __device__ __forceinline__ u64& acc(int a) const { return w(acc_base + a); }
};

// ---- operand fetch ------------------------------------------------------------

template <int ACCESS, int PRED, int R>
__device__ __forceinline__ void fetch(const KParams& kp, const hawk_operand& o, int want,
                                      const Batch<R>& b, const State<R>& s, const int64_t* stage,
                                      u64 (&v)[R]) {
  switch (o.kind) {
    case HAWK_OPND_COLUMN: {
      if (ACCESS == HAWK_COALESCED) {
        const int64_t* c = stage + (size_t)kp.stage_of[o.index] * kp.tile_rows;
#pragma unroll
        for (int j = 0; j < R; ++j) v[j] = (u64)c[b.sidx[j]];
      } else {
        const int64_t* c = reinterpret_cast<const int64_t*>(kp.p.d_columns[o.index]);
        if (b.valid == (1u << R) - 1u) {
#pragma unroll
          for (int j = 0; j < R; j += 2) ldg128(c + b.row[j], v[j], v[j + 1]);
        } else {
#pragma unroll
          for (int j = 0; j < R; ++j) v[j] = ((b.valid >> j) & 1u) ? ldg64(c + b.row[j]) : 0ull;
        }
      }
      break;
    }
    case HAWK_OPND_PAYLOAD: {
      const int64_t* c = reinterpret_cast<const int64_t*>(kp.p.d_columns[o.index]);
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const bool act = PRED == HAWK_PREDICATED ? ((b.valid >> j) & 1u) : ((s.alive >> j) & 1u);
        v[j] = act ? ldg64(c + s.rid(o.probe, j)) : 0ull;
      }
      break;
    }
    case HAWK_OPND_REG: {
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = s.reg(o.index, j);
      break;
    }
    case kOpndRowId: {
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = (u64)(b.row[j] + kp.p.row_offset);
      break;
    }
    default: {  // INT / FLOAT literal
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = (u64)o.bits;
      break;
    }
  }
  // int -> double promotion (planner_reference.cpp:114-128; sql_parser.cpp:527-528)
  if (want == HAWK_F64 && o.type == HAWK_I64) {
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = as_bits((double)(i64)v[j]);
  }
}

// ---- comparisons (planner_reference.cpp:76-95) -------------------------------

template <int R>
__device__ __forceinline__ uint32_t compare_rows(int op, int type, const u64 (&a)[R],
                                                 const u64 (&b)[R]) {
  uint32_t m = 0;
  if (type == HAWK_I64) {
#define HK_CMP(EXPR)                                                      \
  _Pragma("unroll") for (int j = 0; j < R; ++j) {                         \
    const i64 x = (i64)a[j], y = (i64)b[j];                               \
    m |= (uint32_t)(EXPR) << j;                                           \
  }
    switch (op) {
      case HAWK_LT: HK_CMP(x < y) break;
      case HAWK_LE: HK_CMP(x <= y) break;
      case HAWK_EQ: HK_CMP(x == y) break;
      case HAWK_GE: HK_CMP(x >= y) break;
      case HAWK_GT: HK_CMP(x > y) break;
      default: HK_CMP(x != y) break;
    }
#undef HK_CMP
  } else {
#define HK_CMP(EXPR)                                                      \
  _Pragma("unroll") for (int j = 0; j < R; ++j) {                         \
    const double x = as_f64(a[j]), y = as_f64(b[j]);                      \
    m |= (uint32_t)(EXPR) << j;                                           \
  }
    switch (op) {
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

// ---- arithmetic (planner_reference.cpp:106-141): int64 wraps, x/0 = 0 ---------

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

// ---- join tables: HASH_PROBE --------------------------

template <int IMPL, int HFN>
__device__ __forceinline__ int32_t table_find(const hawk_table& t, u64 key) {
  if (key == kEmpty) return -1;
  const u64* s = reinterpret_cast<const u64*>(t.d_slots);
  if (IMPL == HAWK_LINEAR_PROBING) {
    const u64 mask = (u64)t.capacity - 1ull;
    u64 i = hash_slot<HFN>(key, t.seed[0], t.log2_capacity);
    for (;;) {
      u64 k, v;
      ldg128(s + 2 * i, k, v);
      if (k == key) return (int32_t)v;
      if (k == kEmpty) return -1;
      i = (i + 1) & mask;
    }
  } else {
    u64 k, v;
    u64 i = hash_slot<HFN>(key, t.seed[0], t.log2_capacity);
    ldg128(s + 2 * i, k, v);
    if (k == key) return (int32_t)v;
    i = hash_slot<HFN>(key, t.seed[1], t.log2_capacity);
    ldg128(s + 2 * ((u64)t.capacity + i), k, v);
    if (k == key) return (int32_t)v;
    return -1;
  }
}

// HASH_PUT: LP = CAS-claim the key slot then store the
// payload; cuckoo = 128-bit exchange with an eviction chain of <= 32.
template <int IMPL, int HFN>
__device__ __forceinline__ void table_insert(const hawk_table& t, u64 key, u64 payload,
                                             int* flags) {
  u64* s = reinterpret_cast<u64*>(t.d_slots);
  if (key == kEmpty) {  // the EMPTY sentinel cannot be stored
    atomicOr(flags, HAWK_FLAG_TABLE_FULL);
    return;
  }
  if (IMPL == HAWK_LINEAR_PROBING) {
    const u64 mask = (u64)t.capacity - 1ull;
    u64 i = hash_slot<HFN>(key, t.seed[0], t.log2_capacity);
    for (u64 n = 0; n <= mask; ++n) {
      const u64 prev = atomicCAS(s + 2 * i, kEmpty, key);
      if (prev == kEmpty) {
        s[2 * i + 1] = payload;
        return;
      }
      if (prev == key) {  // planner_reference.cpp:171-174
        atomicOr(flags, HAWK_FLAG_DUPLICATE);
        return;
      }
      i = (i + 1) & mask;
    }
    atomicOr(flags, HAWK_FLAG_TABLE_FULL);
  } else {
    u64 k = key, v = payload;
    int sub = 0;
    for (int evictions = 0; evictions <= 32; ++evictions) {
      const u64 i = hash_slot<HFN>(k, t.seed[sub], t.log2_capacity);
      atomic_exch128(s + 2 * ((u64)sub * (u64)t.capacity + i), k, v);
      if (k == kEmpty) return;
      sub ^= 1;  // the evicted pair moves to its slot in the other sub-table
    }
    atomicOr(flags, HAWK_FLAG_CUCKOO_FAIL);
  }
}

// ---- aggregation tables: {state, keys..., accs...} slots --------

__host__ __device__ __forceinline__ u64 agg_identity(int fn, int type) {
  if (fn == HAWK_MIN) return type == HAWK_I64 ? 0x7fffffffffffffffull : 0x7ff0000000000000ull;
  if (fn == HAWK_MAX) return type == HAWK_I64 ? 0x8000000000000000ull : 0xfff0000000000000ull;
  return 0ull;
}

// Finds or inserts the group of `key` (words key[0], key[stride], ...) in an
// aggregation table with 2^log2cap slots (cuckoo: two sub-tables). Returns
// the slot, or nullptr when the table is full (LP) / both cuckoo candidates
// hold other groups. `fresh_counter` counts inserted groups.
template <int IMPL, int HFN, bool SHARED>
__device__ __forceinline__ u64* agg_find_or_insert(const KParams& kp, u64* slots, int log2cap,
                                                  const uint64_t* seeds, const u64* key,
                                                  int stride, u64* fresh_counter) {
  const hawk_pipeline& p = kp.p;
  const int K = p.nkeys;
  const int words = 1 + K + p.naggs;
  u64 x = key[0];
  for (int i = 1; i < K; ++i) x = combine_key(x, key[(size_t)i * stride]);
  const u64 tag = fmix64(x ^ 0x5bd1e9955bd1e995ull) | 1ull;  // odd: never EMPTY(0)/BUSY(2)
  const u64 cap = 1ull << log2cap;
  const int max_tries = IMPL == HAWK_LINEAR_PROBING ? (int)(cap < 4096 ? cap : 4096) : 2;
  u64 pos = hash_slot<HFN>(x, seeds[0], log2cap);
  for (int t = 0; t < max_tries; ++t) {
    if (IMPL == HAWK_CUCKOO && t == 1) pos = cap + hash_slot<HFN>(x, seeds[1], log2cap);
    u64* sl = slots + pos * (u64)words;
    u64 st = ld_volatile(sl);
    if (st == 0ull) {
      const u64 prev = atomicCAS(sl, 0ull, kBusy);
      if (prev == 0ull) {
        for (int i = 0; i < K; ++i) sl[1 + i] = key[(size_t)i * stride];
        for (int a = 0; a < p.naggs; ++a) sl[1 + K + a] = agg_identity(p.aggs[a].fn, p.aggs[a].type);
        if (SHARED) __threadfence_block(); else __threadfence();
        atomicExch(sl, tag);
        if (fresh_counter) atomicAdd(fresh_counter, 1ull);
        return sl;
      }
      st = prev;
    }
    while (st == kBusy) st = ld_volatile(sl);
    if (st == tag) {
      if (SHARED) __threadfence_block(); else __threadfence();
      bool eq = true;
      for (int i = 0; i < K; ++i) eq &= ld_volatile(sl + 1 + i) == key[(size_t)i * stride];
      if (eq) return sl;
    }
    if (IMPL == HAWK_LINEAR_PROBING) pos = (pos + 1) & (cap - 1ull);
  }
  return nullptr;
}

__device__ __forceinline__ void agg_update(u64* acc, int fn, int type, u64 v) {
  if (fn == HAWK_COUNT) {
    atomic_add_i(acc, 1ull);
  } else if (fn == HAWK_SUM) {
    if (type == HAWK_I64) atomic_add_i(acc, v); else atomic_add_f(acc, as_f64(v));
  } else if (fn == HAWK_MIN) {
    if (type == HAWK_I64) atomic_min_i(acc, v); else atomic_min_f(acc, as_f64(v));
  } else {
    if (type == HAWK_I64) atomic_max_i(acc, v); else atomic_max_f(acc, as_f64(v));
  }
}

// merge one partial accumulator (COUNT partials add like SUM)
__device__ __forceinline__ void agg_merge(u64* acc, int fn, int type, u64 v) {
  if (fn == HAWK_COUNT) atomic_add_i(acc, v); else agg_update(acc, fn, type, v);
}

// non-atomic combine of two partial accumulators
__device__ __forceinline__ u64 agg_combine(int fn, int type, u64 a, u64 b) {
  if (fn == HAWK_COUNT || (fn == HAWK_SUM && type == HAWK_I64)) return a + b;
  if (fn == HAWK_SUM) return as_bits(__dadd_rn(as_f64(a), as_f64(b)));
  if (type == HAWK_I64) {
    const i64 x = (i64)a, y = (i64)b;
    return (u64)(fn == HAWK_MIN ? (x < y ? x : y) : (x > y ? x : y));
  }
  const double x = as_f64(a), y = as_f64(b);
  return as_bits(fn == HAWK_MIN ? (x < y ? x : y) : (x > y ? x : y));
}

template <int T>
__device__ __forceinline__ u64 shfl_down64(u64 v, int o) {
  return __shfl_down_sync(0xffffffffu, v, o);
}

}  // namespace hk
