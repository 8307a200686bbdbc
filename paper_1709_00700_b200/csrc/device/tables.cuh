// tables.cuh — open-addressed hash tables in HBM / shared memory:
// join tables (HASH_PUT / HASH_PROBE) and aggregation
// tables (HASH_AGGREGATE).
#pragma once

#include "interp.cuh"

namespace hk {

// ---- join tables: HASH_PROBE --------------------------

// dense key index (hawk_table.d_index): one 4-byte entry per key of the range
__device__ __forceinline__ int32_t index_find(const hawk_table& t, u64 key) {
  const u64 r = key - (u64)t.index_lo;
  return r < (u64)t.index_span ? __ldg(t.d_index + r) : -1;
}

template <int IMPL, int HFN>
__device__ __forceinline__ int32_t table_find(const hawk_table& t, u64 key) {
  if (t.d_index != nullptr) return index_find(t, key);
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

// HASH_PROBE of R rows at once: the home slots of every active row (both
// candidate slots for cuckoo) are loaded before any is inspected, so a warp
// has R (2R) independent random loads in flight instead of one; only rows
// whose home slot holds another key continue the linear-probing walk.
template <int IMPL, int HFN, int R>
__device__ __forceinline__ void table_find_rows(const hawk_table& t, const u64 (&key)[R],
                                                uint32_t act, int32_t (&out)[R]) {
  if (t.d_index != nullptr) {  // dense key range: direct-addressed, R loads in flight
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const u64 r = key[j] - (u64)t.index_lo;
      out[j] = (((act >> j) & 1u) && r < (u64)t.index_span) ? __ldg(t.d_index + r) : -1;
    }
    return;
  }
  const u64* s = reinterpret_cast<const u64*>(t.d_slots);
  u64 k0[R], v0[R], pos[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    pos[j] = hash_slot<HFN>(key[j], t.seed[0], t.log2_capacity);
    if ((act >> j) & 1u) ldg128_keep(s + 2 * pos[j], k0[j], v0[j]);
    else k0[j] = kEmpty, v0[j] = 0;
  }
  if (IMPL == HAWK_LINEAR_PROBING) {
    const u64 mask = (u64)t.capacity - 1ull;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      int32_t r = -1;
      if (((act >> j) & 1u) && key[j] != kEmpty) {
        u64 k = k0[j], v = v0[j], i = pos[j];
        while (k != key[j] && k != kEmpty) {
          i = (i + 1) & mask;
          ldg128(s + 2 * i, k, v);
        }
        r = k == key[j] ? (int32_t)v : -1;
      }
      out[j] = r;
    }
  } else {
    u64 k1[R], v1[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const u64 i = hash_slot<HFN>(key[j], t.seed[1], t.log2_capacity);
      if ((act >> j) & 1u) ldg128_keep(s + 2 * ((u64)t.capacity + i), k1[j], v1[j]);
      else k1[j] = kEmpty, v1[j] = 0;
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const bool ok = ((act >> j) & 1u) && key[j] != kEmpty;
      out[j] = !ok ? -1 : (k0[j] == key[j] ? (int32_t)v0[j] : (k1[j] == key[j] ? (int32_t)v1[j] : -1));
    }
  }
}

// dense key index insert: a plain store of the build row id into the key's
// entry. A duplicate build key (planner_reference.cpp:171-174) leaves fewer
// filled entries than inserted rows, which the build's count pass detects
// (abi.cu: index_fill_count_kernel), so no atomic is needed per row.
// Compiled single-pass builds (HK_INDEX_ATOMIC) exchange the entry instead
// and flag a duplicate on the spot, which saves the count pass over the
// whole index (TPC-H Q3 SF100: 600 MB).
__device__ __forceinline__ void index_insert(const hawk_table& t, u64 key, u64 payload, int* flags) {
  const u64 r = key - (u64)t.index_lo;
  if (r >= (u64)t.index_span) {  // outside the range the index was sized for
    atomicOr(flags, HAWK_FLAG_TABLE_FULL);
    return;
  }
#ifdef HK_INDEX_ATOMIC
  if (atomicExch(t.d_index + r, (int32_t)payload) != -1) atomicOr(flags, HAWK_FLAG_DUPLICATE);
#else
  t.d_index[r] = (int32_t)payload;
#endif
}

// HASH_PUT: LP = CAS-claim the key slot then store the
// payload; cuckoo = 128-bit exchange with an eviction chain of <= 32.
template <int IMPL, int HFN>
__device__ __forceinline__ void table_insert(const hawk_table& t, u64 key, u64 payload,
                                             int* flags) {
  if (t.d_index != nullptr) {
    index_insert(t, key, payload, flags);
    return;
  }
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

// HASH_PUT of R rows: linear probing CAS-claims the home slots of every
// active row back to back (R independent atomics in flight), and only rows
// that lost their home slot walk on; cuckoo inserts row by row.
template <int IMPL, int HFN, int R>
__device__ __forceinline__ void table_insert_rows(const hawk_table& t, const u64 (&key)[R],
                                                  const u64 (&payload)[R], uint32_t act,
                                                  int* flags) {
  if (t.d_index != nullptr) {
#pragma unroll
    for (int j = 0; j < R; ++j)
      if ((act >> j) & 1u) index_insert(t, key[j], payload[j], flags);
    return;
  }
  if (IMPL != HAWK_LINEAR_PROBING) {
#pragma unroll
    for (int j = 0; j < R; ++j)
      if ((act >> j) & 1u) table_insert<IMPL, HFN>(t, key[j], payload[j], flags);
    return;
  }
  u64* s = reinterpret_cast<u64*>(t.d_slots);
  const u64 mask = (u64)t.capacity - 1ull;
  u64 pos[R], prev[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    pos[j] = hash_slot<HFN>(key[j], t.seed[0], t.log2_capacity);
    prev[j] = kEmpty;
    if (((act >> j) & 1u) && key[j] != kEmpty) prev[j] = atomicCAS(s + 2 * pos[j], kEmpty, key[j]);
  }
#pragma unroll
  for (int j = 0; j < R; ++j) {
    if (!((act >> j) & 1u)) continue;
    if (key[j] == kEmpty) {
      atomicOr(flags, HAWK_FLAG_TABLE_FULL);
      continue;
    }
    if (prev[j] == kEmpty) {
      s[2 * pos[j] + 1] = payload[j];
      continue;
    }
    if (prev[j] == key[j]) {
      atomicOr(flags, HAWK_FLAG_DUPLICATE);
      continue;
    }
    u64 i = (pos[j] + 1) & mask;
    bool done = false;
    for (u64 n = 1; n <= mask; ++n) {
      const u64 pv = atomicCAS(s + 2 * i, kEmpty, key[j]);
      if (pv == kEmpty) {
        s[2 * i + 1] = payload[j];
        done = true;
        break;
      }
      if (pv == key[j]) {
        atomicOr(flags, HAWK_FLAG_DUPLICATE);
        done = true;
        break;
      }
      i = (i + 1) & mask;
    }
    if (!done) atomicOr(flags, HAWK_FLAG_TABLE_FULL);
  }
}

// ---- aggregation tables: {state, keys..., accs...} slots --------

constexpr int kAggBucket = 8;  // slots per cuckoo candidate position

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
                                                  int stride, u64* fresh_counter,
                                                  int* out_pos = nullptr) {
  const hawk_pipeline& p = kp.p;
  const int K = p.nkeys;
  const int words = 1 + K + p.naggs;
  u64 x = key[0];
  for (int i = 1; i < K; ++i) x = combine_key(x, key[(size_t)i * stride]);
  // one 64-bit hash gives both the home slot and the tag (odd: never
  // EMPTY(0) / BUSY(2)); the tag filters key comparisons
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
        for (int i = 0; i < K; ++i) sl[1 + i] = key[(size_t)i * stride];
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
      for (int i = 0; i < K; ++i) eq &= ld_volatile(sl + 1 + i) == key[(size_t)i * stride];
      if (eq) {
        if (out_pos) *out_pos = (int)pos;
        return sl;
      }
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

// agg_update on a shared-memory accumulator given by its 32-bit shared
// address: native shared atomics (ATOMS) instead of generic ones
template <int FN, int TY>
__device__ __forceinline__ void agg_update_smem(uint32_t a, u64 v) {
  if constexpr (FN == HAWK_COUNT) {
    asm volatile("atom.shared.add.u64 %0, [%1], 1;" : "=l"(v) : "r"(a) : "memory");
  } else if constexpr (FN == HAWK_SUM && TY == HAWK_I64) {
    asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
  } else if constexpr (FN == HAWK_SUM) {
    asm volatile("red.shared.add.f64 [%0], %1;" ::"r"(a), "d"(as_f64(v)) : "memory");
  } else if constexpr (FN == HAWK_MIN && TY == HAWK_I64) {
    asm volatile("red.shared.min.s64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
  } else if constexpr (FN == HAWK_MAX && TY == HAWK_I64) {
    asm volatile("red.shared.max.s64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
  } else {  // f64 MIN / MAX: CAS loop on the generic address
    agg_update(reinterpret_cast<u64*>(__cvta_shared_to_generic(a)), FN, TY, v);
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


}  // namespace hk
