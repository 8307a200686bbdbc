// csv.cu — CSV ingest into device columns (include/hawk_b200_csv.h).
//
// Semantics are the reference's load_csv (proj/src/storage_csv.cpp:10-155):
// records end at a newline outside quotes, '"' opens a quoted field only at
// the start of a field, "" inside quotes is a literal quote, "\r\n" ends a
// record like "\n", an empty record ends the input, int64 fields follow
// std::from_chars (optional '-', decimal digits, no overflow) and float64
// fields std::stod with the whole field consumed. Strings are coded in
// first-appearance order (storage_table.cpp:127-135).
//
// Device plan: (1) per 1 KB chunk, count quotes; an exclusive scan gives the
// quote parity at every chunk start, so a newline is a record end iff the
// quotes before it are even; (2) count and (3) write the record ends;
// (4) one thread per record runs the reference's state machine over its
// bytes, checks that it ends exactly at the scanned boundary (a quote inside
// an unquoted field defeats the parity scan: the file then goes to the
// reference parser on the host, status HAWK_ERR_UNSUPPORTED), and writes the
// int64 / float64 fields; float fields outside the exactly-rounded fast path
// (<= 19 significant digits, |exponent| <= 22, mantissa < 2^53) are queued
// for std::stod on the host; string fields are hashed; (5) per string column
// a device hash table keeps every distinct string's first row, the host ranks
// them by it, and a last pass writes the codes after comparing each field
// with its representative byte for byte.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hawk_b200.h"
#include "hawk_b200_csv.h"

namespace {

using u64 = unsigned long long;
constexpr int64_t kChunk = 1024;

enum : int {
  kErrNone = 0,
  kErrFields = 1,     // wrong field count
  kErrInt = 2,        // invalid int64 literal
  kErrFloat = 3,      // invalid float64 literal (decided on the host)
  kErrStructure = 4,  // the parity scan disagrees with the state machine
  kErrCollision = 5   // two strings share a 64-bit hash
};

__global__ void quote_count_kernel(const char* __restrict__ t, int64_t n, int64_t* counts, int64_t nchunks) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const int64_t b = c * kChunk, e = min(n, b + kChunk);
  int64_t q = 0;
  for (int64_t i = b; i < e; ++i) q += t[i] == '"';
  counts[c] = q;
}

// record-ending newlines of a chunk (quote parity even before them);
// pass 0 counts, pass 1 writes positions at offsets[c]
__global__ void newline_kernel(const char* __restrict__ t, int64_t n, const int64_t* quotes_before,
                               int64_t nchunks, int64_t* counts, const int64_t* offsets, int64_t* ends,
                               int pass) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const int64_t b = c * kChunk, e = min(n, b + kChunk);
  int parity = (int)(quotes_before[c] & 1);
  int64_t k = 0;
  for (int64_t i = b; i < e; ++i) {
    const char ch = t[i];
    if (ch == '"') parity ^= 1;
    else if (ch == '\n' && parity == 0) {
      if (pass == 1) ends[offsets[c] + k] = i;
      ++k;
    }
  }
  if (pass == 0) counts[c] = k;
}

__device__ __forceinline__ int64_t record_start(const int64_t* ends, int64_t r) {
  return r == 0 ? 0 : ends[r - 1] + 1;
}

// first empty record (ends the input, storage_csv.cpp:81)
__global__ void empty_record_kernel(const char* __restrict__ t, int64_t n, const int64_t* ends, int64_t nrec,
                                    u64* first_empty) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrec; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = record_start(ends, r), e = ends[r];
    const bool newline_ended = e < n;
    if (e == s || (newline_ended && e == s + 1 && t[s] == '\r')) atomicMin(first_empty, (u64)r);
  }
}

struct ColumnOut {
  int32_t kind;
  int64_t* data;
  u64* hash;   // strings: FNV-1a of the unescaped field
  u64* loc;    // strings: field start << 24 | raw length << 1 | quoted
};

struct ParseArgs {
  const char* t;
  int64_t n;
  const int64_t* ends;
  int64_t first;  // first data record (header skipped)
  int64_t rows;
  char delim;
  int32_t ncols;
  ColumnOut cols[64];
  u64* error;     // (record << 16 | field << 4 | kind), atomicMin
  u64* escapes;   // float fields for the host: (record << 16 | field, loc) pairs
  u64* nescapes;
  int64_t max_escapes;
};

__device__ __forceinline__ void report(const ParseArgs& a, int64_t r, int f, int kind) {
  atomicMin(a.error, ((u64)r << 16) | ((u64)(f & 0xfff) << 4) | (u64)kind);
}

// from_chars(int64): optional '-', one or more digits, no overflow
__device__ bool parse_int64(const char* s, int64_t len, int64_t& out) {
  if (len <= 0) return false;
  int64_t i = 0;
  const bool neg = s[0] == '-';
  if (neg) i = 1;
  if (i >= len) return false;
  u64 v = 0;
  const u64 lim = neg ? 9223372036854775808ull : 9223372036854775807ull;
  for (; i < len; ++i) {
    const unsigned d = (unsigned)(s[i] - '0');
    if (d > 9) return false;
    if (v > (lim - d) / 10) return false;
    v = v * 10 + d;
  }
  out = neg ? (int64_t)(0 - v) : (int64_t)v;
  return true;
}

// exactly rounded fast path: [-]D+[.D*][(e|E)[+-]D+], <= 19 significant
// digits, mantissa < 2^53, |effective exponent| <= 22; else the host decides
__device__ int parse_float_fast(const char* s, int64_t len, double& out) {
  int64_t i = 0;
  bool neg = false;
  if (i < len && s[i] == '-') neg = true, ++i;
  u64 m = 0;
  int digits = 0, frac = 0, intd = 0;
  for (; i < len && s[i] >= '0' && s[i] <= '9'; ++i, ++intd) {
    if (m == 0 && s[i] == '0') continue;
    if (++digits > 19) return 0;
    m = m * 10 + (u64)(s[i] - '0');
  }
  if (intd == 0) return 0;
  if (i < len && s[i] == '.') {
    ++i;
    for (; i < len && s[i] >= '0' && s[i] <= '9'; ++i) {
      ++frac;
      if (m == 0 && s[i] == '0') continue;
      if (++digits > 19) return 0;
      m = m * 10 + (u64)(s[i] - '0');
    }
  }
  int e10 = 0;
  if (i < len && (s[i] == 'e' || s[i] == 'E')) {
    ++i;
    bool eneg = false;
    if (i < len && (s[i] == '+' || s[i] == '-')) eneg = s[i] == '-', ++i;
    int ed = 0;
    for (; i < len && s[i] >= '0' && s[i] <= '9'; ++i) {
      if (++ed > 4) return 0;
      e10 = e10 * 10 + (s[i] - '0');
    }
    if (ed == 0) return 0;
    if (eneg) e10 = -e10;
  }
  if (i != len) return 0;
  e10 -= frac;
  if (m >= (1ull << 53) || e10 < -22 || e10 > 22) return 0;
  const double p10[] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                        1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
  double v = (double)m;
  v = e10 >= 0 ? __dmul_rn(v, p10[e10]) : __ddiv_rn(v, p10[-e10]);
  out = neg ? -v : v;
  return 1;
}

__global__ void parse_kernel(const __grid_constant__ ParseArgs a) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < a.rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rec = a.first + r;
    const int64_t s = record_start(a.ends, rec), e = a.ends[rec];
    // the reference state machine (storage_csv.cpp:12-85) over [s, e]
    int64_t pos = s;
    int f = 0;
    bool ok = true;
    while (ok) {
      const int64_t fs = pos;  // raw field start
      bool quoted = false, was_quoted = false, field_empty = true;
      u64 h = 1469598103934665603ull;
      // numeric fields are parsed from the raw bytes when unquoted; quoted
      // numeric fields go through a small copy
      char buf[64];
      int blen = 0;
      bool buf_over = false;
      for (;;) {
        if (pos >= e) break;
        const char c = a.t[pos];
        if (quoted) {
          if (c == '"') {
            if (pos + 1 < e && a.t[pos + 1] == '"') {
              h = (h ^ (unsigned char)'"') * 1099511628211ull;
              if (blen < 64) buf[blen++] = '"'; else buf_over = true;
              pos += 2;
              field_empty = false;
              continue;
            }
            quoted = false;
            ++pos;
            continue;
          }
          h = (h ^ (unsigned char)c) * 1099511628211ull;
          if (blen < 64) buf[blen++] = c; else buf_over = true;
          field_empty = false;
          ++pos;
          continue;
        }
        if (c == '"' && field_empty) {
          quoted = was_quoted = true;
          ++pos;
          continue;
        }
        if (c == a.delim) break;
        if (c == '\r' && pos + 1 < a.n && a.t[pos + 1] == '\n' && pos + 1 == e) {
          ++pos;  // the '\r' of a "\r\n" terminator
          continue;
        }
        h = (h ^ (unsigned char)c) * 1099511628211ull;
        if (blen < 64) buf[blen++] = c; else buf_over = true;
        field_empty = false;
        ++pos;
      }
      if (quoted) {  // the record's end lies inside quotes: the scan disagreed
        report(a, r, f, kErrStructure);
        ok = false;
        break;
      }
      const int64_t fe = pos;
      if (f < a.ncols) {
        const ColumnOut& col = a.cols[f];
        if (col.kind == HAWK_CSV_INT64) {
          int64_t v = 0;
          if (buf_over || !parse_int64(buf, blen, v)) report(a, r, f, kErrInt);
          col.data[r] = v;
        } else if (col.kind == HAWK_CSV_FLOAT64) {
          double v = 0;
          if (!buf_over && parse_float_fast(buf, blen, v)) {
            col.data[r] = __double_as_longlong(v);
          } else {
            const u64 k = atomicAdd(a.nescapes, 1ull);
            if ((int64_t)k < a.max_escapes) {
              a.escapes[2 * k] = ((u64)r << 16) | (u64)f;
              a.escapes[2 * k + 1] =
                  ((u64)fs << 24) | ((u64)(fe - fs < (1 << 23) - 1 ? fe - fs : (1 << 23) - 1) << 1) | (was_quoted ? 1u : 0u);
            }
          }
        } else {
          col.hash[r] = h == 0 ? 1 : h;
          col.loc[r] = ((u64)fs << 24) | ((u64)(fe - fs < (1 << 23) - 1 ? fe - fs : (1 << 23) - 1) << 1) | (was_quoted ? 1u : 0u);
        }
      }
      ++f;
      if (pos >= e) break;
      ++pos;  // the delimiter
    }
    if (ok && f != a.ncols) report(a, r, min(f, a.ncols), kErrFields);
  }
}

// ---- string dictionaries -----------------------------------------------------------

struct DictSlot {
  u64 hash;  // 0 = empty
  u64 row;   // first row with this string; later its code
};

__global__ void dict_init_kernel(DictSlot* slots, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    slots[i] = DictSlot{0ull, ~0ull};
}

__global__ void dict_insert_kernel(DictSlot* slots, u64 mask, const u64* hash, int64_t rows) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const u64 h = hash[r];
    u64 i = (h * 0x9e3779b97f4a7c15ull) & mask;
    for (;;) {
      const u64 prev = atomicCAS(&slots[i].hash, 0ull, h);
      if (prev == 0ull || prev == h) {
        atomicMin(&slots[i].row, (u64)r);
        break;
      }
      i = (i + 1) & mask;
    }
  }
}

__global__ void dict_compact_kernel(const DictSlot* slots, int64_t nslots, u64* out, u64* count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nslots; i += (int64_t)gridDim.x * blockDim.x)
    if (slots[i].hash != 0ull) {
      const u64 k = atomicAdd(count, 1ull);
      out[2 * k] = (u64)i;             // slot
      out[2 * k + 1] = slots[i].row;   // first row
    }
}

__global__ void dict_set_code_kernel(DictSlot* slots, const u64* slot_of, const int64_t* code, int64_t n) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    slots[slot_of[k]].row = ((u64)slots[slot_of[k]].row << 32) | (u64)code[k];  // first row : code
}

__device__ bool same_field(const char* t, int64_t n, u64 la, u64 lb) {
  // compares two fields' unescaped contents (quoted fields may hold "")
  int64_t ia = (int64_t)(la >> 24), ea = ia + (int64_t)((la >> 1) & ((1u << 23) - 1));
  int64_t ib = (int64_t)(lb >> 24), eb = ib + (int64_t)((lb >> 1) & ((1u << 23) - 1));
  const bool qa = la & 1, qb = lb & 1;
  auto next = [&](int64_t& i, int64_t e, bool q, bool& inq, char& out) -> bool {
    while (i < e) {
      const char c = t[i];
      if (q && c == '"') {
        if (inq && i + 1 < e && t[i + 1] == '"') {
          out = '"';
          i += 2;
          return true;
        }
        inq = !inq;
        ++i;
        continue;
      }
      if (c == '\r' && i + 1 == e && e < n && t[e] == '\n') {  // the '\r' of a "\r\n" terminator
        ++i;
        return false;
      }
      out = c;
      ++i;
      return true;
    }
    return false;
  };
  bool inqa = false, inqb = false;
  for (;;) {
    char ca = 0, cb = 0;
    const bool ha = next(ia, ea, qa, inqa, ca), hb = next(ib, eb, qb, inqb, cb);
    if (ha != hb) return false;
    if (!ha) return true;
    if (ca != cb) return false;
  }
}

__global__ void dict_code_kernel(const char* t, int64_t n, const DictSlot* slots, u64 mask, const u64* hash,
                                 const u64* loc, int64_t rows, int64_t* out, u64* error, int field) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const u64 h = hash[r];
    u64 i = (h * 0x9e3779b97f4a7c15ull) & mask;
    while (slots[i].hash != h) i = (i + 1) & mask;
    const u64 v = slots[i].row;
    const int64_t first = (int64_t)(v >> 32);
    out[r] = (int64_t)(v & 0xffffffffull);
    if (first != r && !same_field(t, n, loc[r], loc[first]))
      atomicMin(error, ((u64)r << 16) | ((u64)(field & 0xfff) << 4) | (u64)kErrCollision);
  }
}

int32_t cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return HAWK_OK;
  if (e == cudaErrorMemoryAllocation) return HAWK_ERR_OUT_OF_MEMORY;
  std::fprintf(stderr, "hawk_b200 csv: CUDA error %s\n", cudaGetErrorString(e));
  return HAWK_ERR_CUDA;
}

#define HK_TRY(expr)                                   \
  do {                                                 \
    cudaError_t e_ = (expr);                           \
    if (e_ != cudaSuccess) return cuda_status(e_);     \
  } while (0)

int blocks_for(int64_t n, int per = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 148 * 16));
}

// reference field text (storage_csv.cpp quoting rules) of raw bytes [s, e)
std::string unescape(const std::string& text, int64_t s, int64_t e, bool quoted) {
  std::string out;
  bool inq = false;
  for (int64_t i = s; i < e; ++i) {
    const char c = text[(size_t)i];
    if (quoted && c == '"') {
      if (inq && i + 1 < e && text[(size_t)i + 1] == '"') {
        out.push_back('"');
        ++i;
        continue;
      }
      inq = !inq;
      continue;
    }
    if (c == '\r' && i + 1 == e && e < (int64_t)text.size() && text[(size_t)e] == '\n') continue;
    out.push_back(c);
  }
  return out;
}

}  // namespace

struct hawk_csv {
  hawk_ctx* ctx = nullptr;
  cudaStream_t stream = nullptr;
  std::string text;  // host copy (lexicon text, float fields for std::stod)
  char* d_text = nullptr;
  int64_t* d_ends = nullptr;
  int64_t records = 0, first = 0, rows = 0;
  char delim = ',';
  std::vector<std::vector<std::string>> lexicons;
  std::string error;
  int32_t host_parsed = 0;
};

extern "C" {

int32_t hawk_b200_csv_open(hawk_ctx* ctx, const void* text, int64_t bytes, char delimiter, int32_t header,
                           hawk_csv** out) {
  if (!ctx || (!text && bytes) || bytes < 0 || !out) return HAWK_ERR_ARGUMENT;
  auto* c = new hawk_csv;
  c->ctx = ctx;
  c->stream = static_cast<cudaStream_t>(hawk_b200_ctx_stream(ctx));
  c->text.assign(static_cast<const char*>(text), (size_t)bytes);
  c->delim = delimiter;
  cudaSetDevice(hawk_b200_ctx_device(ctx));
  const int64_t n = bytes;
  auto fail = [&](int32_t st) {
    hawk_b200_csv_close(c);
    return st;
  };
#define HK_CSV_TRY(expr)                                \
  do {                                                  \
    cudaError_t e_ = (expr);                            \
    if (e_ != cudaSuccess) return fail(cuda_status(e_)); \
  } while (0)
  HK_CSV_TRY(cudaMalloc(&c->d_text, (size_t)std::max<int64_t>(n, 1)));
  if (n) HK_CSV_TRY(cudaMemcpyAsync(c->d_text, text, (size_t)n, cudaMemcpyHostToDevice, c->stream));
  const int64_t nchunks = std::max<int64_t>(1, (n + kChunk - 1) / kChunk);
  int64_t *d_q = nullptr, *d_qs = nullptr, *d_cnt = nullptr, *d_off = nullptr;
  HK_CSV_TRY(cudaMalloc(&d_q, (size_t)(nchunks + 1) * 8));
  HK_CSV_TRY(cudaMalloc(&d_qs, (size_t)(nchunks + 1) * 8));
  HK_CSV_TRY(cudaMalloc(&d_cnt, (size_t)(nchunks + 1) * 8));
  HK_CSV_TRY(cudaMalloc(&d_off, (size_t)(nchunks + 1) * 8));
  HK_CSV_TRY(cudaMemsetAsync(d_q, 0, (size_t)(nchunks + 1) * 8, c->stream));
  HK_CSV_TRY(cudaMemsetAsync(d_cnt, 0, (size_t)(nchunks + 1) * 8, c->stream));
  quote_count_kernel<<<(unsigned)((nchunks + 255) / 256), 256, 0, c->stream>>>(c->d_text, n, d_q, nchunks);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_q, d_qs, nchunks + 1, c->stream);
  void* d_tmp = nullptr;
  HK_CSV_TRY(cudaMalloc(&d_tmp, std::max<size_t>(tmp_bytes, 16)));
  cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_q, d_qs, nchunks + 1, c->stream);
  newline_kernel<<<(unsigned)((nchunks + 255) / 256), 256, 0, c->stream>>>(c->d_text, n, d_qs, nchunks, d_cnt,
                                                                           nullptr, nullptr, 0);
  cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_cnt, d_off, nchunks + 1, c->stream);
  int64_t terminators = 0;
  HK_CSV_TRY(cudaMemcpyAsync(&terminators, d_off + nchunks, 8, cudaMemcpyDeviceToHost, c->stream));
  HK_CSV_TRY(cudaStreamSynchronize(c->stream));
  HK_CSV_TRY(cudaMalloc(&c->d_ends, (size_t)(terminators + 2) * 8));
  newline_kernel<<<(unsigned)((nchunks + 255) / 256), 256, 0, c->stream>>>(c->d_text, n, d_qs, nchunks, d_cnt,
                                                                           d_off, c->d_ends, 1);
  int64_t records = terminators;
  int64_t tail_start = 0;
  if (terminators > 0)
    HK_CSV_TRY(cudaMemcpyAsync(&tail_start, c->d_ends + terminators - 1, 8, cudaMemcpyDeviceToHost, c->stream));
  HK_CSV_TRY(cudaStreamSynchronize(c->stream));
  if (terminators > 0) tail_start += 1;
  if (tail_start < n) {  // bytes after the last newline form one more record
    const int64_t end = n;
    HK_CSV_TRY(cudaMemcpyAsync(c->d_ends + terminators, &end, 8, cudaMemcpyHostToDevice, c->stream));
    ++records;
  }
  u64* d_first_empty = reinterpret_cast<u64*>(d_q);  // reuse
  const u64 none = ~0ull;
  HK_CSV_TRY(cudaMemcpyAsync(d_first_empty, &none, 8, cudaMemcpyHostToDevice, c->stream));
  if (records > 0)
    empty_record_kernel<<<blocks_for(records), 256, 0, c->stream>>>(c->d_text, n, c->d_ends, records, d_first_empty);
  u64 first_empty = none;
  HK_CSV_TRY(cudaMemcpyAsync(&first_empty, d_first_empty, 8, cudaMemcpyDeviceToHost, c->stream));
  HK_CSV_TRY(cudaStreamSynchronize(c->stream));
  HK_CSV_TRY(cudaGetLastError());
  cudaFree(d_q);
  cudaFree(d_qs);
  cudaFree(d_cnt);
  cudaFree(d_off);
  cudaFree(d_tmp);
#undef HK_CSV_TRY
  c->records = first_empty == none ? records : (int64_t)first_empty;
  c->first = header && c->records > 0 ? 1 : 0;
  c->rows = c->records - c->first;
  *out = c;
  return HAWK_OK;
}

int64_t hawk_b200_csv_rows(const hawk_csv* c) { return c ? c->rows : -1; }
const char* hawk_b200_csv_error(const hawk_csv* c) { return c ? c->error.c_str() : ""; }
int32_t hawk_b200_csv_host_parsed(const hawk_csv* c) { return c ? c->host_parsed : 0; }

int64_t hawk_b200_csv_lexicon_size(const hawk_csv* c, int32_t col) {
  if (!c || col < 0 || (size_t)col >= c->lexicons.size()) return 0;
  return (int64_t)c->lexicons[(size_t)col].size();
}

const char* hawk_b200_csv_lexicon(const hawk_csv* c, int32_t col, int64_t code) {
  if (!c || col < 0 || (size_t)col >= c->lexicons.size() || code < 0 ||
      (size_t)code >= c->lexicons[(size_t)col].size())
    return nullptr;
  return c->lexicons[(size_t)col][(size_t)code].c_str();
}

int32_t hawk_b200_csv_parse(hawk_csv* c, int32_t ncols, const int32_t* kinds, int64_t* const* d_columns,
                            int64_t* error_record, int32_t* error_field) {
  if (!c || ncols < 1 || ncols > 64 || !kinds || !d_columns) return HAWK_ERR_ARGUMENT;
  cudaSetDevice(hawk_b200_ctx_device(c->ctx));
  c->lexicons.assign((size_t)ncols, {});
  c->error.clear();
  if (error_record) *error_record = -1;
  if (error_field) *error_field = -1;
  const int64_t rows = c->rows;
  if (rows <= 0) return HAWK_OK;
  ParseArgs a{};
  a.t = c->d_text;
  a.n = (int64_t)c->text.size();
  a.ends = c->d_ends;
  a.first = c->first;
  a.rows = rows;
  a.delim = c->delim;
  a.ncols = ncols;
  std::vector<void*> scratch;
  auto cleanup = [&] {
    for (void* p : scratch) cudaFree(p);
  };
  auto alloc = [&](size_t bytes, void** p) {
    cudaError_t e = cudaMalloc(p, std::max<size_t>(bytes, 16));
    if (e == cudaSuccess) scratch.push_back(*p);
    return e;
  };
#define HK_P_TRY(expr)                                      \
  do {                                                      \
    cudaError_t e_ = (expr);                                \
    if (e_ != cudaSuccess) {                                \
      cleanup();                                            \
      return cuda_status(e_);                               \
    }                                                       \
  } while (0)
  for (int f = 0; f < ncols; ++f) {
    a.cols[f].kind = kinds[f];
    a.cols[f].data = d_columns[f];
    if (kinds[f] == HAWK_CSV_STRING) {
      HK_P_TRY(alloc((size_t)rows * 8, reinterpret_cast<void**>(&a.cols[f].hash)));
      HK_P_TRY(alloc((size_t)rows * 8, reinterpret_cast<void**>(&a.cols[f].loc)));
    }
  }
  const int64_t max_escapes = std::min<int64_t>(rows * ncols, int64_t(1) << 22);
  u64* d_ctrl = nullptr;  // [0] error, [1] escape count
  HK_P_TRY(alloc(16, reinterpret_cast<void**>(&d_ctrl)));
  HK_P_TRY(alloc((size_t)max_escapes * 16, reinterpret_cast<void**>(&a.escapes)));
  const u64 init[2] = {~0ull, 0ull};
  HK_P_TRY(cudaMemcpyAsync(d_ctrl, init, 16, cudaMemcpyHostToDevice, c->stream));
  a.error = d_ctrl;
  a.nescapes = d_ctrl + 1;
  a.max_escapes = max_escapes;
  parse_kernel<<<blocks_for(rows), 256, 0, c->stream>>>(a);
  HK_P_TRY(cudaGetLastError());
  u64 ctrl[2];
  HK_P_TRY(cudaMemcpyAsync(ctrl, d_ctrl, 16, cudaMemcpyDeviceToHost, c->stream));
  HK_P_TRY(cudaStreamSynchronize(c->stream));
  auto fail_with = [&](u64 err) {
    const int64_t r = (int64_t)(err >> 16);
    const int f = (int)((err >> 4) & 0xfff), kind = (int)(err & 15);
    if (error_record) *error_record = r;
    if (error_field) *error_field = f;
    cleanup();
    if (kind == kErrStructure || kind == kErrCollision) {
      c->error = kind == kErrStructure ? "quoting the parallel record scan cannot follow (record " +
                                             std::to_string(r) + ")"
                                       : "string hash collision";
      c->host_parsed = 1;
      return HAWK_ERR_UNSUPPORTED;  // the caller parses on the host (storage_csv.cpp)
    }
    c->error = kind == kErrFields ? "record " + std::to_string(r) + ": wrong number of fields"
               : kind == kErrInt  ? "record " + std::to_string(r) + " field " + std::to_string(f) +
                                       ": invalid int64 literal"
                                  : "record " + std::to_string(r) + " field " + std::to_string(f) +
                                       ": invalid float64 literal";
    return HAWK_ERR_INVALID_PARAMS;
  };
  if (ctrl[0] != ~0ull) return fail_with(ctrl[0]);
  // float fields for std::stod (storage_csv.cpp:95-106), patched into the columns
  const int64_t nesc = (int64_t)ctrl[1];
  if (nesc > max_escapes) {
    cleanup();
    c->error = "too many float fields outside the device fast path";
    c->host_parsed = 1;
    return HAWK_ERR_UNSUPPORTED;
  }
  if (nesc > 0) {
    std::vector<u64> esc((size_t)nesc * 2);
    HK_P_TRY(cudaMemcpy(esc.data(), a.escapes, esc.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<std::vector<std::pair<int64_t, int64_t>>> patches((size_t)ncols);
    for (int64_t k = 0; k < nesc; ++k) {
      const u64 id = esc[(size_t)(2 * k)], loc = esc[(size_t)(2 * k + 1)];
      const int64_t r = (int64_t)(id >> 16);
      const int f = (int)(id & 0xffff);
      const int64_t s0 = (int64_t)(loc >> 24), len = (int64_t)((loc >> 1) & ((1u << 23) - 1));
      const std::string field = unescape(c->text, s0, s0 + len, loc & 1);
      double v = 0;
      bool ok = true;
      try {
        std::size_t used = 0;
        v = std::stod(field, &used);
        ok = used == field.size();
      } catch (const std::exception&) {
        ok = false;
      }
      if (!ok) return fail_with(((u64)r << 16) | ((u64)f << 4) | (u64)kErrFloat);
      int64_t bits;
      std::memcpy(&bits, &v, 8);
      patches[(size_t)f].push_back({r, bits});
    }
    for (int f = 0; f < ncols; ++f)
      for (const auto& [r, bits] : patches[(size_t)f])
        HK_P_TRY(cudaMemcpyAsync(d_columns[f] + r, &bits, 8, cudaMemcpyHostToDevice, c->stream));
    HK_P_TRY(cudaStreamSynchronize(c->stream));
  }
  // string dictionaries in first-appearance order
  for (int f = 0; f < ncols; ++f) {
    if (kinds[f] != HAWK_CSV_STRING) continue;
    int L = 4;
    while ((int64_t(1) << L) < 2 * rows) ++L;
    const int64_t nslots = int64_t(1) << L;
    DictSlot* slots = nullptr;
    HK_P_TRY(alloc((size_t)nslots * sizeof(DictSlot), reinterpret_cast<void**>(&slots)));
    dict_init_kernel<<<blocks_for(nslots), 256, 0, c->stream>>>(slots, nslots);  // empty, row ~0
    dict_insert_kernel<<<blocks_for(rows), 256, 0, c->stream>>>(slots, (u64)(nslots - 1), a.cols[f].hash, rows);
    HK_P_TRY(cudaGetLastError());
    HK_P_TRY(cudaStreamSynchronize(c->stream));
    u64* d_list = nullptr;
    u64* d_count = nullptr;
    HK_P_TRY(alloc((size_t)rows * 16, reinterpret_cast<void**>(&d_list)));
    HK_P_TRY(alloc(8, reinterpret_cast<void**>(&d_count)));
    HK_P_TRY(cudaMemsetAsync(d_count, 0, 8, c->stream));
    dict_compact_kernel<<<blocks_for(nslots), 256, 0, c->stream>>>(slots, nslots, d_list, d_count);
    u64 distinct = 0;
    HK_P_TRY(cudaMemcpyAsync(&distinct, d_count, 8, cudaMemcpyDeviceToHost, c->stream));
    HK_P_TRY(cudaStreamSynchronize(c->stream));
    std::vector<u64> list((size_t)distinct * 2);
    HK_P_TRY(cudaMemcpy(list.data(), d_list, list.size() * 8, cudaMemcpyDeviceToHost));
    std::vector<size_t> order((size_t)distinct);
    for (size_t k = 0; k < order.size(); ++k) order[k] = k;
    std::sort(order.begin(), order.end(), [&](size_t x, size_t y) { return list[2 * x + 1] < list[2 * y + 1]; });
    std::vector<int64_t> code((size_t)distinct);
    std::vector<u64> first_loc((size_t)distinct);
    for (size_t rank = 0; rank < order.size(); ++rank) code[order[rank]] = (int64_t)rank;
    // the representatives' text
    std::vector<std::string>& lex = c->lexicons[(size_t)f];
    lex.resize((size_t)distinct);
    for (size_t k = 0; k < (size_t)distinct; ++k) {
      u64 loc = 0;
      HK_P_TRY(cudaMemcpy(&loc, a.cols[f].loc + list[2 * k + 1], 8, cudaMemcpyDeviceToHost));
      const int64_t s = (int64_t)(loc >> 24), len = (int64_t)((loc >> 1) & ((1u << 23) - 1));
      lex[(size_t)code[k]] = unescape(c->text, s, s + len, loc & 1);
    }
    u64* d_slot_of = nullptr;
    int64_t* d_code = nullptr;
    HK_P_TRY(alloc((size_t)distinct * 8, reinterpret_cast<void**>(&d_slot_of)));
    HK_P_TRY(alloc((size_t)distinct * 8, reinterpret_cast<void**>(&d_code)));
    std::vector<u64> slot_of((size_t)distinct);
    for (size_t k = 0; k < (size_t)distinct; ++k) slot_of[k] = list[2 * k];
    HK_P_TRY(cudaMemcpy(d_slot_of, slot_of.data(), slot_of.size() * 8, cudaMemcpyHostToDevice));
    HK_P_TRY(cudaMemcpy(d_code, code.data(), code.size() * 8, cudaMemcpyHostToDevice));
    dict_set_code_kernel<<<blocks_for((int64_t)distinct), 256, 0, c->stream>>>(slots, d_slot_of, d_code,
                                                                                (int64_t)distinct);
    dict_code_kernel<<<blocks_for(rows), 256, 0, c->stream>>>(c->d_text, a.n, slots, (u64)(nslots - 1), a.cols[f].hash,
                                                             a.cols[f].loc, rows, d_columns[f], d_ctrl, f);
    HK_P_TRY(cudaMemcpyAsync(ctrl, d_ctrl, 8, cudaMemcpyDeviceToHost, c->stream));
    HK_P_TRY(cudaStreamSynchronize(c->stream));
    if (ctrl[0] != ~0ull) return fail_with(ctrl[0]);
  }
#undef HK_P_TRY
  cleanup();
  return HAWK_OK;
}

int32_t hawk_b200_csv_close(hawk_csv* c) {
  if (!c) return HAWK_OK;
  if (c->d_text) cudaFree(c->d_text);
  if (c->d_ends) cudaFree(c->d_ends);
  delete c;
  return HAWK_OK;
}

}  // extern "C"
