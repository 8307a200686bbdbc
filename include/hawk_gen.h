/* hawk_gen.h — deterministic, counter-based synthetic TPC-H / SSB-shaped data.
 *
 * There is no dbgen and no network, so the benchmark tables are generated
 * in-process. Every value is a pure function of
 * (seed, table, column, row): each GPU generates its own shard of a fact table
 * on the device, and the host regenerates byte-identical chunks for the CPU
 * oracle. The same header compiles for host (C/C++) and device (CUDA).
 *
 * All columns are int64, as the reference stores them
 * (/root/reference/proj/include/hawk/storage/column.hpp:63-64). String columns
 * are dictionary codes into the lexicons below (codes in lexicon order; the
 * parity harness re-encodes to the reference's first-appearance order,
 * /root/reference/proj/src/storage_table.cpp:127-135). Dates are yyyymmdd
 * int64, so date predicates are plain integer comparisons (the reference
 * grammar has no date literals, /root/reference/proj/src/sql_parser.cpp:172-193).
 */
#ifndef HAWK_GEN_H
#define HAWK_GEN_H

#include <stdint.h>

#ifdef __CUDACC__
#define HG_FN __host__ __device__ __forceinline__
#else
#define HG_FN static inline
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum hawk_gen_table {
  HG_LINEITEM = 0,  /* TPC-H lineitem, 6M * sf rows (4 per order)            */
  HG_ORDERS = 1,    /* TPC-H orders, 1.5M * sf rows                           */
  HG_CUSTOMER = 2,  /* TPC-H customer, 150K * sf rows                         */
  HG_LINEORDER = 3, /* SSB lineorder, 6M * sf rows                            */
  HG_DDATE = 4,     /* SSB date dimension, 2556 rows                          */
  HG_SCUSTOMER = 5, /* SSB customer, 30K * sf rows                            */
  HG_SUPPLIER = 6,  /* SSB supplier, 2K * sf rows                             */
  HG_PART = 7,      /* SSB part, 200K * floor(1 + log2 sf) rows               */
  HG_NUM_TABLES = 8
};

/* column ids per table */
enum { HG_L_ORDERKEY, HG_L_QUANTITY, HG_L_EXTENDEDPRICE, HG_L_DISCOUNT, HG_L_TAX,
       HG_L_RETURNFLAG, HG_L_LINESTATUS, HG_L_SHIPDATE, HG_L_NCOLS };
enum { HG_O_ORDERKEY, HG_O_CUSTKEY, HG_O_ORDERDATE, HG_O_SHIPPRIORITY, HG_O_NCOLS };
enum { HG_C_CUSTKEY, HG_C_MKTSEGMENT, HG_C_NCOLS };
enum { HG_LO_ORDERDATE, HG_LO_CUSTKEY, HG_LO_PARTKEY, HG_LO_SUPPKEY, HG_LO_QUANTITY,
       HG_LO_DISCOUNT, HG_LO_EXTENDEDPRICE, HG_LO_REVENUE, HG_LO_SUPPLYCOST, HG_LO_NCOLS };
enum { HG_D_DATEKEY, HG_D_YEAR, HG_D_NCOLS };
enum { HG_SC_CUSTKEY, HG_SC_REGION, HG_SC_NATION, HG_SC_NCOLS };
enum { HG_S_SUPPKEY, HG_S_REGION, HG_S_NATION, HG_S_NCOLS };
enum { HG_P_PARTKEY, HG_P_MFGR, HG_P_NCOLS };

#define HG_DDATE_ROWS 2556
#define HG_ORDER_DAYS 2406 /* 1992-01-01 .. 1998-08-02 inclusive */

HG_FN uint64_t hg_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

HG_FN uint64_t hg_stream(uint64_t seed, int table, int col) {
  return hg_splitmix64(seed * 0x9E3779B97F4A7C15ull ^ ((uint64_t)table << 56) ^
                       ((uint64_t)col << 48));
}

HG_FN uint64_t hg_draw(uint64_t stream, int64_t row) {
  return hg_splitmix64(stream ^ hg_splitmix64((uint64_t)row));
}

HG_FN uint64_t hg_mulhi(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

/* uniform integer in [lo, hi] */
HG_FN int64_t hg_uniform(uint64_t stream, int64_t row, int64_t lo, int64_t hi) {
  return lo + (int64_t)hg_mulhi(hg_draw(stream, row), (uint64_t)(hi - lo + 1));
}

/* days since 1970-01-01 for a civil date (proleptic Gregorian) */
HG_FN int32_t hg_days_from_civil(int32_t y, int32_t m, int32_t d) {
  y -= m <= 2;
  int32_t era = (y >= 0 ? y : y - 399) / 400;
  int32_t yoe = y - era * 400;
  int32_t doy = (153 * (m + (m > 2 ? -3 : 9)) + 2) / 5 + d - 1;
  int32_t doe = yoe * 365 + yoe / 4 - yoe / 100 + doy;
  return era * 146097 + doe - 719468;
}

/* day index since 1992-01-01 -> yyyymmdd */
HG_FN int64_t hg_yyyymmdd(int32_t day) {
  int32_t z = day + 8035 + 719468; /* 8035 = days 1970-01-01 .. 1992-01-01 */
  int32_t era = z / 146097;
  int32_t doe = z - era * 146097;
  int32_t yoe = (doe - doe / 1460 + doe / 36524 - doe / 146096) / 365;
  int32_t y = yoe + era * 400;
  int32_t doy = doe - (365 * yoe + yoe / 4 - yoe / 100);
  int32_t mp = (5 * doy + 2) / 153;
  int32_t d = doy - (153 * mp + 2) / 5 + 1;
  int32_t m = mp < 10 ? mp + 3 : mp - 9;
  y += m <= 2;
  return (int64_t)y * 10000 + m * 100 + d;
}

/* day index of 1995-06-17 (TPC-H CURRENTDATE) */
HG_FN int32_t hg_current_day(void) { return 1263; }

HG_FN int64_t hg_rows_scaled(double sf, double base) {
  double r = base * sf + 0.5;
  int64_t n = (int64_t)r;
  return n < 1 ? 1 : n;
}

HG_FN int64_t hg_table_rows(int table, double sf) {
  switch (table) {
    case HG_LINEITEM: return 4 * hg_rows_scaled(sf, 1500000.0);
    case HG_ORDERS: return hg_rows_scaled(sf, 1500000.0);
    case HG_CUSTOMER: return hg_rows_scaled(sf, 150000.0);
    case HG_LINEORDER: return hg_rows_scaled(sf, 6000000.0);
    case HG_DDATE: return HG_DDATE_ROWS;
    case HG_SCUSTOMER: return hg_rows_scaled(sf, 30000.0);
    case HG_SUPPLIER: return hg_rows_scaled(sf, 2000.0);
    case HG_PART: {
      if (sf < 1.0) return hg_rows_scaled(sf, 200000.0);
      int64_t lg = 0;
      double s = sf;
      while (s >= 2.0) { s *= 0.5; ++lg; }
      return 200000 * (1 + lg);
    }
  }
  return 0;
}

HG_FN int hg_table_ncols(int table) {
  switch (table) {
    case HG_LINEITEM: return HG_L_NCOLS;
    case HG_ORDERS: return HG_O_NCOLS;
    case HG_CUSTOMER: return HG_C_NCOLS;
    case HG_LINEORDER: return HG_LO_NCOLS;
    case HG_DDATE: return HG_D_NCOLS;
    case HG_SCUSTOMER: return HG_SC_NCOLS;
    case HG_SUPPLIER: return HG_S_NCOLS;
    case HG_PART: return HG_P_NCOLS;
  }
  return 0;
}

/* o_orderdate as a day index for order i (shared by orders and lineitem) */
HG_FN int32_t hg_order_day(uint64_t seed, int64_t order) {
  return (int32_t)hg_uniform(hg_stream(seed, HG_ORDERS, HG_O_ORDERDATE), order, 0,
                             HG_ORDER_DAYS - 1);
}

HG_FN int32_t hg_ship_day(uint64_t seed, int64_t row) {
  return hg_order_day(seed, row >> 2) +
         (int32_t)hg_uniform(hg_stream(seed, HG_LINEITEM, HG_L_SHIPDATE), row, 1, 121);
}

HG_FN int64_t hg_lo_extendedprice(uint64_t seed, int64_t row) {
  return hg_uniform(hg_stream(seed, HG_LINEORDER, HG_LO_EXTENDEDPRICE), row, 90000, 10494950);
}
HG_FN int64_t hg_lo_discount(uint64_t seed, int64_t row) {
  return hg_uniform(hg_stream(seed, HG_LINEORDER, HG_LO_DISCOUNT), row, 0, 10);
}

/* The value of (table, col, row) at scale factor sf. */
HG_FN int64_t hg_value(int table, int col, int64_t row, double sf, uint64_t seed) {
  const uint64_t st = hg_stream(seed, table, col);
  switch (table) {
    case HG_LINEITEM:
      switch (col) {
        case HG_L_ORDERKEY: return (row >> 2) + 1;
        case HG_L_QUANTITY: return hg_uniform(st, row, 1, 50);
        case HG_L_EXTENDEDPRICE: return hg_uniform(st, row, 90000, 10494950);
        case HG_L_DISCOUNT: return hg_uniform(st, row, 0, 10);
        case HG_L_TAX: return hg_uniform(st, row, 0, 8);
        case HG_L_RETURNFLAG: {
          int32_t receipt = hg_ship_day(seed, row) + (int32_t)hg_uniform(st, row, 1, 30);
          if (receipt <= hg_current_day())
            return (hg_draw(hg_stream(seed, table, 100 + col), row) & 1) ? 'R' : 'A';
          return 'N';
        }
        case HG_L_LINESTATUS: return hg_ship_day(seed, row) > hg_current_day() ? 'O' : 'F';
        case HG_L_SHIPDATE: return hg_yyyymmdd(hg_ship_day(seed, row));
      }
      break;
    case HG_ORDERS:
      switch (col) {
        case HG_O_ORDERKEY: return row + 1;
        case HG_O_CUSTKEY: return hg_uniform(st, row, 1, hg_table_rows(HG_CUSTOMER, sf));
        case HG_O_ORDERDATE: return hg_yyyymmdd(hg_order_day(seed, row));
        case HG_O_SHIPPRIORITY: return 0;
      }
      break;
    case HG_CUSTOMER:
      switch (col) {
        case HG_C_CUSTKEY: return row + 1;
        case HG_C_MKTSEGMENT: return hg_uniform(st, row, 0, 4);
      }
      break;
    case HG_LINEORDER:
      switch (col) {
        case HG_LO_ORDERDATE: return hg_yyyymmdd((int32_t)hg_uniform(st, row, 0, HG_DDATE_ROWS - 1));
        case HG_LO_CUSTKEY: return hg_uniform(st, row, 1, hg_table_rows(HG_SCUSTOMER, sf));
        case HG_LO_PARTKEY: return hg_uniform(st, row, 1, hg_table_rows(HG_PART, sf));
        case HG_LO_SUPPKEY: return hg_uniform(st, row, 1, hg_table_rows(HG_SUPPLIER, sf));
        case HG_LO_QUANTITY: return hg_uniform(st, row, 1, 50);
        case HG_LO_DISCOUNT: return hg_lo_discount(seed, row);
        case HG_LO_EXTENDEDPRICE: return hg_lo_extendedprice(seed, row);
        case HG_LO_REVENUE:
          return hg_lo_extendedprice(seed, row) * (100 - hg_lo_discount(seed, row)) / 100;
        case HG_LO_SUPPLYCOST: return hg_uniform(st, row, 1000, 100000);
      }
      break;
    case HG_DDATE:
      switch (col) {
        case HG_D_DATEKEY: return hg_yyyymmdd((int32_t)row);
        case HG_D_YEAR: return hg_yyyymmdd((int32_t)row) / 10000;
      }
      break;
    case HG_SCUSTOMER:
    case HG_SUPPLIER: {
      const int64_t nation = hg_uniform(hg_stream(seed, table, 2), row, 0, 24);
      switch (col) {
        case 0: return row + 1;
        case 1: return nation / 5;
        case 2: return nation;
      }
      break;
    }
    case HG_PART:
      switch (col) {
        case HG_P_PARTKEY: return row + 1;
        case HG_P_MFGR: return hg_uniform(st, row, 0, 4);
      }
      break;
  }
  return 0;
}

/* ---- schema metadata (host only) ---------------------------------------- */

#define HG_KIND_INT64 0
#define HG_KIND_STRING 2

static inline const char* hg_table_name(int table) {
  static const char* const names[HG_NUM_TABLES] = {"lineitem", "orders",   "customer",
                                                   "lineorder", "ddate",   "customer",
                                                   "supplier",  "part"};
  return (table >= 0 && table < HG_NUM_TABLES) ? names[table] : "";
}

static inline const char* hg_col_name(int table, int col) {
  static const char* const li[] = {"l_orderkey", "l_quantity",   "l_extendedprice", "l_discount",
                                   "l_tax",      "l_returnflag", "l_linestatus",    "l_shipdate"};
  static const char* const od[] = {"o_orderkey", "o_custkey", "o_orderdate", "o_shippriority"};
  static const char* const cu[] = {"c_custkey", "c_mktsegment"};
  static const char* const lo[] = {"lo_orderdate", "lo_custkey", "lo_partkey",
                                   "lo_suppkey",   "lo_quantity", "lo_discount",
                                   "lo_extendedprice", "lo_revenue", "lo_supplycost"};
  static const char* const dd[] = {"d_datekey", "d_year"};
  static const char* const sc[] = {"c_custkey", "c_region", "c_nation"};
  static const char* const su[] = {"s_suppkey", "s_region", "s_nation"};
  static const char* const pa[] = {"p_partkey", "p_mfgr"};
  if (col < 0 || col >= hg_table_ncols(table)) return "";
  switch (table) {
    case HG_LINEITEM: return li[col];
    case HG_ORDERS: return od[col];
    case HG_CUSTOMER: return cu[col];
    case HG_LINEORDER: return lo[col];
    case HG_DDATE: return dd[col];
    case HG_SCUSTOMER: return sc[col];
    case HG_SUPPLIER: return su[col];
    case HG_PART: return pa[col];
  }
  return "";
}

/* number of lexicon entries of a string column, 0 for int64 columns */
static inline int hg_col_lexicon_size(int table, int col) {
  if (table == HG_CUSTOMER && col == HG_C_MKTSEGMENT) return 5;
  if ((table == HG_SCUSTOMER || table == HG_SUPPLIER) && col == 1) return 5;
  if (table == HG_PART && col == HG_P_MFGR) return 5;
  return 0;
}

static inline int hg_col_kind(int table, int col) {
  return hg_col_lexicon_size(table, col) ? HG_KIND_STRING : HG_KIND_INT64;
}

static inline const char* hg_col_lexicon(int table, int col, int code) {
  static const char* const seg[] = {"AUTOMOBILE", "BUILDING", "FURNITURE", "HOUSEHOLD",
                                    "MACHINERY"};
  static const char* const reg[] = {"AFRICA", "AMERICA", "ASIA", "EUROPE", "MIDDLE EAST"};
  static const char* const mfg[] = {"MFGR#1", "MFGR#2", "MFGR#3", "MFGR#4", "MFGR#5"};
  if (code < 0 || code >= hg_col_lexicon_size(table, col)) return "";
  if (table == HG_CUSTOMER) return seg[code];
  if (table == HG_PART) return mfg[code];
  return reg[code];
}

/* exact number of distinct values a column can take (an upper bound used to
 * size aggregation tables); 0 = unknown/unbounded */
static inline int64_t hg_col_domain(int table, int col, double sf) {
  switch (table) {
    case HG_LINEITEM:
      if (col == HG_L_RETURNFLAG) return 3;
      if (col == HG_L_LINESTATUS) return 2;
      if (col == HG_L_ORDERKEY) return hg_table_rows(HG_ORDERS, sf);
      if (col == HG_L_QUANTITY) return 50;
      if (col == HG_L_DISCOUNT) return 11;
      if (col == HG_L_TAX) return 9;
      break;
    case HG_ORDERS:
      if (col == HG_O_ORDERDATE) return HG_ORDER_DAYS;
      if (col == HG_O_SHIPPRIORITY) return 1;
      break;
    case HG_DDATE:
      if (col == HG_D_YEAR) return 7;
      break;
    case HG_SCUSTOMER:
    case HG_SUPPLIER:
      if (col == 1) return 5;
      if (col == 2) return 25;
      break;
    case HG_CUSTOMER:
      if (col == HG_C_MKTSEGMENT) return 5;
      break;
    case HG_PART:
      if (col == HG_P_MFGR) return 5;
      break;
    case HG_LINEORDER:
      if (col == HG_LO_QUANTITY) return 50;
      if (col == HG_LO_DISCOUNT) return 11;
      break;
  }
  return 0;
}

#ifdef __cplusplus
}
#endif

#endif /* HAWK_GEN_H */
