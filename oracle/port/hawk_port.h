/* TEST INFRASTRUCTURE ONLY — never linked into the product.
 *
 * hawk_port: a CPU restatement of the reference oracle's semantics
 * (/root/reference/proj/src/planner_reference.cpp) for the five BASELINE
 * queries, streaming over column arrays instead of
 * materialising one RefRow per base row (planner_reference.cpp:145-155), so it
 * runs at SF10..SF100 where reference_execute does not fit in RAM
 * (SURVEY.md §0.4). It is pinned bit-exactly against reference_execute at
 * small scale factors by tests/test_oracle.py, and doubles as the host-parallel
 * CPU baseline ("port" in bench.py's cpu_baseline).
 *
 * Result rows are written in SELECT order, one int64 word per value; float
 * values (AVG) are stored as IEEE-754 bit patterns.
 */
#ifndef HAWK_PORT_H
#define HAWK_PORT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { PORT_Q6 = 0, PORT_Q1 = 1, PORT_SSB11 = 2, PORT_SSB41 = 3, PORT_Q3 = 4 };

/* Fills rows [begin, begin + n) of a generated column (include/hawk_gen.h). */
void port_gen(int table, int col, double sf, uint64_t seed, int64_t begin, int64_t n,
              int64_t* out, int threads);

/* Number of output columns of a query. */
int port_width(int query);

/* Runs `query` over materialised columns. `cols` lists, in order:
 *   Q6    : l_shipdate, l_discount, l_quantity, l_extendedprice           (n rows)
 *   Q1    : l_shipdate, l_returnflag, l_linestatus, l_quantity,
 *           l_extendedprice, l_discount, l_tax                            (n rows)
 *   SSB11 : lo_orderdate, lo_discount, lo_quantity, lo_extendedprice     (n rows)
 *           + d_datekey, d_year                                          (dim_rows[0])
 *   SSB41 : lo_custkey, lo_suppkey, lo_partkey, lo_orderdate, lo_revenue,
 *           lo_supplycost                                                (n rows)
 *           + c_custkey, c_region, c_nation (dim_rows[0])
 *           + s_suppkey, s_region (dim_rows[1]) + p_partkey, p_mfgr (dim_rows[2])
 *           + d_datekey, d_year (dim_rows[3])
 *   Q3    : l_orderkey, l_shipdate, l_extendedprice, l_discount          (n rows)
 *           + o_orderkey, o_custkey, o_orderdate, o_shippriority         (dim_rows[0])
 *           + c_custkey, c_mktsegment                                    (dim_rows[1])
 * String columns are codes: `codes` gives the code of each string literal the
 * query compares with (SSB41: 'AMERICA' in c_region, in s_region, then the
 * codes of 'MFGR#3','MFGR#4','MFGR#5'; Q3: 'BUILDING'); -1 = absent.
 * Returns the number of result rows written to out (capacity out_rows);
 * -1 if out is too small. */
int64_t port_run(int query, const int64_t* const* cols, int64_t n, const int64_t* dim_rows,
                 const int64_t* codes, int threads, int64_t* out, int64_t out_rows);

/* The streaming form (SF100): the same query over fact rows
 * [row_begin, row_begin + n) of the generated tables at scale factor sf, each
 * worker regenerating its fact rows chunk by chunk (include/hawk_gen.h);
 * dimension tables are generated whole. Nothing fact-sized is materialised. */
int64_t port_run_gen(int query, double sf, uint64_t seed, int64_t row_begin, int64_t n,
                     const int64_t* codes, int threads, int64_t* out, int64_t out_rows);

#ifdef __cplusplus
}
#endif

#endif /* HAWK_PORT_H */
