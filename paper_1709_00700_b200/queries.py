"""The benchmark queries in the reference's SQL grammar.

BASELINE queries from SURVEY.md Appendix A (all five parse, lower and run in
the reference oracle), and the paper's micro-benchmarks (PAPER.md:405-406,
:579-580, :1509, :1523) over gen_lineorder
(/root/reference/proj/src/storage_generator.cpp:33-65).
"""
from __future__ import annotations

from . import datagen as dg

TPCH_Q6 = ("select sum(l_extendedprice*l_discount) as revenue from lineitem "
           "where l_shipdate >= 19940101 and l_shipdate < 19950101 and l_discount >= 5 "
           "and l_discount <= 7 and l_quantity < 24")

TPCH_Q1 = ("select l_returnflag, l_linestatus, sum(l_quantity) as sum_qty, "
           "sum(l_extendedprice) as sum_base_price, "
           "sum(l_extendedprice*(100-l_discount)) as sum_disc_price, "
           "sum(l_extendedprice*(100-l_discount)*(100+l_tax)) as sum_charge, "
           "avg(l_quantity) as avg_qty, avg(l_extendedprice) as avg_price, "
           "avg(l_discount) as avg_disc, count(*) as count_order from lineitem "
           "where l_shipdate <= 19980902 group by l_returnflag, l_linestatus")

SSB_Q11 = ("select sum(lo_extendedprice*lo_discount) as revenue from ddate, lineorder "
           "where lo_orderdate = d_datekey and d_year = 1993 and lo_discount >= 1 "
           "and lo_discount <= 3 and lo_quantity < 25")

SSB_Q41 = ("select d_year, c_nation, sum(lo_revenue - lo_supplycost) as profit "
           "from ddate, customer, supplier, part, lineorder "
           "where lo_custkey = c_custkey and lo_suppkey = s_suppkey and lo_partkey = p_partkey "
           "and lo_orderdate = d_datekey and c_region = 'AMERICA' and s_region = 'AMERICA' "
           "and p_mfgr <> 'MFGR#3' and p_mfgr <> 'MFGR#4' and p_mfgr <> 'MFGR#5' "
           "group by d_year, c_nation")

TPCH_Q3 = ("select l_orderkey, sum(l_extendedprice*(100-l_discount)) as revenue, o_orderdate, "
           "o_shippriority from orders, customer, lineitem "
           "where c_mktsegment = 'BUILDING' and c_custkey = o_custkey and l_orderkey = o_orderkey "
           "and o_orderdate < 19950315 and l_shipdate > 19950315 "
           "group by l_orderkey, o_orderdate, o_shippriority")

# paper micro-benchmarks over gen_lineorder (+ gen_part / gen_supplier)
LISTING1 = "select lo_linenumber, lo_quantity, lo_revenue from lineorder where lo_quantity<25"
LISTING2 = ("select lo_linenumber, lo_quantity, lo_revenue from lineorder where lo_quantity<25 "
            "and lo_discount<=3 and lo_discount>=1 and lo_revenue>4900000")
LISTING8 = "select sum(lo_quantity) from lineorder group by lo_shipmode"
LISTING9 = "select lo_partkey, sum(lo_quantity) from lineorder group by lo_partkey"
JOIN2 = ("select p_size, sum(lo_revenue), count(*) from part, supplier, lineorder "
         "where lo_partkey = p_partkey and lo_suppkey = s_suppkey and p_size < 25 group by p_size")
Q6_ON_LINEORDER = ("select sum(lo_extendedprice*lo_discount) as revenue from lineorder where "
                   "lo_orderdate >= 19940101 and lo_orderdate < 19950101 and lo_discount >= 5 "
                   "and lo_discount <= 7 and lo_quantity < 24")

# BASELINE configs -> (sql, tables it needs, fact table)
BENCH = {
    "tpch_q6": (TPCH_Q6, [dg.LINEITEM], dg.LINEITEM),
    "tpch_q1": (TPCH_Q1, [dg.LINEITEM], dg.LINEITEM),
    "ssb_q11": (SSB_Q11, [dg.DDATE, dg.LINEORDER], dg.LINEORDER),
    "ssb_q41": (SSB_Q41, [dg.DDATE, dg.SCUSTOMER, dg.SUPPLIER, dg.PART, dg.LINEORDER],
                dg.LINEORDER),
    "tpch_q3": (TPCH_Q3, [dg.ORDERS, dg.CUSTOMER, dg.LINEITEM], dg.LINEITEM),
}

# columns each query reads (algorithmic bytes)
FACT_COLUMNS = {
    "tpch_q6": ["l_shipdate", "l_discount", "l_quantity", "l_extendedprice"],
    "tpch_q1": ["l_shipdate", "l_returnflag", "l_linestatus", "l_quantity", "l_extendedprice",
                "l_discount", "l_tax"],
    "ssb_q11": ["lo_orderdate", "lo_discount", "lo_quantity", "lo_extendedprice"],
    "ssb_q41": ["lo_custkey", "lo_suppkey", "lo_partkey", "lo_orderdate", "lo_revenue",
                "lo_supplycost"],
    "tpch_q3": ["l_orderkey", "l_shipdate", "l_extendedprice", "l_discount"],
}
