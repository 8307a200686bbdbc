"""Synthetic TPC-H / SSB-shaped tables (include/hawk_gen.h) on the host.

Values come from the same counter-based generator the device uses
(hawk_b200_gen_column_host), so a host table and its device twin
(Engine.generate) hold identical rows. String columns are re-encoded to the
reference's first-appearance dictionary order
(/root/reference/proj/src/storage_table.cpp:127-135) so the parity harness can
hand the same codes to the reference oracle and to the engine.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native
from .engine import INT64, STRING, Column

LINEITEM, ORDERS, CUSTOMER, LINEORDER, DDATE, SCUSTOMER, SUPPLIER, PART = range(8)

_SEG = ["AUTOMOBILE", "BUILDING", "FURNITURE", "HOUSEHOLD", "MACHINERY"]
_REG = ["AFRICA", "AMERICA", "ASIA", "EUROPE", "MIDDLE EAST"]
_MFG = ["MFGR#1", "MFGR#2", "MFGR#3", "MFGR#4", "MFGR#5"]

# (table name, [(column, lexicon or None, domain)]) — mirrors hawk_gen.h
SCHEMA = {
    LINEITEM: ("lineitem", [("l_orderkey", None), ("l_quantity", None), ("l_extendedprice", None),
                            ("l_discount", None), ("l_tax", None), ("l_returnflag", None),
                            ("l_linestatus", None), ("l_shipdate", None)]),
    ORDERS: ("orders", [("o_orderkey", None), ("o_custkey", None), ("o_orderdate", None),
                        ("o_shippriority", None)]),
    CUSTOMER: ("customer", [("c_custkey", None), ("c_mktsegment", _SEG)]),
    LINEORDER: ("lineorder", [("lo_orderdate", None), ("lo_custkey", None), ("lo_partkey", None),
                              ("lo_suppkey", None), ("lo_quantity", None), ("lo_discount", None),
                              ("lo_extendedprice", None), ("lo_revenue", None),
                              ("lo_supplycost", None)]),
    DDATE: ("ddate", [("d_datekey", None), ("d_year", None)]),
    SCUSTOMER: ("customer", [("c_custkey", None), ("c_region", _REG), ("c_nation", None)]),
    SUPPLIER: ("supplier", [("s_suppkey", None), ("s_region", _REG), ("s_nation", None)]),
    PART: ("part", [("p_partkey", None), ("p_mfgr", _MFG)]),
}


def table_rows(table: int, sf: float) -> int:
    """hg_table_rows (include/hawk_gen.h)."""
    def scaled(base):
        return max(1, int(base * sf + 0.5))
    if table == LINEITEM:
        return 4 * scaled(1500000.0)
    if table == ORDERS:
        return scaled(1500000.0)
    if table == CUSTOMER:
        return scaled(150000.0)
    if table == LINEORDER:
        return scaled(6000000.0)
    if table == DDATE:
        return 2556
    if table == SCUSTOMER:
        return scaled(30000.0)
    if table == SUPPLIER:
        return scaled(2000.0)
    if table == PART:
        if sf < 1.0:
            return scaled(200000.0)
        lg, s = 0, sf
        while s >= 2.0:
            s *= 0.5
            lg += 1
        return 200000 * (1 + lg)
    raise ValueError(table)


def gen_column(table: int, col: int, sf: float, seed: int, begin: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    st = _native.b200().hawk_b200_gen_column_host(table, col, sf, seed, begin, n,
                                                    out.ctypes.data_as(C.c_void_p))
    if st != 0:
        raise RuntimeError(f"gen_column({table},{col}) failed: {st}")
    return out


def first_appearance(codes: np.ndarray, lexicon: list[str]) -> tuple[np.ndarray, list[str]]:
    """Re-encodes codes so the lexicon is in first-appearance order."""
    if len(codes) == 0:
        return codes.copy(), []
    uniq, first = np.unique(codes, return_index=True)
    order = uniq[np.argsort(first)]
    remap = np.full(len(lexicon), -1, dtype=np.int64)
    remap[order] = np.arange(len(order))
    return remap[codes], [lexicon[i] for i in order]


def host_table(table: int, sf: float, seed: int = 42, begin: int = 0,
               rows: int | None = None) -> tuple[str, list[Column]]:
    """A generated table as host columns (strings in first-appearance order)."""
    name, cols = SCHEMA[table]
    n = table_rows(table, sf) - begin if rows is None else rows
    out = []
    for ci, (cname, lex) in enumerate(cols):
        vals = gen_column(table, ci, sf, seed, begin, n)
        if lex is None:
            out.append(Column(cname, INT64, vals))
        else:
            codes, order = first_appearance(vals, lex)
            out.append(Column(cname, STRING, codes, order))
    return name, out
