"""TEST INFRASTRUCTURE: builds identical inputs for the reference oracle and
the B200 engine, and compares their result tables with the reference's own
compare_result_tables (/root/reference/proj/src/planner_result.cpp:48-84)."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle_bridge import OraDb, OraTable, result_table  # noqa: E402
from paper_1709_00700_b200 import datagen as dg  # noqa: E402
from paper_1709_00700_b200 import queries as Q  # noqa: E402

MICRO = [("listing1", Q.LISTING1), ("listing2", Q.LISTING2), ("listing8", Q.LISTING8),
         ("listing9", Q.LISTING9), ("join2", Q.JOIN2), ("q6_lineorder", Q.Q6_ON_LINEORDER)]
BENCH = [(k, v[0]) for k, v in Q.BENCH.items()]

_TPCH = [dg.LINEITEM, dg.ORDERS, dg.CUSTOMER]
_SSB = [dg.LINEORDER, dg.DDATE, dg.SCUSTOMER, dg.SUPPLIER, dg.PART]


def micro_tables(n: int, seed: int) -> list[OraTable]:
    """gen_lineorder(n, seed) + gen_part/gen_supplier(1000, seed), SURVEY Appendix B."""
    return [OraTable.generated("lineorder", n, seed), OraTable.generated("part", 1000, seed),
            OraTable.generated("supplier", 1000, seed)]


def bench_tables(db: str, sf: float, seed: int = 42) -> list[OraTable]:
    """Synthetic TPC-H ('tpch') or SSB ('ssb') tables at scale factor sf."""
    out = []
    for t in (_TPCH if db == "tpch" else _SSB):
        name, cols = dg.host_table(t, sf, seed)
        out.append(OraTable.from_columns(name, cols))
    return out


def oracle_db(tables: list[OraTable]) -> OraDb:
    db = OraDb()
    for t in tables:
        db.add(t)
    return db


def load_engine(engine, tables: list[OraTable]):
    for t in tables:
        engine.put_table(t.name, t.columns(), distinct=t.distinct())


def compare(expected: OraTable, result) -> str | None:
    return expected.compare(result_table(result))
