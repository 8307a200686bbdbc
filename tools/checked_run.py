"""Instrumented run (compute-sanitizer is closed on this GPU pool): every
compiled program carries device-side bounds checks (engine option "checked",
-DHK_CHECKED: column rows inside the driver's extent, payload row ids >= 0,
compaction-queue capacity, private-accumulator words, CTA-table slots, dense
lookaside indices), and every query's result is compared with the reference's
reference_execute. Covers every kernel role under four variants: AGGREGATE /
HASH_AGGREGATE local and global, PROJECT single- and multi-pass, HASH_PUT
single/multi, compacted probe chains, CROSS_JOIN, the BASELINE shapes.
  python tools/checked_run.py  -> one line per query, "violations: 0" at the end"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

import harness  # noqa: E402
from oracle_bridge import OraTable  # noqa: E402
from paper_1709_00700_b200 import Engine  # noqa: E402
from paper_1709_00700_b200 import queries as Q  # noqa: E402
from paper_1709_00700_b200.engine import INT64, Column, HawkError  # noqa: E402

CONFIGS = [
    "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8",
    "multi_pass/sequential/predicated/tm=1024;global_hash/sequential/predicated/cuckoo/multiply_shift/wg=128",
    "single_pass/coalesced/predicated/u=2;local_hash/coalesced/predicated/cuckoo/murmur/wg=512/ht=1/u=2",
    "multi_pass/coalesced/branched/tm=64/u=4;global_hash/coalesced/branched/linear_probing/murmur/wg=1024/u=4",
]


def main():
    failures = violations = checked = 0
    e = Engine(0)
    e.set_option("checked", 1)
    tables = harness.micro_tables(50000, 7)
    harness.load_engine(e, tables)
    db = harness.oracle_db(tables)
    xa = [Column("a_k", INT64, np.array([3, 1, 4], np.int64)), Column("a_w", INT64, np.array([2, 7, 1], np.int64))]
    e.put_table("xa", xa)
    db.add(OraTable.from_columns("xa", xa))
    sqls = [sql for _, sql in harness.MICRO] + [
        "select lo_quantity, min(lo_revenue), max(lo_discount * 0.5) from lineorder group by lo_quantity",
        "select count(*), sum(lo_quantity*a_w) from xa, lineorder where a_w < 5 and lo_quantity < 10",
    ]
    runs = [(e, db, sql) for sql in sqls]
    extra = []
    for db_name, keys in (("tpch", ("tpch_q6", "tpch_q1", "tpch_q3")), ("ssb", ("ssb_q11", "ssb_q41"))):
        e2 = Engine(0)
        e2.set_option("checked", 1)
        t2 = harness.bench_tables(db_name, 0.05, 42)
        harness.load_engine(e2, t2)
        db2 = harness.oracle_db(t2)
        extra.append(e2)
        runs += [(e2, db2, Q.BENCH[k][0]) for k in keys]
    for eng, odb, sql in runs:
        expected = odb.execute(sql)
        for cfg in CONFIGS:
            checked += 1
            try:
                diff = harness.compare(expected, eng.run(sql, cfg))
            except HawkError as ex:
                if "bounds check" in str(ex):
                    violations += 1
                failures += 1
                print(f"FAIL {sql[:60]} [{cfg}]: {ex}", flush=True)
                continue
            if diff is not None:
                failures += 1
                print(f"DIFF {sql[:60]} [{cfg}]: {diff}", flush=True)
        print(f"ok {sql[:90]}", flush=True)
    for x in extra:
        x.close()
    e.close()
    print(f"checked runs: {checked}, violations: {violations}, failures: {failures}", flush=True)
    sys.exit(1 if failures else 0)


if __name__ == "__main__":
    main()
