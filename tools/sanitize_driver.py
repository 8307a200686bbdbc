"""Exercises every kernel role of libhawk_b200 once per jit mode on small
inputs, for compute-sanitizer (tools/sanitize.sh): AGGREGATE local/global,
HASH_AGGREGATE local/global (private accumulators, CTA table, dense
lookaside), PROJECT single-pass and multi-pass (count/scan/scatter),
HASH_PUT single/multi-pass (LP, cuckoo, dense index, key bitmaps), probes with
live-row compaction, CROSS_JOIN expansion, the standalone table / prefix-sum
/ column-range kernels, the group merge and the CSV parser."""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

import harness  # noqa: E402
from paper_1709_00700_b200 import Engine  # noqa: E402
from paper_1709_00700_b200 import queries as Q  # noqa: E402
from paper_1709_00700_b200.engine import FLOAT64, INT64, STRING, Column  # noqa: E402

CONFIGS = [
    "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8",
    "multi_pass/sequential/predicated/tm=1024;global_hash/sequential/predicated/cuckoo/multiply_shift/wg=128",
    "single_pass/coalesced/predicated/u=2;local_hash/coalesced/predicated/cuckoo/murmur/wg=64/ht=1/u=2",
    "multi_pass/coalesced/branched/tm=64/u=4;global_hash/coalesced/branched/linear_probing/murmur/wg=1024/u=4",
]


def main():
    jit_modes = [int(x) for x in os.environ.get("SAN_JIT", "1,0").split(",")]
    e = Engine(0)
    tables = harness.micro_tables(int(os.environ.get("SAN_ROWS", "20000")), 7)
    harness.load_engine(e, tables)
    e.put_table("xa", [Column("a_k", INT64, np.array([3, 1, 4], np.int64)),
                       Column("a_w", INT64, np.array([2, 7, 1], np.int64))])
    sqls = [sql for _, sql in harness.MICRO] + [
        "select lo_quantity, min(lo_revenue), max(lo_discount * 0.5) from lineorder group by lo_quantity",
        "select count(*), sum(lo_quantity*a_w) from xa, lineorder where a_w < 5 and lo_quantity < 10",
    ]
    for jit in jit_modes:
        e.set_option("jit", jit)
        for cfg in CONFIGS:
            for sql in sqls:
                e.run(sql, cfg)
        print(f"jit={jit}: {len(CONFIGS) * len(sqls)} queries", flush=True)
    # BASELINE shapes at a tiny scale (dense index, bitmaps, compaction drains)
    for db_name, keys in (("tpch", ("tpch_q6", "tpch_q1", "tpch_q3")), ("ssb", ("ssb_q11", "ssb_q41"))):
        e2 = Engine(0)
        harness.load_engine(e2, harness.bench_tables(db_name, 0.002, 42))
        for key in keys:
            for cfg in CONFIGS[:2]:
                e2.run(Q.BENCH[key][0], cfg)
        e2.close()
    # CSV ingest
    with tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False) as f:
        f.write('1,"a,b",1.5,x\n2,"q""q",2.5e-3,y\n3,c,7,x\n')
    e.load_csv(f.name, "csvt", [("k", INT64), ("s", STRING), ("p", FLOAT64), ("t", STRING)])
    os.unlink(f.name)
    print("done", flush=True)
    e.close()


if __name__ == "__main__":
    main()
