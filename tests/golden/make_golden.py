"""Generates the golden fixtures by running the REFERENCE oracle
(reference_execute, /root/reference/proj/src/planner_reference.cpp:331, built
unmodified into oracle/_ref/libhawk_oracle.so).

  known_answers.json  SURVEY.md Appendix B micro-benchmarks on gen_lineorder
  bench_sf0.01.json   the five BASELINE queries on synthetic TPC-H/SSB, SF 0.01

Run from the repo root:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import struct
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import harness  # noqa: E402


def encode_rows(table) -> list[list]:
    rows = []
    for row in table.canonical_rows():
        enc = []
        for v in row:
            if isinstance(v, float):
                enc.append({"f64": struct.unpack("<q", struct.pack("<d", v))[0]})
            else:
                enc.append(v)
        rows.append(enc)
    return rows


def main():
    known = []
    for n, seed in [(10000, 7), (100000, 42)]:
        db = harness.oracle_db(harness.micro_tables(n, seed))
        for name, sql in harness.MICRO:
            r = db.execute(sql)
            known.append({"query": name, "sql": sql, "n": n, "seed": seed, "rows": r.rows,
                          "checksum": f"{r.checksum():016x}",
                          "result": encode_rows(r) if r.rows <= 64 else None})
    with open(os.path.join(HERE, "known_answers.json"), "w") as f:
        json.dump(known, f, indent=1)

    bench = []
    for key, sql in harness.BENCH:
        db_name = "ssb" if key.startswith("ssb") else "tpch"
        db = harness.oracle_db(harness.bench_tables(db_name, 0.01, 42))
        r = db.execute(sql)
        bench.append({"query": key, "sql": sql, "sf": 0.01, "seed": 42, "rows": r.rows,
                      "checksum": f"{r.checksum():016x}", "result": encode_rows(r)})
    with open(os.path.join(HERE, "bench_sf0.01.json"), "w") as f:
        json.dump(bench, f, indent=1)
    print(f"wrote {len(known)} known answers, {len(bench)} bench fixtures")


if __name__ == "__main__":
    main()
