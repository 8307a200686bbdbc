"""Variant exploration of one BASELINE query on the B200:
Algorithm 1 (learn_variant_configuration) and the full aggregation-variant
space of the terminal pipeline (896 configurations, enumerate_variant_space),
each measured with CUDA events (median of 3, pruned above 1 s).

  python tools/sweep_space.py <query> [sf] [--full] > profiles/sweep_<query>.jsonl
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1709_00700_b200 import Engine  # noqa: E402
from paper_1709_00700_b200 import queries as Q  # noqa: E402

q = sys.argv[1]
sf = float(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else bench.DEFAULT_SF[q]
full = "--full" in sys.argv
e = Engine(0)
e.set_option("jit", 1)
bench.load_tables(e, q, sf, 42, 0, 1)
sql = Q.BENCH[q][0]
proj = bench.DEFAULT_CONFIG[q].split(";")[0]

t0 = time.time()
learned = e.learn([sql], q=3, prune_ms=1000.0, reps=3)
print(json.dumps({"query": q, "sf": sf, "kind": "learned (Algorithm 1)", **learned,
                  "seconds": time.time() - t0}), flush=True)
if full:
    term = e.pipeline_count(sql) - 1
    n, _ = e.space_size(sql, term)
    t0 = time.time()
    rows = []
    for i in range(n):
        agg = e.space_config(sql, term, i)
        cfg = proj + ";" + agg
        try:
            ms = e.measure([sql], cfg, prune_ms=1000.0, reps=3)
        except Exception as ex:  # noqa: BLE001
            ms = float("inf")
            print(json.dumps({"config": cfg, "error": str(ex)[:200]}), flush=True)
        rows.append((ms, cfg))
        print(json.dumps({"i": i, "config": cfg, "ms": ms}), flush=True)
    rows.sort()
    print(json.dumps({"query": q, "sf": sf, "kind": "full exploration", "space": n,
                      "seconds": time.time() - t0, "best": rows[:10],
                      "worst_finite": [r for r in rows if r[0] != float("inf")][-3:],
                      "learned_ms": learned["ms"]}), flush=True)
