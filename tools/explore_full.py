"""Full exploration of the 896 aggregation variants of one BASELINE query's
terminal pipeline on a B200, projection fixed to the learned
configuration; CSV with every configuration's time and, for every +inf, why
(pruned > 1 s, or the error class: CapacityExceeded, DuplicateKey, ...).
  python tools/explore_full.py <query> [sf] [jit] -> profiles/explore_r02_<query>.csv"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1709_00700_b200 import Engine  # noqa: E402
from paper_1709_00700_b200 import queries as Q  # noqa: E402

q = sys.argv[1]
sf = float(sys.argv[2]) if len(sys.argv) > 2 else bench.BASELINE_SF[q]
jit = int(sys.argv[3]) if len(sys.argv) > 3 else 0
e = Engine(0)
e.set_option("jit", jit)
bench.load_tables(e, q, sf, 42, 0, 1)
t0 = time.time()
out = os.path.join(ROOT, "profiles", f"explore_r02_{q}.csv")
r = e.explore([Q.BENCH[q][0]], "aggregation", fixed=bench.default_config(q).split(";")[0] + ";",
              reps=1, csv_path=out)
rows = open(out).read().splitlines()[1:]
status = {}
for row in rows:
    st = row.split(",")[4]
    status[st] = status.get(st, 0) + 1
print(json.dumps({**r, "query": q, "sf": sf, "jit": jit, "seconds": time.time() - t0, "status": status}))
