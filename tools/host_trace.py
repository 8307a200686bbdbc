"""Per-phase host/device time of one query run (HAWK_TRACE=1): python tools/host_trace.py q [sf]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1709_00700_b200 import Engine  # noqa: E402
from paper_1709_00700_b200 import queries as Q  # noqa: E402

q = sys.argv[1]
sf = float(sys.argv[2]) if len(sys.argv) > 2 else bench.DEFAULT_SF[q]
e = Engine(0)
e.set_option("jit", 1)
bench.load_tables(e, q, sf, 42, 0, 1)
sql, cfg = Q.BENCH[q][0], bench.DEFAULT_CONFIG[q]
for i in range(4):
    if i == 3:
        os.environ["HAWK_TRACE"] = "1"
    t0 = time.perf_counter()
    r = e.run(sql, cfg)
    dt = (time.perf_counter() - t0) * 1e3
    print(f"{q} run {i}: wall {dt:.3f} ms  engine wall {r.wall_ms:.3f}  kernel {r.kernel_ms:.3f}", file=sys.stderr)
