"""Host-side cost of one query call (run on a B200 under gpurun):
  python tools/host_overhead.py tpch_q6 1
Times engine.run back to back without L2 flushes: wall clock per call
(time.perf_counter), device time per call (CUDA events on the engine's
stream), and the C++ engine's own wall time (metrics), so the Python /
ctypes share, the engine's host share and the device share separate."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import bench  # noqa: E402
from paper_1709_00700_b200 import Engine, _native  # noqa: E402
from paper_1709_00700_b200 import queries as Q  # noqa: E402


def main():
    import torch
    query, sf = sys.argv[1], float(sys.argv[2])
    cfg = os.environ.get("AB_CONFIG") or bench.default_config(query)
    e = Engine(0)
    e.set_option("jit", 1)
    bench.load_tables(e, query, sf, 42, 0, 1)
    stream = torch.cuda.ExternalStream(_native.b200().hawk_b200_ctx_stream(e.ctx), device=torch.device("cuda", 0))
    sql = Q.BENCH[query][0]
    for _ in range(20):
        e.run(sql, cfg)
    torch.cuda.synchronize()
    walls, devs, engine_ms, kernels = [], [], [], []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(200):
        a.record(stream)
        t0 = time.perf_counter()
        r = e.run(sql, cfg)
        t1 = time.perf_counter()
        b.record(stream)
        b.synchronize()
        walls.append((t1 - t0) * 1e3)
        devs.append(a.elapsed_time(b))
        engine_ms.append(r.wall_ms)
        kernels.append(r.kernel_ms)
        del r
    med = statistics.median
    print(json.dumps({"query": query, "sf": sf, "config": cfg, "calls": 200,
                      "python_call_ms": med(walls), "engine_wall_ms": med(engine_ms),
                      "events_ms": med(devs), "kernels_ms": med(kernels)}))
    e.close()


if __name__ == "__main__":
    main()
