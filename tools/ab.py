"""A/B of engine options on one BASELINE query (run on a B200 under gpurun):
  python tools/ab.py ssb_q41 100 "dense_join=0" "dense_join=1,drain_rows=1" ...
Each option set: whole-query ms/step and terminal-kernel ms (CUDA events, L2
flushed or inputs > L2), 2 repetitions of --steps 10 after 3 warm-ups.
Prints one JSON line per (option set, repetition)."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import bench  # noqa: E402
from paper_1709_00700_b200 import Engine, _native  # noqa: E402
from paper_1709_00700_b200 import queries as Q  # noqa: E402


def main():
    query, sf = sys.argv[1], float(sys.argv[2])
    sets = sys.argv[3:] or [""]
    cfg = os.environ.get("AB_CONFIG") or bench.default_config(query)
    import torch
    e = Engine(0)
    e.set_option("jit", 1)
    bench.load_tables(e, query, sf, 42, 0, 1)
    stream = torch.cuda.ExternalStream(_native.b200().hawk_b200_ctx_stream(e.ctx), device=torch.device("cuda", 0))
    sql = os.environ.get("AB_SQL") or Q.BENCH[query][0]
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    flush = dg_bytes(query, sf) < 4 * l2
    for rep in range(2):
        for opts in sets:
            defaults = {}
            for kv in filter(None, opts.split(",")):
                k, v = kv.split("=")
                defaults[k] = int(v)
                e.set_option(k, int(v))
            try:
                total, outs = bench.timed_steps(e, stream, lambda: e.run(sql, cfg), 10, 3, flush)
                term = statistics.mean(r.pipelines[-1]["kernel_ms"] for r in outs)
                kern = statistics.mean(r.kernel_ms for r in outs)
                fact = Q.FACT_COLUMNS[query]
                per = e.table_rows(bench_fact_name(query))
                frac = per * len(fact) * 8 / term / 1e6 / bench.measured_peak()[0]
                print(json.dumps({"query": query, "sf": sf, "opts": opts, "config": cfg, "rep": rep, "ms_per_step": total / 10,
                                  "kernels_ms": kern, "terminal_ms": term, "terminal_frac": frac,
                                  "pipelines": [round(p["kernel_ms"], 4) for p in outs[-1].pipelines]}), flush=True)
            except Exception as ex:  # noqa: BLE001
                print(json.dumps({"query": query, "opts": opts, "error": str(ex)}), flush=True)
            # restore the defaults of this set's keys
            for k in defaults:
                e.set_option(k, DEFAULTS.get(k, 1))
    e.close()


DEFAULTS = {"dense_join": 1, "drain_rows": 0, "split_bits": 1, "compact": 1, "dense_keys": 1,
            "priv_groups": -1, "min_ctas": 0, "stage": 0, "pass_sync": 0, "l2_distance": 0, "jit": 1}


def bench_fact_name(query):
    from paper_1709_00700_b200 import datagen as dg
    return dg.SCHEMA[Q.BENCH[query][2]][0]


def dg_bytes(query, sf):
    from paper_1709_00700_b200 import datagen as dg
    return dg.table_rows(Q.BENCH[query][2], sf) * len(Q.FACT_COLUMNS[query]) * 8


if __name__ == "__main__":
    main()
