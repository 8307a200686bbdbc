"""Benchmark: input tuples/s and HBM roofline fraction of a BASELINE query on
1..8 B200s (BASELINE.json metric), beside the reference's CPU path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--query tpch_q1] [--sf 10]
                  [--config "<proj>;<agg>"] [--impl ours|reference]

One step = one execution of every pipeline of the query over the resident
synthetic tables (fact table row-sharded over ranks, weak scaling: each rank
holds an SF-sized shard of an N*SF table). Printed: one JSON line (rank 0).
Default workload: TPC-H Q1 at SF10 (BASELINE.json configs[1]).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "input tuples/sec & HBM GB/s (roofline frac) per TPC-H/SSB query, 1/2/4/8 B200"

# learned/selected variant per query (--config overrides)
DEFAULT_CONFIG = {
    "tpch_q6": "single_pass/sequential/branched/u=2;global_hash/sequential/branched/linear_probing/multiply_shift/wg=256/u=2",
    "tpch_q1": "single_pass/coalesced/branched;local_hash/coalesced/predicated/linear_probing/murmur/wg=256/ht=8",
    "ssb_q11": "single_pass/coalesced/branched/u=4;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=64",
    "ssb_q41": "single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256",
    "tpch_q3": "single_pass/coalesced/branched/u=4;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=64",
}
DEFAULT_SF = {"tpch_q6": 1.0, "tpch_q1": 10.0, "ssb_q11": 10.0, "ssb_q41": 10.0, "tpch_q3": 10.0}
WORKLOAD_NAME = {"tpch_q6": "TPC-H Q6", "tpch_q1": "TPC-H Q1", "ssb_q11": "SSB Q1.1",
                 "ssb_q41": "SSB Q4.1", "tpch_q3": "TPC-H Q3"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--query", default="tpch_q1", choices=sorted(DEFAULT_CONFIG))
    ap.add_argument("--sf", type=float, default=None)
    ap.add_argument("--config", default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-rows", type=int, default=4_000_000)
    ap.add_argument("--prefetch", type=int, default=None, help="TMA pipeline depth (pass tiles)")
    ap.add_argument("--stage", type=int, default=0,
                    help="1: TMA-staged pass tiles (coalesced); 0: coalesced 128-bit loads from HBM")
    ap.add_argument("--min-ctas", type=int, default=None,
                    help="compiled programs: __launch_bounds__ minimum CTAs per SM")
    ap.add_argument("--compact", type=int, default=None,
                    help="compiled, branched: compact live rows after the first probe (1) or not (0)")
    ap.add_argument("--pass-sync", type=int, default=None,
                    help="unstaged coalesced tiles: CTA barrier after every pass (1) or not (0)")
    ap.add_argument("--l2-distance", type=int, default=None,
                    help="unstaged coalesced tiles: L2 bulk-prefetch distance (passes, 0 = off)")
    ap.add_argument("--jit", type=int, default=1,
                    help="1: compiled programs (NVRTC), 0: the AOT interpreter instantiations")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="exchange backend for N>1 (gloo: host-side exchange, for checking the "
                         "multi-rank path when fewer GPUs than ranks are visible)")
    ap.add_argument("--sweep", nargs="*", default=None,
                    help="time each given config (or a built-in list) and print one line per config")
    return ap.parse_args()


SWEEP = [
    "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=1",
    "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=4",
    "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=128/ht=8",
    "single_pass/sequential/branched;local_hash/sequential/branched/linear_probing/murmur/wg=256/ht=4",
    "single_pass/coalesced/branched;global_hash/coalesced/predicated/linear_probing/murmur/wg=256",
    "single_pass/coalesced/predicated;local_hash/coalesced/predicated/linear_probing/murmur/wg=256/ht=1",
    "single_pass/sequential/branched;local_hash/sequential/branched/linear_probing/murmur/wg=256/ht=1",
    "multi_pass/coalesced/branched/tm=1024;local_hash/coalesced/branched/linear_probing/murmur/wg=512/ht=1",
    "single_pass/coalesced/branched/u=2;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=1/u=2",
    "single_pass/coalesced/branched/u=4;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=1/u=4",
    "single_pass/coalesced/branched;local_hash/coalesced/branched/cuckoo/murmur/wg=256/ht=1",
    "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/ht=8",
    "single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/murmur/wg=256",
    "single_pass/coalesced/branched;global_hash/coalesced/branched/cuckoo/murmur/wg=1024",
    "multi_pass/coalesced/branched/tm=16384;local_hash/coalesced/branched/linear_probing/murmur/wg=1024/ht=1",
]


def run_sweep(args):
    import torch
    from paper_1709_00700_b200 import Engine
    from paper_1709_00700_b200 import queries as Q
    query = args.query
    sf = args.sf or DEFAULT_SF[query]
    engine = Engine(0)
    if args.prefetch is not None:
        engine.set_option("prefetch_passes", args.prefetch)
    engine.set_option("jit", args.jit)
    engine.set_option("stage", args.stage)
    if args.l2_distance is not None:
        engine.set_option("l2_distance", args.l2_distance)
    if args.pass_sync is not None:
        engine.set_option("pass_sync", args.pass_sync)
    if args.compact is not None:
        engine.set_option("compact", args.compact)
    if args.min_ctas is not None:
        engine.set_option("min_ctas", args.min_ctas)
    load_tables(engine, query, sf, args.seed, 0, 1)
    sql = Q.BENCH[query][0]
    for cfg in (args.sweep or SWEEP):
        try:
            for _ in range(2):
                engine.run(sql, cfg)
            ks, ws = [], []
            for _ in range(5):
                r = engine.run(sql, cfg)
                ks.append(r.kernel_ms)
                ws.append(r.wall_ms)
            print(json.dumps({"query": query, "sf": sf, "config": cfg, "kernel_ms": min(ks),
                              "wall_ms": min(ws), "pipelines": r.pipelines}), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"query": query, "config": cfg, "error": str(e)}), flush=True)
    engine.close()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def keep_busy(self, step, n: int = 3, max_s: float = 5.0):
        """Short timed regions end before nvidia-smi answers: keep running the
        same (untimed) step until n samples were taken under this load."""
        t0 = time.perf_counter()
        while self._proc and len(self.samples) < n and time.perf_counter() - t0 < max_s:
            step()

    def __exit__(self, *exc):
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=2)
            except Exception:
                self._proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[3:7]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def algorithmic_bytes(query: str, fact_rows: int, dims: dict) -> int:
    """scanned rows x referenced columns x 8 B (+ build inserts
    x 16 B); dimension tables <= L2 count their scan only."""
    from paper_1709_00700_b200 import queries as Q
    b = fact_rows * len(Q.FACT_COLUMNS[query]) * 8
    for rows, cols in dims.values():
        b += rows * cols * 8
    return b


def dims_for(query: str, sf: float) -> dict:
    from paper_1709_00700_b200 import datagen as dg
    if query == "ssb_q11":
        return {"ddate": (dg.table_rows(dg.DDATE, sf), 2)}
    if query == "ssb_q41":
        return {"ddate": (dg.table_rows(dg.DDATE, sf), 2),
                "customer": (dg.table_rows(dg.SCUSTOMER, sf), 2),
                "supplier": (dg.table_rows(dg.SUPPLIER, sf), 2),
                "part": (dg.table_rows(dg.PART, sf), 2)}
    if query == "tpch_q3":
        return {"orders": (dg.table_rows(dg.ORDERS, sf), 4), "customer": (dg.table_rows(dg.CUSTOMER, sf), 2)}
    return {}


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own reference_execute (oracle/_ref, 1 thread)
# on a bounded sample, and our multi-threaded restatement (oracle/port)
# ---------------------------------------------------------------------------

def cpu_reference_sample(query: str, sf: float, seed: int, sample_rows: int, reps: int = 1):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bridge import OraDb, OraTable
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200 import queries as Q
    sql, tables, fact = Q.BENCH[query]
    db = OraDb()
    n_fact = 0
    for t in tables:
        rows = dg.table_rows(t, sf)
        if t == fact:
            rows = min(rows, sample_rows)
            n_fact = rows
        name, cols = dg.host_table(t, sf, seed, 0, rows)
        db.add(OraTable.from_columns(name, cols))
    times = []
    for _ in range(max(1, reps)):
        t0 = time.perf_counter()
        db.execute(sql)
        times.append(time.perf_counter() - t0)
    return n_fact, times


def cpu_port(query: str, sf: float, seed: int, threads: int):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_oracle import _port_inputs
    from oracle_bridge import port_run
    q, cols, n, dims, codes = _port_inputs(query, sf, seed)
    t0 = time.perf_counter()
    port_run(q, cols, n, dims, codes, threads, out_rows=max(1024, n // 2))
    return n, time.perf_counter() - t0


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    sf = args.sf or DEFAULT_SF[args.query]
    sample = args.cpu_sample_rows
    n_fact, _ = cpu_reference_sample(args.query, sf, args.seed, sample, reps=0 or 1)
    times = []
    for i in range(args.warmup + args.steps):
        _, t = cpu_reference_sample(args.query, sf, args.seed, sample, reps=1)
        if i >= args.warmup:
            times.append(t[0])
    ms = statistics.mean(times) * 1e3
    value = n_fact / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"{WORKLOAD_NAME[args.query]} SF{sf:g}", "query": args.query, "sf": sf,
                   "sample_fact_rows": n_fact},
        "cpu_baseline": {"value": value, "unit": "tuples/s", "cores": 1, "kind": "reference",
                         "sample": f"reference_execute (oracle/_ref, unmodified reference sources) over the "
                                   f"first {n_fact} fact rows of the SF{sf:g} workload per step"},
        "e2e": {"value": value, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def load_tables(engine, query: str, sf: float, seed: int, rank: int, world: int):
    """Generates the query's tables in HBM: the fact table as this rank's shard
    of an (world x sf) table, dimensions replicated."""
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200 import queries as Q
    _, tables, fact = Q.BENCH[query]
    global_sf = sf * world
    per = dg.table_rows(fact, sf)
    for t in tables:
        if t == fact:
            engine.generate(t, global_sf, seed, rank * per, per)
        else:
            engine.generate(t, global_sf, seed)
    return per


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.sweep is not None:
        run_sweep(args)
        return
    rank, world, local = dist_env()
    import torch
    if world > 1:
        import torch.distributed as dist
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    from paper_1709_00700_b200 import Engine, _native
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200 import queries as Q
    from paper_1709_00700_b200.distributed import all_gather_rows

    query = args.query
    sf = args.sf or DEFAULT_SF[query]
    cfg = args.config or DEFAULT_CONFIG[query]
    sql = Q.BENCH[query][0]
    engine = Engine(local)
    engine.set_option("jit", args.jit)
    engine.set_option("stage", args.stage)
    if args.l2_distance is not None:
        engine.set_option("l2_distance", args.l2_distance)
    if args.pass_sync is not None:
        engine.set_option("pass_sync", args.pass_sync)
    if args.compact is not None:
        engine.set_option("compact", args.compact)
    if args.min_ctas is not None:
        engine.set_option("min_ctas", args.min_ctas)
    per_rank = load_tables(engine, query, sf, args.seed, rank, world)
    lib = _native.b200()
    stream = torch.cuda.ExternalStream(lib.hawk_b200_ctx_stream(engine.ctx), device=torch.device("cuda", local))
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    dims = dims_for(query, sf * world)
    alg_bytes = algorithmic_bytes(query, per_rank, dims)
    flush = alg_bytes < 4 * l2

    xdev = torch.device("cuda", local) if args.backend == "nccl" else torch.device("cpu")

    def step():
        """One query: (result, kernels launched). N>1: shard partials, NCCL
        all-gather of the partial rows, device merge + finalise."""
        if world == 1:
            r = engine.run(sql, cfg)
            return r, r.launches
        part = engine.run_partial(sql, cfg)
        gathered = all_gather_rows(part.rows, device=xdev)
        r = engine.finalize(sql, gathered, cfg)
        return r, part.launches + r.launches

    for _ in range(args.warmup):
        if flush:
            engine.flush_l2()
        r, _ = step()
    kernel_ms, launches = [], 0
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    total_ms = 0.0
    with Clocks(local) as clocks:
        for _ in range(args.steps):
            if flush:
                engine.flush_l2()
            start.record(stream)
            r, n_launch = step()
            end.record(stream)
            end.synchronize()
            total_ms += start.elapsed_time(end)
            kernel_ms.append(r.kernel_ms if world == 1 else 0.0)
            launches += n_launch
        if world == 1:
            clocks.keep_busy(step)
        else:  # every rank runs the same number of extra (untimed) steps, ~0.4 s
            t = torch.tensor([total_ms / args.steps], device=xdev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            for _ in range(min(20000, int(400.0 / max(float(t.item()), 1e-3)) + 1)):
                step()
    torch.cuda.synchronize()
    if world > 1:
        t = torch.tensor([total_ms], device=xdev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = per_rank * world / (ms_per_step / 1e3)

    # dominant kernel = the terminal pipeline's kernels (event-timed on the engine stream)
    term = r.pipelines[-1] if r.pipelines else {"kernel_ms": 0.0}
    peak, peak_kind = measured_peak()
    term_ms = statistics.mean([p for p in kernel_ms]) if world == 1 else float("nan")
    build_ms = sum(p["kernel_ms"] for p in r.pipelines[:-1]) if r.pipelines else 0.0
    term_only_ms = max(1e-9, (term_ms - build_ms)) if world == 1 else float("nan")
    fact_bytes = per_rank * len(Q.FACT_COLUMNS[query]) * 8
    achieved = fact_bytes / (term_only_ms / 1e3) / 1e9 if world == 1 else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(query)
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"{WORKLOAD_NAME[query]} SF{sf:g}" + (f" per GPU (x{world})" if world > 1 else ""),
                   "query": query, "sf_per_gpu": sf, "fact_rows_per_gpu": per_rank, "variant": cfg,
                   "l2": ("flushed between steps" if flush else
                          f"inputs larger than L2 ({alg_bytes / 1e9:.2f} GB vs {l2 / 1e6:.0f} MB)"),
                   "parallelism": f"dp{world} (fact rows sharded, dimensions replicated)"},
        "hbm_gbs": alg_bytes / (ms_per_step / 1e3) / 1e9,
        "gpu_launches": launches,
    }
    if world == 1:
        line["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                            "frac": achieved / peak, "traffic": traffic,
                            "kernel": "terminal pipeline (pipeline_kernel) of " + WORKLOAD_NAME[query],
                            "algorithmic_bytes_per_launch": fact_bytes,
                            "kernel_ms": term_only_ms, "peak_kind": peak_kind}
    line["clocks"] = clocks.summary()

    if not args.no_e2e:
        line["e2e"] = e2e_measure(engine, query, sf, args, step, rank, world, per_rank)
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        n_fact, times = cpu_reference_sample(query, sf, args.seed, args.cpu_sample_rows, reps=1)
        ref_rate = n_fact / times[0]
        threads = os.cpu_count() or 1
        pn, pt = cpu_port(query, sf, args.seed, threads)
        line["cpu_baseline"] = {
            "value": ref_rate, "unit": "tuples/s", "cores": 1, "kind": "reference",
            "sample": f"reference_execute (unmodified reference sources, oracle/_ref) over the first "
                      f"{n_fact} fact rows of {WORKLOAD_NAME[query]} SF{sf:g}; single-threaded by design "
                      f"(SPEC.md:179)"}
        line["cpu_port"] = {"value": pn / pt, "unit": "tuples/s", "cores": threads, "kind": "port",
                            "sample": f"oracle/port restatement over all {pn} fact rows, {threads} threads"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    engine.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def e2e_measure(engine, query, sf, args, step, rank, world, per_rank):
    """Same metric through the engine's C ABI with HOST inputs: each step copies
    this rank's fact-table shard (the referenced columns) from pinned host
    memory into HBM (hawk_engine_put_columns), runs the query (N>1: partials,
    NCCL all-gather, merge) and reads the result back (D2H). Timed per step as
    the max over ranks."""
    import ctypes as C

    import numpy as np
    import torch
    from paper_1709_00700_b200 import _native
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200 import queries as Q
    from paper_1709_00700_b200.engine import INT64, Column
    lib = _native.b200()
    _, _, fact = Q.BENCH[query]
    name, schema = dg.SCHEMA[fact]
    global_sf = sf * world
    n = per_rank
    wanted = Q.FACT_COLUMNS[query]
    host, pinned, domains = [], [], []
    for ci, (cname, lex) in enumerate(schema):
        if cname not in wanted:
            continue
        domains.append(lib.hawk_b200_gen_column_domain(fact, ci, global_sf))
        p = C.c_void_p()
        assert lib.hawk_b200_host_alloc(n * 8, C.byref(p)) == 0
        pinned.append(p)
        arr = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_int64)), shape=(n,))
        arr[:] = dg.gen_column(fact, ci, global_sf, args.seed, rank * n, n)
        host.append(Column(cname, INT64 if lex is None else 2, arr, None if lex is None else lex))
    engine.drop(name)
    times, h2d, d2h = [], sum(c.values.nbytes for c in host), 0
    for i in range(args.warmup + args.steps):
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        engine.put_table(name, host, distinct=domains, row_offset=rank * n)
        r, _ = step()
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
        d2h = sum(c.values.nbytes for c in r.columns)
    for p in pinned:
        lib.hawk_b200_host_free(p)
    ms = statistics.mean(times) * 1e3
    if world > 1:
        t = torch.tensor([ms], device="cuda" if torch.distributed.get_backend() == "nccl" else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": n * world / (ms / 1e3), "unit": "tuples/s", "h2d_bytes_per_step": h2d * world,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms,
            "path": "hawk_engine_put_columns (pinned host -> HBM) + hawk_engine_run (C ABI)"
                    + (" / run_partial + NCCL all-gather + finalize" if world > 1 else "")}


if __name__ == "__main__":
    main()
