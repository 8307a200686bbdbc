"""Benchmark: input tuples/s and HBM roofline fraction of the BASELINE queries
on 1..8 B200s (BASELINE.json metric), beside the reference's CPU path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--query tpch_q1] [--sf 10]
                  [--config "<proj>;<agg>"] [--impl ours|reference] [--no-per-query]

One step = one execution of every pipeline of the query over the resident
synthetic tables (fact table row-sharded over ranks, weak scaling: each rank
holds an SF-sized shard of an N*SF table). Printed: one JSON line (rank 0).
Headline workload: TPC-H Q1 at SF10 (BASELINE.json configs[1]); at N=1 the
line also carries a `per_query` block with every BASELINE configuration at
its own scale factor (Q6 SF1, Q1 SF10, SSB Q1.1 SF10, SSB Q4.1 SF100,
TPC-H Q3 SF100).

--impl reference: the reference's own CPU path (reference_execute, compiled
unmodified into oracle/_ref) over the same whole workload on every host core
(tests/ref_sharded.py), rank 0 only.
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

# the variant per query: the configuration Algorithm 1 learned on a B200
# (tools/learn_all.py -> paper_1709_00700_b200/learned/<query>.conf); these
# literals are only the fallback when no learned file exists (--config overrides)
DEFAULT_CONFIG = {
    "tpch_q6": "single_pass/sequential/branched/u=2;global_hash/sequential/branched/linear_probing/multiply_shift/wg=256/u=2",
    "tpch_q1": "single_pass/coalesced/branched;local_hash/coalesced/predicated/linear_probing/murmur/wg=256/ht=8",
    "ssb_q11": "single_pass/coalesced/branched/u=4;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=64",
    "ssb_q41": "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/ht=8",
    "tpch_q3": "single_pass/coalesced/branched/u=4;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=64",
}
# BASELINE.json configs: the scale factor each query is quoted at
BASELINE_SF = {"tpch_q6": 1.0, "tpch_q1": 10.0, "ssb_q11": 10.0, "ssb_q41": 100.0, "tpch_q3": 100.0}
DEFAULT_SF = BASELINE_SF


def default_config(query: str) -> str:
    """The learned configuration of `query` (key-value file), else the fallback."""
    path = os.path.join(ROOT, "paper_1709_00700_b200", "learned", f"{query}.conf")
    if os.path.exists(path):
        from paper_1709_00700_b200.engine import load_config
        return load_config(path)
    return DEFAULT_CONFIG[query]


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
    ap.add_argument("--no-per-query", action="store_true",
                    help="N=1: skip the per_query block (every BASELINE configuration)")
    ap.add_argument("--per-query-steps", type=int, default=10)
    ap.add_argument("--prefetch", type=int, default=None, help="TMA pipeline depth (pass tiles)")
    ap.add_argument("--stage", type=int, default=None,
                    help="1: TMA-staged pass tiles (coalesced); 0: coalesced loads from HBM")
    ap.add_argument("--min-ctas", type=int, default=None,
                    help="compiled programs: __launch_bounds__ minimum CTAs per SM")
    ap.add_argument("--compact", type=int, default=None,
                    help="compiled, branched: compact live rows after the first probe (1) or not (0)")
    ap.add_argument("--pass-sync", type=int, default=None,
                    help="unstaged coalesced tiles: CTA barrier after every pass (1) or not (0)")
    ap.add_argument("--l2-distance", type=int, default=None,
                    help="unstaged coalesced tiles: L2 bulk-prefetch distance (passes, 0 = off)")
    ap.add_argument("--option", action="append", default=[],
                    help="extra engine option name=value (hawk_b200_ctx_set_option)")
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
    "single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/murmur/wg=256",
    "single_pass/coalesced/branched;global_hash/coalesced/branched/cuckoo/murmur/wg=1024",
]


def apply_options(engine, args):
    engine.set_option("jit", args.jit)
    for name, val in (("prefetch_passes", args.prefetch), ("stage", args.stage),
                      ("l2_distance", args.l2_distance), ("pass_sync", args.pass_sync),
                      ("compact", args.compact), ("min_ctas", args.min_ctas)):
        if val is not None:
            engine.set_option(name, val)
    for o in args.option:
        k, v = o.split("=", 1)
        engine.set_option(k, int(v))


def run_sweep(args):
    from paper_1709_00700_b200 import Engine
    from paper_1709_00700_b200 import queries as Q
    query = args.query
    sf = args.sf or DEFAULT_SF[query]
    engine = Engine(0)
    apply_options(engine, args)
    load_tables(engine, query, sf, args.seed, 0, 1)
    sql = Q.BENCH[query][0]
    for cfg in (args.sweep or SWEEP):
        try:
            for _ in range(2):
                engine.run(sql, cfg)
            ks, ws = [], []
            for _ in range(5):
                engine.flush_l2()
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


def host_info() -> dict:
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from ref_sharded import cpu_model
    return {"cpu_model": cpu_model(), "cores": os.cpu_count() or 1}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
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


def workload_config(query: str, sf: float, world: int) -> dict:
    """The `config` object of both arms (same workload, same keys)."""
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200 import queries as Q
    fact = Q.BENCH[query][2]
    per = dg.table_rows(fact, sf)
    cfg = {"workload": f"{WORKLOAD_NAME[query]} SF{sf * world:g}", "query": query, "sf": sf * world,
           "fact_rows": per * world}
    if world > 1:
        cfg["parallelism"] = (f"dp{world} (fact rows sharded, SF{sf:g} per GPU"
                              + (", orders co-partitioned by orderkey)" if query == "tpch_q3" else ")"))
    return cfg


# ---------------------------------------------------------------------------
# algorithmic bytes from measured selectivities
# ---------------------------------------------------------------------------

# count queries giving the probe / update counts of each query's terminal
# pipeline (run untimed through the engine itself)
ACCOUNTING = {
    "tpch_q3": {
        "orders_probes": "select count(*) from lineitem where l_shipdate > 19950315",
        "customer_probes": "select count(*) from orders, lineitem where l_orderkey = o_orderkey "
                           "and o_orderdate < 19950315 and l_shipdate > 19950315",
        "group_updates": "select count(*) from orders, customer, lineitem where c_mktsegment = 'BUILDING' "
                         "and c_custkey = o_custkey and l_orderkey = o_orderkey and o_orderdate < 19950315 "
                         "and l_shipdate > 19950315",
    },
}


def query_bytes(engine, query: str, sf: float, per_rank: int, world: int, result, l2: int) -> dict:
    """scanned rows x referenced columns x 8 B, + build inserts
    x 16 B, + probes / group updates into tables larger than L2 x 32 B (a
    sector). `terminal` counts the fact columns the terminal kernel streams."""
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200 import queries as Q
    _, tables, fact = Q.BENCH[query]
    fact_bytes = per_rank * len(Q.FACT_COLUMNS[query]) * 8
    total = fact_bytes
    detail = {"fact_scan": fact_bytes}
    dim_cols = {dg.DDATE: 2, dg.SCUSTOMER: 3, dg.SUPPLIER: 2, dg.PART: 2, dg.ORDERS: 4, dg.CUSTOMER: 2}
    for t in tables:
        if t != fact:
            b = dg.table_rows(t, sf * world) * dim_cols[t] * 8
            detail[f"scan_{dg.SCHEMA[t][0]}"] = b
            total += b
    inserts = sum(p["rows_out"] for p in result.pipelines[:-1])
    detail["build_inserts"] = inserts * 16
    total += inserts * 16
    if query in ACCOUNTING and not os.environ.get("HAWK_BENCH_NO_ACCOUNTING"):
        big = {}
        # join tables are sized next_pow2(2 x build rows) x 16 B; the orders
        # table exceeds L2 at every SF >= 1, the customer table from SF ~60
        cap = lambda rows: 1 << max(4, (2 * rows - 1).bit_length())  # noqa: E731
        big["orders_probes"] = cap(dg.table_rows(dg.ORDERS, sf * world)) * 16 > l2
        big["customer_probes"] = cap(dg.table_rows(dg.CUSTOMER, sf * world)) * 16 > l2
        big["group_updates"] = True
        for k, sql in ACCOUNTING[query].items():
            n = int(engine.run(sql, default_config(query)).columns[0].values[0])
            detail[k] = n * 32 if big[k] else 0
            total += detail[k]
    return {"terminal": fact_bytes, "whole_query": total, "detail": detail}


# ---------------------------------------------------------------------------
# the reference arm: reference_execute over the whole workload on every core
# ---------------------------------------------------------------------------

def reference_sample_rows(query: str, sf: float, world: int) -> int | None:
    """Whole workload when its reference_execute working set (~300 B per fact
    row, measured) fits in half the host RAM, else a bounded sample."""
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200 import queries as Q
    rows = dg.table_rows(Q.BENCH[query][2], sf) * world
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 64 << 30
    cap = int(avail * 0.5 / 300)
    return None if rows <= cap and rows <= 120_000_000 else min(cap, 60_000_000)


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from ref_sharded import ShardedReference
    query = args.query
    sf = args.sf or DEFAULT_SF[query]
    sample = reference_sample_rows(query, sf, world)
    ref = ShardedReference(query, sf * world, args.seed, fact_rows=sample)
    times = []
    for i in range(args.warmup + args.steps):
        t = ref.timed(1)[0]
        if i >= args.warmup:
            times.append(t)
    ms = statistics.mean(times) * 1e3
    value = ref.fact_rows / (ms / 1e3)
    info = host_info()
    cfg = workload_config(query, sf, world)
    if sample is not None:
        cfg = dict(cfg, fact_rows=ref.fact_rows, sample="first rows of the fact table (host RAM bound)")
    desc = (f"reference_execute (unmodified reference sources, oracle/_ref) over {ref.fact_rows} fact rows "
            f"of {cfg['workload']}, one row shard per host thread ({ref.shards} shards, "
            f"{ref.threads} threads), shard results merged (SUM/COUNT add, AVG = SUM/COUNT)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "tuples/s", "cores": ref.threads, "kind": "reference",
                         "sample": desc, "cpu_model": info["cpu_model"], "host_cores": info["cores"],
                         "table_build_s": ref.build_s},
        "e2e": {"value": value, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def load_tables(engine, query: str, sf: float, seed: int, rank: int, world: int):
    """Generates the query's tables in HBM: the fact table as this rank's shard
    of an (world x sf) table, dimensions replicated — except TPC-H orders,
    which is co-partitioned with lineitem by orderkey range
    (distributed.copartition_range), so Q3's orders build scales as 1/N."""
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200 import queries as Q
    from paper_1709_00700_b200.distributed import copartition_range
    _, tables, fact = Q.BENCH[query]
    global_sf = sf * world
    per = dg.table_rows(fact, sf)
    for t in tables:
        if t == fact:
            engine.generate(t, global_sf, seed, rank * per, per)
        elif fact == dg.LINEITEM and t == dg.ORDERS and world > 1:
            b, e = copartition_range(rank * per, (rank + 1) * per)
            engine.generate(t, global_sf, seed, b, e - b)
        else:
            engine.generate(t, global_sf, seed)
    return per


def drop_tables(engine, query: str):
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200 import queries as Q
    for t in Q.BENCH[query][1]:
        name = dg.SCHEMA[t][0]
        if engine.table_rows(name) >= 0:
            engine.drop(name)


class StepInfo:
    """What a timed step keeps of its result: the metrics only (holding every
    Result alive would make each step allocate fresh host pages)."""

    def __init__(self, r, launches=None):
        self.kernel_ms = r.kernel_ms
        self.pipelines = r.pipelines
        self.launches = r.launches if launches is None else launches
        self.rows = r.rows


def timed_steps(engine, stream, step, steps, warmup, flush, clocks=None, world=1):
    """W untimed steps, then K steps each bracketed by CUDA events on the
    engine's stream. Returns (total ms, per-step StepInfo)."""
    import torch
    for _ in range(warmup):
        if flush:
            engine.flush_l2()
        step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    total_ms, outs = 0.0, []
    for _ in range(steps):
        if flush:
            engine.flush_l2()
        start.record(stream)
        r = step()
        end.record(stream)
        outs.append(StepInfo(*r) if isinstance(r, tuple) else StepInfo(r))
        del r
        end.synchronize()
        total_ms += start.elapsed_time(end)
    torch.cuda.synchronize()
    return total_ms, outs


def ncu_traffic(query: str, sf: float):
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(prof)).get(f"{query}@sf{sf:g}")
    except Exception:
        return None


def measure_query(engine, stream, query, sf, cfg, steps, warmup, l2, peak):
    """One BASELINE configuration at N=1: whole-query and terminal-kernel
    throughput with both roofline fractions (per_query block)."""
    from paper_1709_00700_b200 import datagen as dg
    from paper_1709_00700_b200 import queries as Q
    sql, tables, fact = Q.BENCH[query]
    per = load_tables(engine, query, sf, 42, 0, 1)
    input_tuples = sum(dg.table_rows(t, sf) for t in tables)
    r0 = engine.run(sql, cfg)
    acct = query_bytes(engine, query, sf, per, 1, r0, l2)
    flush = acct["whole_query"] < 4 * l2
    total_ms, outs = timed_steps(engine, stream, lambda: engine.run(sql, cfg), steps, warmup, flush)
    ms = total_ms / steps
    term_ms = statistics.mean(r.pipelines[-1]["kernel_ms"] for r in outs)
    kern_ms = statistics.mean(r.kernel_ms for r in outs)
    out = {
        "workload": f"{WORKLOAD_NAME[query]} SF{sf:g}", "variant": cfg, "fact_rows": per,
        "input_tuples": input_tuples, "value": input_tuples / (ms / 1e3), "unit": "tuples/s",
        "fact_tuples_per_s": per / (ms / 1e3), "ms_per_step": ms, "kernels_ms": kern_ms,
        "terminal_ms": term_ms, "steps": steps, "warmup": warmup,
        "l2": "flushed between steps" if flush else "inputs larger than L2",
        "roofline": {
            "bound": "hbm", "peak": peak, "unit": "GB/s",
            "terminal": {"bytes": acct["terminal"], "achieved": acct["terminal"] / term_ms / 1e6,
                         "frac": acct["terminal"] / term_ms / 1e6 / peak},
            "whole_query": {"bytes": acct["whole_query"], "achieved": acct["whole_query"] / ms / 1e6,
                            "frac": acct["whole_query"] / ms / 1e6 / peak, "detail": acct["detail"]},
            "traffic": ncu_traffic(query, sf),
        },
        "pipelines": [{k: p[k] for k in ("kernel_ms", "rows_in", "rows_out", "grid", "block")}
                      for p in outs[-1].pipelines],
    }
    drop_tables(engine, query)
    return out


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
    from paper_1709_00700_b200 import queries as Q
    from paper_1709_00700_b200.distributed import all_gather_rows

    query = args.query
    sf = args.sf or DEFAULT_SF[query]
    cfg = args.config or default_config(query)
    sql = Q.BENCH[query][0]
    engine = Engine(local)
    apply_options(engine, args)
    per_rank = load_tables(engine, query, sf, args.seed, rank, world)
    lib = _native.b200()
    stream = torch.cuda.ExternalStream(lib.hawk_b200_ctx_stream(engine.ctx), device=torch.device("cuda", local))
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    peak, peak_kind = measured_peak()
    r0 = engine.run(sql, cfg) if world == 1 else None
    acct = query_bytes(engine, query, sf, per_rank, world, r0, l2) if world == 1 else None
    xdev = torch.device("cuda", local) if args.backend == "nccl" else torch.device("cpu")
    comm = None
    if world > 1 and args.backend == "nccl":
        # the engine's own NCCL communicator (include/hawk_b200_comm.h); torch
        # only ships its 128-byte id from rank 0
        from paper_1709_00700_b200 import Communicator
        uid = torch.zeros(128, dtype=torch.uint8, device=xdev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(Communicator.unique_id()), dtype=torch.uint8))
        torch.distributed.broadcast(uid, 0)
        comm = Communicator(engine, world, rank, bytes(uid.cpu().numpy().tobytes()))

    def step():
        """One query: (result, kernels launched). N>1: every rank runs its
        shard, the partials stay in HBM and are gathered to rank 0 with NCCL
        over device buffers, merged there on the device (Engine.run_sharded).
        --backend gloo (ranks sharing one GPU): host exchange + finalize."""
        if world == 1:
            r = engine.run(sql, cfg)
            return r, r.launches
        if comm is not None:
            r = engine.run_sharded(sql, cfg, comm)
            return r, r.launches
        part = engine.run_partial(sql, cfg)
        gathered = all_gather_rows(part.rows, device=xdev)
        r = engine.finalize(sql, gathered, cfg)
        return r, part.launches + r.launches

    flush = (acct["whole_query"] if acct else per_rank * 8 * len(Q.FACT_COLUMNS[query])) < 4 * l2
    with Clocks(local) as clocks:
        total_ms, outs = timed_steps(engine, stream, step, args.steps, args.warmup, flush, world=world)
        if world == 1:
            clocks.keep_busy(step)
        else:  # every rank runs the same number of extra (untimed) steps, ~0.4 s
            t = torch.tensor([total_ms / args.steps], device=xdev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            for _ in range(min(20000, int(400.0 / max(float(t.item()), 1e-3)) + 1)):
                step()
    if world > 1:
        t = torch.tensor([total_ms], device=xdev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = per_rank * world / (ms_per_step / 1e3)
    launches = sum(o.launches for o in outs)

    line = {
        "metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic (include/hawk_gen.h, generated in HBM)",
        "config": workload_config(query, sf, world),
        "variant": cfg,
        "l2": ("flushed between steps" if flush else "inputs larger than L2 "
               f"({per_rank * 8 * len(Q.FACT_COLUMNS[query]) / 1e9:.2f} GB vs {l2 / 1e6:.0f} MB)"),
        "gpu_launches": launches,
    }
    if world == 1:
        term_ms = statistics.mean(o.pipelines[-1]["kernel_ms"] for o in outs)
        achieved = acct["terminal"] / term_ms / 1e6
        line["hbm_gbs"] = acct["whole_query"] / ms_per_step / 1e6
        line["roofline"] = {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": ncu_traffic(query, sf),
            "kernel": f"terminal pipeline (hk_jit_pipeline) of {WORKLOAD_NAME[query]}",
            "algorithmic_bytes_per_launch": acct["terminal"], "kernel_ms": term_ms,
            "peak_kind": peak_kind,
            "whole_query": {"bytes": acct["whole_query"], "achieved": line["hbm_gbs"],
                            "frac": line["hbm_gbs"] / peak, "detail": acct["detail"]},
        }
    line["clocks"] = clocks.summary()

    if not args.no_e2e:
        line["e2e"] = e2e_measure(engine, query, sf, args, step, rank, world, per_rank)
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from ref_sharded import ShardedReference
        info = host_info()
        sample = reference_sample_rows(query, sf, 1)
        ref = ShardedReference(query, sf, args.seed, fact_rows=sample)
        t = min(ref.timed(1))
        line["cpu_baseline"] = {
            "value": ref.fact_rows / t, "unit": "tuples/s", "cores": ref.threads, "kind": "reference",
            "sample": f"reference_execute (unmodified reference sources, oracle/_ref) over {ref.fact_rows} "
                      f"fact rows of {WORKLOAD_NAME[query]} SF{sf:g}, one row shard per host thread "
                      f"({ref.shards} shards), merged; 1 run",
            "cpu_model": info["cpu_model"], "host_cores": info["cores"]}
        del ref
        # the reference's CPU variant (cpu-o), restated in
        # oracle/cpu_o.cpp over the reference's own pipeline programs
        from ref_sharded import cpu_variant_rate
        rate, threads, rows = cpu_variant_rate(query, sf, args.seed)
        line["cpu_variant"] = {
            "value": rate, "unit": "tuples/s", "cores": threads, "kind": "port",
            "sample": f"cpu-o variant (single-pass, local hash, sequential, linear probing, murmur, branched, "
                      f"one worker per host thread) over all {rows} fact rows of {WORKLOAD_NAME[query]} "
                      f"SF{sf:g}; 1 run after 1 warm-up"}
    if world == 1 and not args.no_per_query and args.config is None and args.sf is None:
        drop_tables(engine, query)
        line["per_query"] = {}
        for q in DEFAULT_CONFIG:
            try:
                line["per_query"][q] = measure_query(engine, stream, q, BASELINE_SF[q], default_config(q),
                                                     args.per_query_steps, 3, l2, peak)
            except Exception as e:  # noqa: BLE001 - reported in the line
                line["per_query"][q] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    engine.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def e2e_measure(engine, query, sf, args, step, rank, world, per_rank):
    """Same metric through the engine's C ABI with HOST inputs: each step copies
    this rank's fact-table shard (the referenced columns) from pinned host
    memory into HBM (hawk_engine_put_columns), runs the query (N>1: partials,
    exchange, merge) and reads the result back (D2H). Timed per step as the max
    over ranks."""
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
                    + (" / run_partial + exchange + finalize" if world > 1 else "")}


if __name__ == "__main__":
    main()
