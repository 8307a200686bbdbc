"""Summarises ncu captures into profiles/: per query the terminal kernel's
DRAM traffic, duration, throughput, occupancy and stall mix (full capture) and
the launch list's per-kernel time shares.
  python tools/summarize_ncu.py gpurun_out profiles r01"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

src, dst, tag = sys.argv[1], sys.argv[2], sys.argv[3]
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_of_peak",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.per_cycle_active": "warps_active_per_sm",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "smem_per_block",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_long_scoreboard",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_short_scoreboard",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_barrier",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio": "stall_mio_throttle",
    "lts__t_sectors_op_atom.sum": "l2_atomic_sectors",
    "lts__t_sectors_op_red.sum": "l2_reduction_sectors",
    "l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum": "global_atomic_requests",
    "l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum": "global_reduction_requests",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum": "shared_atomic_wavefronts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "shared_wavefronts",
    "launch__occupancy_limit_registers": "occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem": "occupancy_limit_smem",
    "sm__maximum_warps_per_active_cycle_pct": "theoretical_occupancy_pct",
}
summary = {}
traffic_path = os.path.join(dst, "ncu_traffic.json")
traffic = {k: v for k, v in (json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}).items()
           if "@sf" in k}
PATTERN = os.environ.get("NCU_PATTERN", "*@sf*")
for rep in sorted(glob.glob(os.path.join(src, f"full_{PATTERN}.ncu-rep"))):
    q = os.path.basename(rep)[len("full_"):-len(".ncu-rep")]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        continue
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
    for m, k in METRICS.items():
        if m in hdr:
            i = hdr.index(m)
            d[k] = f"{vals[i]} {units[i]}".strip()
    summary[q] = d
    try:
        def num(m):
            i = hdr.index(m)
            v, u = float(vals[i].replace(",", "")), units[i]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic[q] = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    except Exception:
        pass
launches = {}
SETUP = ("gen_column_kernel", "flush_read_kernel", "column_range_kernel")  # data generation / L2 hygiene / cached stats
for f in sorted(glob.glob(os.path.join(src, f"launches_{PATTERN}.csv"))):
    q = os.path.basename(f)[len("launches_"):-len(".csv")]
    text = open(f).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:]))) if start >= 0 else []
    per = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0][:60]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r.get("Metric Unit", "us"), 1.0)
        per.setdefault(name, [0, 0.0])
        per[name][0] += 1
        per[name][1] += v * scale
    tot = sum(v[1] for v in per.values()) or 1.0
    query_tot = sum(v[1] for k, v in per.items() if not any(s in k for s in SETUP)) or 1.0
    launches[q] = {k: {"launches": c, "us": round(t, 1), "share": round(t / tot, 3),
                       "share_of_query_kernels": None if any(s in k for s in SETUP) else round(t / query_tot, 3)}
                   for k, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1])}
os.makedirs(dst, exist_ok=True)
json.dump(summary, open(os.path.join(dst, f"ncu_full_{tag}.json"), "w"), indent=1)
json.dump(launches, open(os.path.join(dst, f"ncu_launches_{tag}.json"), "w"), indent=1)
json.dump(traffic, open(os.path.join(dst, "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(summary, indent=1)[:4000])
print(json.dumps(launches, indent=1)[:3000])
