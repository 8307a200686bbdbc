"""Aggregates an ncu source page (cuda,sass) to per-source-line instruction
counts and stall samples: python tools/ncu_source_hot.py <report.ncu-rep> [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
cur_file, cur_line, cur_src = "?", "?", ""
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) < 10 or r[0] == "Line No":
        continue
    if r[0]:  # source line row
        cur_line, cur_src = r[0], r[1]
        continue
    try:
        samples, inst = int(r[4]), int(r[7])
    except ValueError:
        continue
    k = (cur_file, cur_line)
    a = agg.setdefault(k, [0, 0, cur_src.strip()[:80]])
    a[0] += inst
    a[1] += samples
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"warp-instructions {tot_i}  stall samples {tot_s}")
for (f, l), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*i/tot_i:5.1f}% inst {100*s/tot_s:5.1f}% smp  {f}:{l}  {src}")
