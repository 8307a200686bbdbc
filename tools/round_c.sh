mkdir -p gpurun_out
fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d["query"], d.get("sf"), round(d.get("kernel_ms", -1), 4), round(d.get("wall_ms", -1), 4), d["config"][:100], d.get("error", ""))'
for sf in 0.01 0.1 10; do
timeout 600 python bench.py --query tpch_q6 --sf $sf --sweep \
 "single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/murmur/wg=256" \
 "single_pass/coalesced/branched;global_hash/sequential/branched/linear_probing/murmur/wg=256/u=4" \
 2>&1 | python3 -c "$fmt"
done
CFG1='single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=1'
python bench.py --query tpch_q1 --sweep "$CFG1" > gpurun_out/q1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pipeline_kernel -s 3 -c 1 -o gpurun_out/q1c_prof python bench.py --query tpch_q1 --sweep "$CFG1" > gpurun_out/q1_ncu.log 2>&1
cat gpurun_out/q1_plain.log | python3 -c "$fmt"
