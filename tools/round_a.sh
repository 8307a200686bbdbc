mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d["query"], round(d.get("kernel_ms", -1), 4), d["config"][:120], d.get("error", ""))'
timeout 600 python bench.py --query tpch_q1 --sweep \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=1" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=128/ht=8" \
 "single_pass/coalesced/branched;local_hash/coalesced/predicated/linear_probing/murmur/wg=256/ht=8" \
 "single_pass/coalesced/branched;local_hash/sequential/branched/linear_probing/murmur/wg=256/ht=8" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8/u=2" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/cuckoo/murmur/wg=256/ht=8" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=64/ht=64" \
 2>&1 | python3 -c "$fmt"
CFG6='single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/murmur/wg=256/u=4'
CFG1='single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8'
python bench.py --query tpch_q6 --sweep "$CFG6" > gpurun_out/q6_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pipeline_kernel -s 3 -c 1 -o gpurun_out/q6b_prof python bench.py --query tpch_q6 --sweep "$CFG6" > gpurun_out/q6_ncu.log 2>&1
python bench.py --query tpch_q1 --sweep "$CFG1" > gpurun_out/q1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pipeline_kernel -s 3 -c 1 -o gpurun_out/q1b_prof python bench.py --query tpch_q1 --sweep "$CFG1" > gpurun_out/q1_ncu.log 2>&1
cat gpurun_out/q6_plain.log gpurun_out/q1_plain.log | python3 -c "$fmt"
