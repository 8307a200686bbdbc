fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(d["query"], round(d.get("kernel_ms", -1), 4), d["config"][:110], d.get("error", "")[:200], [round(p["kernel_ms"],3) for p in d.get("pipelines", [])])'
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
P="single_pass/coalesced/branched"
C1="$P;local_hash/coalesced/predicated/linear_probing/murmur/wg=256/ht=8"
for m in 0 2 4; do echo "== q1 min_ctas $m"; timeout 600 python bench.py --query tpch_q1 --min-ctas $m --sweep "$C1" "$P;local_hash/coalesced/predicated/linear_probing/murmur/wg=256/ht=4" "$P;local_hash/coalesced/predicated/linear_probing/murmur/wg=256/ht=16" 2>&1 | python3 -c "$fmt"; done
echo "== q3 build unroll"
timeout 600 python bench.py --query tpch_q3 --sweep "$P/u=2;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=64" "$P/u=4;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=64" "single_pass/sequential/branched/u=4;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=64" 2>&1 | python3 -c "$fmt"
timeout 900 python tools/sweep_space.py tpch_q1 10 > gpurun_out/sweep_tpch_q1_sf10.jsonl 2> gpurun_out/sweep_q1.err; cat gpurun_out/sweep_tpch_q1_sf10.jsonl | cut -c1-300
