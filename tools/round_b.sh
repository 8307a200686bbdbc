mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d["query"], round(d.get("kernel_ms", -1), 4), d["config"][:120], d.get("error", ""))'
for pf in 2 3; do
echo "stages=$pf"
timeout 600 python bench.py --query tpch_q6 --prefetch $pf --sweep \
 "single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/murmur/wg=256" \
 "single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/murmur/wg=128" \
 "single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/murmur/wg=256/u=2" \
 "single_pass/coalesced/branched;global_hash/coalesced/predicated/linear_probing/murmur/wg=256/u=2" \
 "single_pass/coalesced/branched;global_hash/sequential/branched/linear_probing/murmur/wg=256/u=4" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8" \
 2>&1 | python3 -c "$fmt"
timeout 600 python bench.py --query tpch_q1 --prefetch $pf --sweep \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=1" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=128/ht=8" \
 "single_pass/coalesced/branched;local_hash/coalesced/predicated/linear_probing/murmur/wg=256/ht=8" \
 "single_pass/coalesced/branched;local_hash/sequential/branched/linear_probing/murmur/wg=256/ht=8" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8/u=2" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=64/ht=64" \
 2>&1 | python3 -c "$fmt"
done
