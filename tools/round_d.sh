mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d["query"], d.get("sf"), round(d.get("kernel_ms", -1), 4), d["config"][:110], d.get("error", ""))'
timeout 600 python bench.py --query tpch_q1 --sweep \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=1" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/ht=8" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=128/ht=8" \
 "single_pass/coalesced/branched;local_hash/coalesced/predicated/linear_probing/murmur/wg=256/ht=8" \
 "single_pass/coalesced/branched;local_hash/sequential/branched/linear_probing/murmur/wg=256/ht=8" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=64/ht=64" \
 2>&1 | python3 -c "$fmt"
