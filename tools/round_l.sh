fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(d["query"], d.get("sf"), round(d.get("kernel_ms", -1), 4), d["config"][:100], d.get("error", "")[:300])'
for st in 1 0; do
echo "stage=$st"
timeout 600 python bench.py --query tpch_q6 --stage $st --sweep \
 "single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/murmur/wg=256" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8" \
 "single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/murmur/wg=128" \
 2>&1 | python3 -c "$fmt"
timeout 600 python bench.py --query tpch_q1 --stage $st --sweep \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=128/ht=8" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=64/ht=8" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=128/ht=8/u=2" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8" \
 2>&1 | python3 -c "$fmt"
done
