fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(d["query"], d.get("sf"), round(d.get("kernel_ms", -1), 4), d["config"][:100], d.get("error", "")[:300], [(round(p["kernel_ms"],3), p["rows_out"]) for p in d.get("pipelines", [])])'
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for q in ssb_q11 ssb_q41 tpch_q3; do
timeout 600 python bench.py --query $q --sweep \
 "single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/murmur/wg=256" \
 "single_pass/coalesced/branched;global_hash/coalesced/branched/cuckoo/murmur/wg=256" \
 "single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256" \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8" \
 2>&1 | python3 -c "$fmt"
done
bash tools/profile_all.sh
