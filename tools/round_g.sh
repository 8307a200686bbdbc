timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d["query"], d.get("sf"), round(d.get("kernel_ms", -1), 4), round(d.get("wall_ms", -1), 4), d["config"][:110], d.get("error", ""), [ (p["kernel_ms"], p["rows_out"]) for p in d.get("pipelines", [])])'
for q in ssb_q11 ssb_q41 tpch_q3; do
timeout 600 python bench.py --query $q --sweep \
 "single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=1" \
 "multi_pass/coalesced/branched/tm=1024;global_hash/coalesced/branched/linear_probing/murmur/wg=256" \
 "single_pass/coalesced/branched;global_hash/coalesced/branched/cuckoo/murmur/wg=256" \
 2>&1 | python3 -c "$fmt"
done
