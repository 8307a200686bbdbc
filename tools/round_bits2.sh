fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(d["query"], round(d.get("kernel_ms", -1), 4), d["config"][:110], d.get("error", "")[:200], [round(p["kernel_ms"],3) for p in d.get("pipelines", [])])'
P="single_pass/coalesced/branched"
for env in "" "HAWK_NO_KEY_BITMAPS=1"; do
for q in ssb_q41 tpch_q3 ssb_q11; do
echo "== $q $env"
env $env timeout 600 python bench.py --query $q --sweep \
 "$P;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256" \
 "$P/u=4;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=64" \
 "$P;global_hash/coalesced/branched/cuckoo/multiply_shift/wg=256" \
 2>&1 | python3 -c "$fmt"
done; done
echo "== q1"; timeout 600 python bench.py --query tpch_q1 --sweep "$P;local_hash/coalesced/predicated/linear_probing/murmur/wg=256/ht=8" 2>&1 | python3 -c "$fmt"
echo "== q6"; timeout 600 python bench.py --query tpch_q6 --sweep "single_pass/sequential/branched/u=2;global_hash/sequential/branched/linear_probing/multiply_shift/wg=256/u=2" "$P;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256" 2>&1 | python3 -c "$fmt"
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
