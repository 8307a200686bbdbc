fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(d["query"], round(d.get("kernel_ms", -1), 4), d["config"][:110], d.get("error", "")[:200], [round(p["kernel_ms"],3) for p in d.get("pipelines", [])])'
G="single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256"
G2="single_pass/coalesced/branched/u=2;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/u=2"
L="single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8"
for q in tpch_q1 ssb_q41 tpch_q3 ssb_q11; do
 for opt in "--stage 1" "--stage 0 --pass-sync 1" "--stage 0 --pass-sync 0" "--stage 1" "--stage 0 --pass-sync 1" "--stage 0 --pass-sync 0"; do
  echo "== $q $opt"
  if [ $q = tpch_q1 ]; then C="$L"; else C="$G $G2"; fi
  timeout 600 python bench.py --query $q $opt --sweep $C 2>&1 | python3 -c "$fmt"
 done
done
