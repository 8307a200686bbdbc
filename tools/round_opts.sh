fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(d["query"], round(d.get("kernel_ms", -1), 4), d["config"][:110], d.get("error", "")[:200], [round(p["kernel_ms"],3) for p in d.get("pipelines", [])])'
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
G="single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256"
G2="single_pass/coalesced/branched/u=2;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/u=2"
GS="single_pass/sequential/branched;global_hash/sequential/branched/linear_probing/multiply_shift/wg=256"
GS2="single_pass/sequential/branched/u=2;global_hash/sequential/branched/linear_probing/multiply_shift/wg=256/u=2"
L="single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8"
for q in tpch_q1 ssb_q41 tpch_q3 ssb_q11 tpch_q6; do
 for opt in "--stage 1" "--stage 0 --l2-distance 0" "--stage 0 --l2-distance 1" "--stage 0 --l2-distance 2" "--stage 0 --l2-distance 4"; do
  echo "== $q $opt"
  if [ $q = tpch_q1 ]; then C="$L"; else C="$G $G2 $GS $GS2"; fi
  timeout 600 python bench.py --query $q $opt --sweep $C 2>&1 | python3 -c "$fmt"
 done
done
