fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(d["query"], round(d.get("kernel_ms", -1), 4), d["config"][:110], d.get("error", "")[:200], [round(p["kernel_ms"],3) for p in d.get("pipelines", [])])'
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
P="single_pass/coalesced/branched"
Q1S="$P;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8 $P;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/ht=8 $P;local_hash/coalesced/branched/cuckoo/multiply_shift/wg=256/ht=8 $P;local_hash/coalesced/predicated/linear_probing/murmur/wg=256/ht=8 $P;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=1 $P;local_hash/coalesced/branched/linear_probing/murmur/wg=128/ht=8 $P/u=2;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8/u=2"
timeout 600 python bench.py --query tpch_q1 --sweep $Q1S 2>&1 | python3 -c "$fmt"
echo "== stage0"
timeout 600 python bench.py --query tpch_q1 --stage 0 --sweep $Q1S 2>&1 | python3 -c "$fmt"
echo "== dense off"
python - <<'PY'
import subprocess
PY
for q in ssb_q41 tpch_q6; do
timeout 600 python bench.py --query $q --sweep \
 "$P;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256" \
 "$P;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/ht=8" \
 "single_pass/sequential/branched/u=2;global_hash/sequential/branched/linear_probing/multiply_shift/wg=256/u=2" \
 2>&1 | python3 -c "$fmt"
done
