fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(d["query"], round(d.get("kernel_ms", -1), 4), d["config"][:110], d.get("error", "")[:200], [round(p["kernel_ms"],3) for p in d.get("pipelines", [])])'
P="single_pass/coalesced/branched"
timeout 600 python bench.py --query tpch_q1 --sweep \
 "$P;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=8" \
 "$P;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/ht=8" \
 "$P;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=128/ht=8" \
 "$P;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/ht=1" \
 "$P;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/ht=64" \
 "$P;local_hash/coalesced/predicated/linear_probing/multiply_shift/wg=256/ht=8" \
 "$P;local_hash/sequential/branched/linear_probing/multiply_shift/wg=256/ht=8" \
 "$P;local_hash/sequential/predicated/linear_probing/multiply_shift/wg=256/ht=8" \
 "$P;local_hash/coalesced/branched/cuckoo/multiply_shift/wg=256/ht=8" \
 "$P/u=2;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/ht=8/u=2" \
 2>&1 | python3 -c "$fmt"
timeout 600 python bench.py --query tpch_q1 --stage 0 --pass-sync 0 --sweep \
 "$P;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/ht=8" 2>&1 | python3 -c "$fmt"
for q in ssb_q41 tpch_q3 ssb_q11; do
timeout 600 python bench.py --query $q --sweep \
 "$P;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256" \
 "$P/u=2;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256" \
 "$P;global_hash/coalesced/predicated/linear_probing/multiply_shift/wg=256" \
 "$P;global_hash/coalesced/branched/cuckoo/multiply_shift/wg=256" \
 "$P;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/ht=8" \
 2>&1 | python3 -c "$fmt"
done
