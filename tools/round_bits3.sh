fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(d["query"], round(d.get("kernel_ms", -1), 4), d["config"][:110], d.get("error", "")[:200], [round(p["kernel_ms"],3) for p in d.get("pipelines", [])])'
P="single_pass/coalesced/branched"
for m in 0 1 4 5 0 5; do
echo "== mask $m"
HAWK_BITMAP_PROBES=$m timeout 600 python bench.py --query ssb_q41 --sweep \
 "$P;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256" "$P;global_hash/coalesced/branched/cuckoo/multiply_shift/wg=256" 2>&1 | python3 -c "$fmt"
done
HAWK_TRACE=1 python tools/host_trace.py ssb_q41 2>&1 | grep -i "probe\|run 3" | head
