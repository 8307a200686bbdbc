fmt='import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:300]); continue
    print(d["query"], d["sf"], round(d.get("kernel_ms", -1), 4), d.get("error", "")[:200], [round(p["kernel_ms"],3) for p in d.get("pipelines", [])])'
C="single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/multiply_shift/wg=256"
for sf in 10 100; do for env in "" "HAWK_NO_KEY_BITMAPS=1" "" "HAWK_NO_KEY_BITMAPS=1"; do
echo "== $sf $env"; env $env timeout 900 python bench.py --query ssb_q41 --sf $sf --sweep "$C" 2>&1 | python3 -c "$fmt"
done; done
HAWK_TRACE=1 python tools/host_trace.py ssb_q41 2>&1 | grep -v Warn | tail -3
python - <<'PY'
import sys; sys.path.insert(0,'.')
import bench
from paper_1709_00700_b200 import Engine, queries as Q
e=Engine(0); bench.load_tables(e,'ssb_q41',10,42,0,1)
print(e.explain(Q.BENCH['ssb_q41'][0], bench.DEFAULT_CONFIG['ssb_q41']))
PY
