mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for pf in 0 2 4; do
  timeout 300 python bench.py --query tpch_q6 --prefetch $pf --sweep 2>&1 | python3 -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print('pf=$pf', d['query'], round(d.get('kernel_ms', -1), 4), d['config'][:110], d.get('error', ''))"
done
timeout 600 python bench.py --query tpch_q1 --sweep 2>&1 | python3 -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(d['query'], round(d.get('kernel_ms', -1), 4), d['config'][:110], d.get('error', ''))"
