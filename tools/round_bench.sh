timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for q in tpch_q1 tpch_q6 ssb_q11 ssb_q41 tpch_q3; do
  timeout 900 python bench.py --query $q > gpurun_out/bench_$q.json 2> gpurun_out/bench_$q.err
  python3 -c "
import json,sys
d=json.loads(open('gpurun_out/bench_$q.json').read().strip().splitlines()[-1])
r=d.get('roofline',{}); e=d.get('e2e',{}); c=d.get('cpu_baseline',{})
print('$q', round(d['value']/1e9,2), 'Gt/s', round(d['ms_per_step'],4), 'ms', 'frac', round(r.get('frac',0),3), 'kern', round(r.get('kernel_ms',0),4), 'e2e', round(e.get('value',0)/1e9,3), 'cpu', round(c.get('value',0)/1e6,2), d['clocks'])
" || tail -5 gpurun_out/bench_$q.err
done
bash tools/profile_all.sh
