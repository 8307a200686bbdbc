timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for q in tpch_q1 tpch_q6 ssb_q11 ssb_q41 tpch_q3; do
  timeout 900 python bench.py --query $q > gpurun_out/bench_$q.json 2> gpurun_out/bench_$q.err
  python3 -c "
import json,sys
d=json.loads(open('gpurun_out/bench_$q.json').read().strip().splitlines()[-1])
r=d.get('roofline',{}); e=d.get('e2e',{}); c=d.get('cpu_baseline',{})
print('$q', round(d['value']/1e9,2), 'Gt/s', round(d['ms_per_step'],4), 'ms', 'frac', round(r.get('frac',0),3), 'kern', round(r.get('kernel_ms',0),4), 'e2e', round(e.get('value',0)/1e9,3), round(e.get('ms_per_step',0),2), 'cpu', round(c.get('value',0)/1e6,2), d['clocks'])
" || tail -5 gpurun_out/bench_$q.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --backend gloo --steps 3 --warmup 3 --query tpch_q3 --sf 1 --no-cpu-baseline 2> gpurun_out/n2.err | tail -1 | cut -c1-400; tail -2 gpurun_out/n2.err
