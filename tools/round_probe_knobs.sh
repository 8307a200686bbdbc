# probe pipelines (SSB Q4.1, TPC-H Q3 at SF10): launch/prefetch knobs, no rebuild
mkdir -p gpurun_out
run() {
  timeout 150 python bench.py --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | python3 -c "
import sys, json
d = json.loads(sys.stdin.read())
r = d['roofline']
print('$*', round(r['kernel_ms'], 4), round(r['frac'], 3), round(d['ms_per_step'], 4))"
}
for q in ssb_q41 tpch_q3; do
  run --query $q
  for mc in 1 2 3 4; do run --query $q --min-ctas $mc; done
  for l2 in 1 2 4; do run --query $q --l2-distance $l2; done
  run --query $q --compact 0
  run --query $q
done
