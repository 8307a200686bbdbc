# scan-only pipelines: TMA-staged + per-pass barrier vs unstaged coalesced loads, no barrier
mkdir -p gpurun_out
run() {
  timeout 120 python bench.py --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | python3 -c "
import sys, json
d = json.loads(sys.stdin.read())
r = d['roofline']
print('$*', round(r['kernel_ms'], 4), round(r['frac'], 3), round(d['ms_per_step'], 4))"
}
for rep in 1 2; do
  for q in tpch_q1 tpch_q6; do
    run --query $q
    run --query $q --stage 0 --pass-sync 0
    run --query $q --stage 0 --pass-sync 0 --min-ctas 3
  done
done
run --query tpch_q1 --sf 1
run --query tpch_q1 --sf 1 --stage 0 --pass-sync 0
