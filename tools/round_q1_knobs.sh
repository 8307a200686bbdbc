# TPC-H Q1 SF10 terminal kernel vs launch/staging knobs (no rebuild needed)
mkdir -p gpurun_out
run() {
  timeout 120 python bench.py --query tpch_q1 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | python3 -c "
import sys, json
d = json.loads(sys.stdin.read())
r = d['roofline']
print('$*', round(r['kernel_ms'], 4), round(r['frac'], 3), round(d['ms_per_step'], 4))"
}
run
for mc in 2 3 4; do run --min-ctas $mc; done
for pf in 1 3 4; do run --prefetch $pf; done
run --stage 0
run --stage 0 --l2-distance 2
run --stage 0 --pass-sync 0
run --config "single_pass/coalesced/predicated;local_hash/coalesced/predicated/linear_probing/murmur/wg=256/ht=8"
run --config "single_pass/coalesced/branched;local_hash/coalesced/predicated/linear_probing/murmur/wg=512/ht=8"
run --config "single_pass/coalesced/branched;local_hash/coalesced/predicated/linear_probing/murmur/wg=128/ht=8"
run --config "single_pass/coalesced/branched;local_hash/coalesced/predicated/linear_probing/multiply_shift/wg=256/ht=8/u=2"
