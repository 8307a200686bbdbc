#!/bin/bash
# One GPU round trip (run under gpurun): parity tests, smoke, bench (both arms).
# Logs land in gpurun_out/ (merged back by gpurun).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
TESTS=${TESTS:-tests}
timeout ${TEST_TIMEOUT:-1500} python -m pytest $TESTS -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
if [ -z "$SKIP_SMOKE" ]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -8 gpurun_out/smoke.log
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  tail -c 600 gpurun_out/bench.err
  timeout 900 python bench.py --impl reference ${BENCH_ARGS:-} > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
  tail -c 600 gpurun_out/bench_ref.err
fi
