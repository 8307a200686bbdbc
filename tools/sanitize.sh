#!/bin/bash
# compute-sanitizer over every kernel role (tools/sanitize_driver.py), both jit
# modes: memcheck, racecheck (shared-memory hazards), synccheck. Run on a B200:
#   bash tools/sanitize.sh   -> gpurun_out/sanitize_<tool>.log
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  SAN_ROWS=${SAN_ROWS:-20000} timeout 2400 compute-sanitizer --tool $tool $extra --print-limit 50 \
      --error-exitcode 9 python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_$tool.log
  tail -4 gpurun_out/sanitize_$tool.log
done
