#!/bin/bash
# ncu evidence per BASELINE configuration (1 GPU): a plain run first, then the
# launch list (gpu__time_duration.sum, --clock-control none) and one
# --set full capture of the terminal pipeline kernel; outputs in gpurun_out/
# as launches_<q>@sf<S>.csv / full_<q>@sf<S>.ncu-rep, then
#   python tools/summarize_ncu.py gpurun_out profiles r02
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
export HAWK_BENCH_NO_ACCOUNTING=1
for qs in ${@:-tpch_q6:1:1 tpch_q1:10:1 ssb_q11:10:2 ssb_q41:100:5 tpch_q3:100:3}; do
  IFS=: read q sf np <<< "$qs"
  tag="$q@sf$sf"
  cmd="python bench.py --query $q --sf $sf --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-per-query"
  skip=$((np * 2 + np - 1))   # the first run + the warm-up step, then the timed step's terminal kernel
  timeout 600 $cmd > gpurun_out/plain_$tag.log 2>&1 || { echo "$tag plain failed"; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
      --log-file gpurun_out/launches_$tag.csv $cmd > gpurun_out/ncu_launch_$tag.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:hk_jit -s $skip -c 1 \
      --metrics lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum \
      -o gpurun_out/full_$tag $cmd > gpurun_out/ncu_full_$tag.log 2>&1
  echo "$tag ncu rc=$?"
done
