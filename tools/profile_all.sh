# ncu evidence for profiles/: per query, a plain run, then the launch list and
# one --set full capture of the terminal pipeline kernel (1 GPU).
# usage: bash tools/profile_all.sh [queries...]
mkdir -p gpurun_out
qs="${@:-tpch_q1 tpch_q6 ssb_q11 ssb_q41 tpch_q3}"
for q in $qs; do
  case $q in tpch_q1|tpch_q6) np=1;; ssb_q11) np=2;; ssb_q41) np=5;; tpch_q3) np=3;; esac
  skip=$((np * 2 + np - 1))   # warm-up run + first timed run, then the terminal kernel
  cmd="python bench.py --query $q --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
  $cmd > gpurun_out/plain_$q.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$q.csv $cmd > gpurun_out/ncu_launch_$q.log 2>&1
  $cmd > gpurun_out/plain2_$q.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:pipeline -s $skip -c 1 -o gpurun_out/full_$q $cmd > gpurun_out/ncu_full_$q.log 2>&1
done
