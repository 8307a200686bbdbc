timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for q in tpch_q1 tpch_q6 ssb_q11 ssb_q41 tpch_q3; do
  timeout 900 python bench.py --query $q > gpurun_out/bench_$q.json 2> gpurun_out/bench_$q.err || tail -3 gpurun_out/bench_$q.err
done
for q in ssb_q41 tpch_q3; do
  timeout 1200 python bench.py --query $q --sf 100 --no-e2e > gpurun_out/bench_sf100_$q.json 2> gpurun_out/bench_sf100_$q.err || tail -3 gpurun_out/bench_sf100_$q.err
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
bash tools/profile_all.sh
