mkdir -p gpurun_out
CFG6='single_pass/coalesced/branched;global_hash/coalesced/branched/linear_probing/murmur/wg=256'
CFG1='single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/multiply_shift/wg=256/ht=8'
python bench.py --query tpch_q6 --sweep "$CFG6" > gpurun_out/q6_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pipeline_kernel -s 3 -c 1 -o gpurun_out/q6_prof python bench.py --query tpch_q6 --sweep "$CFG6" > gpurun_out/q6_ncu.log 2>&1
python bench.py --query tpch_q1 --sweep "$CFG1" > gpurun_out/q1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pipeline_kernel -s 3 -c 1 -o gpurun_out/q1_prof python bench.py --query tpch_q1 --sweep "$CFG1" > gpurun_out/q1_ncu.log 2>&1
python -m pytest tests/test_gpu_parity.py -q -x -k "round_trip" 2>&1 | tail -3
ls -la gpurun_out
