mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "baseline_queries_match_oracle and tpch" 2>&1 | grep -E "Error|assert|diff|FAILED|passed|failed" | head -20
CFG1='single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=1'
python bench.py --query tpch_q1 --sweep "$CFG1" > gpurun_out/q1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pipeline_kernel -s 3 -c 1 -o gpurun_out/q1d_prof python bench.py --query tpch_q1 --sweep "$CFG1" > gpurun_out/q1_ncu.log 2>&1
