CFG1='single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=128/ht=8'
python bench.py --query tpch_q1 --stage 0 --sweep "$CFG1" > gpurun_out/q1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pipeline -s 3 -c 1 -o gpurun_out/q1k_prof python bench.py --query tpch_q1 --stage 0 --sweep "$CFG1" > gpurun_out/q1_ncu.log 2>&1
tail -2 gpurun_out/q1_ncu.log
