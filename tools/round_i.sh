CFG1='single_pass/coalesced/branched;local_hash/coalesced/branched/linear_probing/murmur/wg=256/ht=1/u=2'
python bench.py --query tpch_q1 --sweep "$CFG1" > gpurun_out/q1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:pipeline -s 3 -c 1 -o gpurun_out/q1j_prof python bench.py --query tpch_q1 --sweep "$CFG1" > gpurun_out/q1_ncu.log 2>&1
tail -3 gpurun_out/q1_ncu.log
