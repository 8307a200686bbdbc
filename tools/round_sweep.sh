timeout 900 python -m pytest tests -m gpu -x -q -k "parity and (baseline or sharded or micro)" 2>&1 | tail -2
timeout 1500 python tools/sweep_space.py tpch_q3 100 --full > gpurun_out/sweep_tpch_q3_sf100.jsonl 2> gpurun_out/sweep_q3.err; tail -2 gpurun_out/sweep_q3.err
timeout 1500 python tools/sweep_space.py ssb_q41 100 --full > gpurun_out/sweep_ssb_q41_sf100.jsonl 2> gpurun_out/sweep_q41.err; tail -2 gpurun_out/sweep_q41.err
timeout 900 python tools/sweep_space.py tpch_q1 10 > gpurun_out/sweep_tpch_q1_sf10.jsonl 2> gpurun_out/sweep_q1.err; tail -2 gpurun_out/sweep_q1.err
