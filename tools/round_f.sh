timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "baseline_queries_match_oracle and tpch and ht=64" 2>&1 | grep -E "^E " | head -10
