timeout 300 python -m pytest tests/test_attn_gpu.py tests/test_infonce_gpu.py -x -q 2>&1 | tail -15
timeout 300 python scripts/bench_attn.py 2>&1 | tail -4
