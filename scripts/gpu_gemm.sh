set -x
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -15
timeout 300 python scripts/bench_gemm.py 2>&1 | tail -12
