set -x
timeout 600 python -m pytest tests/test_model_gpu.py tests/test_gemm_gpu.py -x -q 2>&1 | tail -25
