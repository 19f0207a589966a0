set -x
timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_model_gpu.py -x -q 2>&1 | tail -5
timeout 300 python scripts/bench_gemm.py 2>&1 | tail -12
timeout 900 python bench.py --workload train --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -2
