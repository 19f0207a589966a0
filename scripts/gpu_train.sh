set -x
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -3
timeout 900 python bench.py --workload train --steps 5 --warmup 3 2>&1 | tail -5
