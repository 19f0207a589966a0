timeout 300 python -m pytest tests/test_k1_gpu.py tests/test_model_gpu.py -x -q 2>&1 | tail -15
timeout 300 python bench.py --workload augment --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-1500
