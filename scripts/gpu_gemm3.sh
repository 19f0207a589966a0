timeout 240 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -2
timeout 240 python scripts/bench_gemm.py 2>&1 | tail -13 | cut -c1-125
echo NOPAIR
AVB_GEMM_NO_PAIR=1 timeout 240 python scripts/bench_gemm.py 2>&1 | grep -E "qkv_fwd|sq8192|fc2_fwd|wgrad" | cut -c1-110
