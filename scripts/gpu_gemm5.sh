for i in 1 2; do
timeout 200 python scripts/bench_gemm.py 2>&1 | grep -E "gelu|fc2_dgrad\"" | cut -c1-100
echo PAIR_AUX; AVB_GEMM_PAIR_AUX=1 timeout 200 python scripts/bench_gemm.py 2>&1 | grep -E "gelu" | cut -c1-100
echo NOPAIR; AVB_GEMM_NO_PAIR=1 timeout 200 python scripts/bench_gemm.py 2>&1 | grep -E "gelu" | cut -c1-100
done
AVB_GEMM_PAIR_AUX=1 timeout 200 python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -1
