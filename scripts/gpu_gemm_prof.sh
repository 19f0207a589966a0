timeout 300 python scripts/bench_gemm.py 2>&1 | tail -12
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 4 -c 1 -o gpurun_out/gemm_fc1 python scripts/prof_gemm.py > gpurun_out/ncu_gemm.log 2>&1; tail -1 gpurun_out/ncu_gemm.log
