timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/gemm_pair python scripts/prof_gemm2.py > /dev/null 2>&1
ls -la gpurun_out/gemm_pair.ncu-rep
