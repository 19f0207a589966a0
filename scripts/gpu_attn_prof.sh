timeout 300 python scripts/bench_attn2.py 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 2 -c 1 -o gpurun_out/attn_bwd_prof python scripts/prof_attn.py > gpurun_out/ncu_attn_bwd.log 2>&1; tail -2 gpurun_out/ncu_attn_bwd.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 2 -c 1 -o gpurun_out/attn_fwd_prof python scripts/prof_attn.py > gpurun_out/ncu_attn_fwd.log 2>&1; tail -2 gpurun_out/ncu_attn_fwd.log
