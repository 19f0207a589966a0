timeout 300 python -m pytest tests/test_infonce_gpu.py -x -q 2>&1 | tail -15
ncu --set full --clock-control none --import-source on -k regex:attn_ -s 3 -c 3 -o gpurun_out/attn_prof python scripts/prof_attn.py > gpurun_out/ncu_attn.log 2>&1
tail -2 gpurun_out/ncu_attn.log
