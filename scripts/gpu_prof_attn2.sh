ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/attn_fwd4 python scripts/prof_attn.py > gpurun_out/ncu_attn2.log 2>&1
tail -2 gpurun_out/ncu_attn2.log
timeout 300 python -m pytest tests/test_clip_gpu.py -x -q 2>&1 | tail -15
