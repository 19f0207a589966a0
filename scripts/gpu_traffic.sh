timeout 300 ncu --set full --clock-control none -k regex:attn_bwd_kernel -c 1 -o gpurun_out/traffic_attn_bwd python scripts/prof_attn.py > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:attn_fwd_kernel -s 2 -c 1 -o gpurun_out/traffic_attn_fwd python scripts/prof_attn.py > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1v4 -s 2 -c 1 -o gpurun_out/traffic_k1 python bench.py --workload augment --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/train_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/train_launches.csv
