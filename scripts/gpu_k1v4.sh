set -x
timeout 600 python -m pytest tests/test_k1_gpu.py -x -q 2>&1 | tail -15
timeout 300 python bench.py --workload augment --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_augment.json 2> gpurun_out/bench_augment.err; tail -c 900 gpurun_out/bench_augment.json
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k1v4 -s 2 -c 1 -o gpurun_out/k1v4 python bench.py --workload augment --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_k1v4.log 2>&1; tail -3 gpurun_out/ncu_k1v4.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/augment_launches.csv python bench.py --workload augment --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
