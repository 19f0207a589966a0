set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log; tail -30 gpurun_out/pytest_gpu.log
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -3
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_train.json 2> gpurun_out/bench_train.err; tail -c 600 gpurun_out/bench_train.json
timeout 300 python bench.py --workload augment --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_augment.json 2> gpurun_out/bench_augment.err; tail -c 800 gpurun_out/bench_augment.json
