set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/host_cpu.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_train.json 2> gpurun_out/bench_train.err; tail -c 3000 gpurun_out/bench_train.json
python bench.py --workload augment --steps 20 --warmup 5 > gpurun_out/bench_augment.json 2> gpurun_out/bench_augment.err; tail -c 1500 gpurun_out/bench_augment.json
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2>&1; tail -c 1000 gpurun_out/bench_reference.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/train_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/augment_launches.csv python bench.py --workload augment --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out
