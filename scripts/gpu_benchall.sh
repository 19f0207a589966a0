lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/host_cpu.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_train.json 2> gpurun_out/bench_train.err; tail -c 400 gpurun_out/bench_train.json
timeout 600 python bench.py --workload augment --steps 20 --warmup 5 > gpurun_out/bench_augment.json 2> gpurun_out/bench_augment.err; tail -c 300 gpurun_out/bench_augment.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2>&1; tail -c 300 gpurun_out/bench_reference.json
timeout 600 python bench.py --workload clip --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_clip.json 2> gpurun_out/bench_clip.err; tail -c 200 gpurun_out/bench_clip.json
timeout 900 python bench.py --workload train-l14 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_l14.json 2> gpurun_out/bench_l14.err; tail -c 200 gpurun_out/bench_l14.json
