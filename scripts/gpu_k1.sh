set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -20
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py --workload augment --steps 20 --warmup 5 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/k1_launches.csv python bench.py --workload augment --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_rrc -s 3 -c 1 -o gpurun_out/k1_prof python bench.py --workload augment --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_k1.log 2>&1
tail -3 gpurun_out/ncu_k1.log
