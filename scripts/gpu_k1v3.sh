timeout 300 python -m pytest tests/test_k1_gpu.py tests/test_model_gpu.py -x -q 2>&1 | tail -15
timeout 300 python bench.py --workload augment --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])"
AVB_K1_V2=1 timeout 300 python bench.py --workload augment --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('v2', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])"
bash scripts/gpu_train3.sh
