timeout 900 python bench.py --workload train --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); print(json.dumps(d['gemm_shapes'], indent=0)); print(json.dumps(d['kernels']))"
