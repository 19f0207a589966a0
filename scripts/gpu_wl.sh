timeout 600 python bench.py --workload clip --steps 5 --warmup 3 2>&1 | tail -1 | cut -c1-900
timeout 600 python bench.py --workload train-l14 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['attn_tflops'], d['roofline'])"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline'])
for k,v in sorted(d['kernels'].items(), key=lambda kv:-kv[1]['total_ms'])[:8]: print(k, round(v['total_ms']/5,3), round(v.get('share_of_step',0),3))"
