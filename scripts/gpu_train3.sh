timeout 900 python bench.py --workload train --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('attn_tflops'))
for k,v in sorted(d['kernels'].items(), key=lambda kv:-kv[1]['total_ms']): print(k, round(v['total_ms']/5,3), 'ms/step', round(v.get('share_of_step',0),3), v.get('tflops'))"
