timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_train.json 2> gpurun_out/bench_train.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_train.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d.get('attn_tflops'), d['e2e']['value'], d['clocks'])
for k,v in sorted(d['kernels'].items(), key=lambda kv:-kv[1]['total_ms']): print(k, round(v['total_ms']/d['steps'],3), 'ms/step', round(v.get('share_of_step',0),3), v.get('tflops'))
PY
