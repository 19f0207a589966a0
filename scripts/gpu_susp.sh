for r in 1 2; do for H in 0 20000; do
AVB_LIB=$PWD/scripts/micro/lib_s$H.so timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('H=$H', round(d['value'],1), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {k: round(v['total_ms']/d['steps'],2) for k,v in d['kernels'].items() if k in ('gemm_all','attn_bwd','attn_fwd')})"
done; done
