#!/usr/bin/env bash
# same-box A/B of the K1 identity kernel through bench.py --workload feed (base.so vs ident.so)
O=${OUT:-gpurun_out/v45}; mkdir -p $O
AVB_LIB=${TESTLIB:-scratch_libs/ident.so} timeout 600 python -m pytest tests/test_k1_gpu.py tests/test_api_gpu.py -q -x 2>&1 | tail -3 > $O/tests.txt
for rep in 1 2 3; do for L in ${LIBS:-scratch_libs/base.so scratch_libs/ident.so}; do
  echo "== $L" >> $O/ab.txt
  AVB_LIB=$L timeout 300 python bench.py --workload feed --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('ms', round(r['ms_per_launch'],4), 'GBs', round(r['achieved'],0), 'frac', round(r['frac'],3), 'e2e', round(d['e2e']['value'],0))" >> $O/ab.txt 2>&1
done; done
