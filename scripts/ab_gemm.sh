#!/usr/bin/env bash
# usage: scripts/ab_gemm.sh outdir lib1 lib2 ... : GEMM parity tests on the in-tree lib, then same-box GEMM + train A/B
O=$1; shift; mkdir -p $O
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_bench_shapes_gpu.py -q -x 2>&1 | tail -2 > $O/tests.txt
for rep in 1 2; do for L in "$@"; do
  echo "== $L" >> $O/ab.txt
  AVB_LIB=$L timeout 300 python scripts/bench_gemm.py >> $O/ab.txt 2>&1
  AVB_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-breakdown 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('train', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'mhz', d['clocks']['sm_mhz'])" >> $O/ab.txt 2>&1
done; done
