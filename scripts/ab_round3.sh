#!/usr/bin/env bash
# same-box A/B: base (HEAD), nohint (new LN), hint (new LN + try_wait suspend hint = in-tree)
O=gpurun_out/v3; mkdir -p $O
python -m pytest tests/test_model_gpu.py -q -x -k "layernorm" > $O/ln_tests.txt 2>&1
for rep in 1 2; do
for L in scratch_libs/base.so scratch_libs/nohint.so scratch_libs/hint.so; do
  echo "== $L" >> $O/ab.txt
  AVB_LIB=$L timeout 300 python scripts/bench_ln.py >> $O/ab.txt 2>&1
  AVB_LIB=$L timeout 300 python scripts/bench_attn_bwd.py >> $O/ab.txt 2>&1
done
done
for L in scratch_libs/base.so scratch_libs/hint.so; do
  echo "== $L" >> $O/ab_gemm.txt
  AVB_LIB=$L timeout 300 python scripts/bench_gemm.py >> $O/ab_gemm.txt 2>&1
done
for L in scratch_libs/base.so scratch_libs/hint.so scratch_libs/base.so scratch_libs/hint.so; do
  echo "== $L" >> $O/ab_train.txt
  AVB_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-breakdown | head -c 400 >> $O/ab_train.txt 2>&1
  echo >> $O/ab_train.txt
done
