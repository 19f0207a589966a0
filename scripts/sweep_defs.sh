#!/usr/bin/env bash
# Same-box A/B of compile-time variants: each argument is a define set ("" = default build);
# every variant is built into its own library file and timed with $BENCH (default scripts/bench_attn_bwd.py).
BENCH=${BENCH:-scripts/bench_attn_bwd.py}
i=0
for defs in "$@"; do
  out=/tmp/sweep_lib_$i.so
  AVB_NVCC_DEFS="$defs" python - <<PY > /dev/null
import shutil
from paper_2309_16669_b200 import build as B
shutil.copy(B.build(), "$out")
PY
  echo "== [$defs]"
  AVB_LIB=$out timeout 300 python $BENCH 2>&1 | tail -3
  i=$((i+1))
done
