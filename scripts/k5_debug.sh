#!/usr/bin/env bash
# K5 v2 failure bisection on the GPU box: debug builds into separate library files.
set -u
build() {  # $1 = out lib, $2 = defines
  AVB_NVCC_DEFS="$2" python - <<PY
import os, shutil
from paper_2309_16669_b200 import build as B
lib = B.build()
shutil.copy(lib, "$1")
PY
}
build /tmp/lib_knobs.so "-DAVB_DEBUG_KNOBS"
build /tmp/lib_serial.so "-DAVB_DEBUG_KNOBS -DK5_DBG_SERIAL"
for lib in /tmp/lib_knobs.so /tmp/lib_serial.so; do
  for grid in 1 8 148; do
    echo "== $lib grid=$grid"
    AVB_LIB=$lib AVB_ATTN_BWD_GRID=$grid timeout 60 python scripts/repro_bwd.py 64 128 12 0 0 2>&1 | grep -i "error\|^d" | head -2
  done
done
