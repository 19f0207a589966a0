#!/usr/bin/env bash
# usage: scripts/ab_attn.sh outdir testlib lib1 lib2 ... : attention tests on testlib, then same-box K4/K5 A/B
O=$1; T=$2; shift 2; mkdir -p $O
AVB_LIB=$T timeout 600 python -m pytest tests/test_attn_gpu.py tests/test_bench_shapes_gpu.py -q -x 2>&1 | tail -3 > $O/tests.txt
for rep in 1 2; do for L in "$@"; do echo "== $L" >> $O/ab.txt; AVB_LIB=$L timeout 300 python scripts/bench_attn_bwd.py >> $O/ab.txt 2>&1; done; done
