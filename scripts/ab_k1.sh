#!/usr/bin/env bash
# usage: scripts/ab_k1.sh outdir testlib lib1 lib2 ... : K1 tests on testlib, then same-box K1 A/B (bench_k1.py)
O=$1; T=$2; shift 2; mkdir -p $O
AVB_LIB=$T timeout 600 python -m pytest tests/test_k1_gpu.py tests/test_capi.py -q -x 2>&1 | tail -3 > $O/tests.txt
for rep in 1 2 3; do for L in "$@"; do echo "== $L" >> $O/ab.txt; AVB_LIB=$L timeout 300 python scripts/bench_k1.py >> $O/ab.txt 2>&1; done; done
