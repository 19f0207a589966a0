#!/usr/bin/env bash
# ncu evidence for profiles/<round>/ (run on the GPU box; 1 GPU; never wrap a multi-rank command).
set -u
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O
NCU="ncu --set full --import-source on --clock-control none"
$NCU -k regex:attn_bwd_kernel -s 1 -c 1 -o $O/attn_bwd python scripts/prof_attn.py > $O/ncu_attn_bwd.log 2>&1
$NCU -k regex:attn_fwd_kernel -s 2 -c 1 -o $O/attn_fwd python scripts/prof_attn.py > $O/ncu_attn_fwd.log 2>&1
$NCU -k regex:k1v4 -s 3 -c 1 -o $O/k1 python scripts/bench_k1.py > $O/ncu_k1.log 2>&1
$NCU -k regex:gemm_kernel -s 3 -c 3 -o $O/gemm python scripts/prof_gemm.py > $O/ncu_gemm.log 2>&1
$NCU -k regex:ln_fwd -s 3 -c 1 -o $O/ln python scripts/bench_ln.py > $O/ncu_ln.log 2>&1
$NCU -k regex:ln_bwd_kernel -s 3 -c 1 -o $O/ln_bwd python scripts/bench_ln.py > $O/ncu_ln_bwd.log 2>&1
# every launch of the default bench command (cold-cache, serialised: compare shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-breakdown > $O/launches_bench.log 2>&1
ls -la $O
