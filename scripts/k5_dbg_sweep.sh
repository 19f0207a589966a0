#!/usr/bin/env bash
# K5 trace-build experiment sweep: per-step cycles with parts of the compute-warp work disabled
# (AVB_ATTN_DBG bits, see BwdArgs::dbg).  Run on the GPU box; builds the trace library in place.
AVB_NVCC_DEFS=-DAVB_ATTN_TRACE_HOOKS python -m paper_2309_16669_b200.build > /dev/null
for d in ${@:-0 1 2 4 8 16 6 14 30 31}; do
  echo "== AVB_ATTN_DBG=$d"
  AVB_ATTN_DBG=$d TRACE_STEPS=40 python scripts/trace_attn_bwd.py 2>&1 | grep -E "bwd ms|mean cycles|^40 "
done
