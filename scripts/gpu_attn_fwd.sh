timeout 120 python scripts/dbg_bwd.py 2>/dev/null | cut -c1-150
timeout 300 python -m pytest tests/test_attn_gpu.py -x -q 2>&1 | tail -2
timeout 300 python scripts/bench_attn2.py 2>&1 | tail -1 | cut -c1-70
timeout 120 python scripts/trace_attn_bwd.py 2>&1 | tail -4
