for D in 0 5 0 13 0; do echo "dbg=$D $(AVB_ATTN_DBG=$D timeout 100 python scripts/bench_attn2.py 2>&1 | tail -1 | cut -c1-60)"; done
nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu --format=csv
