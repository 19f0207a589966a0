python - <<'PY'
import torch, ctypes
print("SMs", torch.cuda.get_device_properties(0).multi_processor_count)
PY
timeout 240 python -m pytest tests/test_gemm_gpu.py -x -q 2>&1 | tail -2
timeout 240 python scripts/bench_gemm.py 2>&1 | tail -13 | cut -c1-140
