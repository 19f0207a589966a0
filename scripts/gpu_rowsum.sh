set -x
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_model_gpu.py tests/test_clip_gpu.py -x -q 2>&1 | tail -5
bash scripts/gpu_train3.sh
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/train_full.json
python -c "import json; d=json.load(open('gpurun_out/train_full.json')); print(d['value'], d['e2e'], d['gpu_launches'], d['clocks'])"
