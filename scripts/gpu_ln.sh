timeout 300 python -m pytest tests/test_model_gpu.py tests/test_clip_gpu.py -x -q 2>&1 | tail -3
bash scripts/gpu_train3.sh
