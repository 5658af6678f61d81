timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py -q -x -k "attention or attn or win" --timeout 120 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
