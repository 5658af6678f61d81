timeout 240 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention or attn or win" --timeout 60 2>&1 | tail -3
