timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "concurrent" --timeout 200 2>&1 | tail -2
