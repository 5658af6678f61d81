timeout 400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_relpos.py -q -x -k "attention or relpos" --timeout 60 2>&1 | tail -2
