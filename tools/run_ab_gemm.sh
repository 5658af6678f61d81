timeout 200 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm" --timeout 60 2>&1 | tail -2
timeout 200 python tools/gemm_ab.py 48 proj,proj16,fc2 2>&1 | tail -12
