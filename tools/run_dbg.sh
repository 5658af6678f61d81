timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or mlp" --timeout 120 2>&1 | tail -2
timeout 400 python tools/gemm_ab.py 48 proj,fc2 2>&1 | tail -2
