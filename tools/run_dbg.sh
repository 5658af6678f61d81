timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or mlp" --timeout 100 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_encoder.py tests/test_gpu_api.py -q -x --timeout 300 2>&1 | tail -3
timeout 300 python tools/gemm_ab.py 48 proj,fc2 2>&1 | tail -2
