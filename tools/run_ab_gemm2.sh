timeout 200 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or mlp" --timeout 60 2>&1 | tail -2
timeout 300 python tools/gemm_ab.py 48 fc1,qkv,fc1nogelu 2>&1 | tail -3
