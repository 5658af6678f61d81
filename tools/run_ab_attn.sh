timeout 400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_relpos.py -q -x -k "attention or relpos" --timeout 120 2>&1 | tail -2
timeout 100 python tools/attn_ab.py global 64 2>&1 | tail -2
