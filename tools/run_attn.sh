timeout 200 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention" --timeout 60 2>&1 | tail -2
timeout 100 python tools/attn_bench.py both 64 2>&1 | grep default
