timeout 200 python -m pytest tests/test_gpu_kernels.py -q -x -k "layernorm or ln" --timeout 60 2>&1 | tail -2
timeout 100 python tools/ln_ab.py 2>&1 | tail -6
