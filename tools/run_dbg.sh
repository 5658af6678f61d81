timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "global or many_items" --timeout 120 2>&1 | tail -2
timeout 300 python tools/attn_ab.py global 16 stripes 2>&1 | grep -A1 median
