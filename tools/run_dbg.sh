timeout 240 python -m pytest tests/test_gpu_kernels.py -q -x -k "global or many_items or o_rows or rows" --timeout 60 2>&1 | tail -3
timeout 200 python tools/attn_ab.py global 16 stripes 2>&1 | grep -A1 median
