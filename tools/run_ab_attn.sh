timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention_local or attention_window or row_map" --timeout 120 2>&1 | tail -2
timeout 100 python tools/attn_ab.py local 64 rows 2>&1 | tail -7
