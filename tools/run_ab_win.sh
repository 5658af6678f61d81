timeout 100 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention_local or attention_window" --timeout 30 2>&1 | tail -2
timeout 100 python tools/attn_ab.py local 64 2>&1 | tail -7
