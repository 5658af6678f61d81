timeout 120 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention_global or many_items" --timeout 40 2>&1 | tail -3
timeout 100 python tools/attn_bench.py global 64 2>&1 | tail -3
timeout 100 python tools/glob_trace.py 2>&1 | tail -14
