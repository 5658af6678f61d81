timeout 60 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention_local or attention_window" --timeout 30 2>&1 | tail -3
timeout 60 python tools/attn_bench.py local 64 2>&1 | tail -8
timeout 60 python tools/win_trace.py 0.4 2>&1 | tail -12
