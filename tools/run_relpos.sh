timeout 40 python tools/relpos_debug.py 4096 2 2 0.3 unit 2>&1 | tail -2
timeout 40 python tools/relpos_debug.py 4096 2 2 0.3 fused 2>&1 | tail -2
timeout 400 python -m pytest tests/test_gpu_relpos.py -q -x --timeout 120 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x --timeout 120 -k "attention" 2>&1 | tail -2
timeout 100 python tools/attn_bench.py global 64 2>&1 | tail -3
