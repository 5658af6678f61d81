# TMA residual epilogue (EPI 3) vs HEAD's LSU epilogue: GEMM tests, then paired A/B on proj / fc2
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "gemm or mlp" --timeout 100 2>&1 | tail -3
timeout 300 python tools/gemm_ab.py 48 proj,fc2 2>&1 | tail -4
ZS_G2_LSU=1 timeout 300 python tools/gemm_ab.py 48 proj 2>&1 | tail -2
