# Window attention: parity tests + A/B timing of library variants (ZS_AB_LIBS) on one B200.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py tests/test_gpu_relpos.py -q -x -k "attention or attn or win or relpos" --timeout 120 2>&1 | tail -2
timeout 300 python tools/attn_ab.py local 64 2>&1 | tail -6
timeout 300 python tools/attn_ab.py local 64 rows 2>&1 | tail -6
