# Global attention: parity tests + A/B timing of library variants (ZS_AB_LIBS) on one B200.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py tests/test_gpu_relpos.py -q -x -k "attention or attn or glob or relpos" --timeout 120 2>&1 | tail -3
timeout 300 python tools/attn_ab.py global 16 2>&1 | tail -12
timeout 300 python tools/attn_ab.py global 16 stripes 2>&1 | tail -12
