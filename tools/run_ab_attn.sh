timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention_global or large_bias" --timeout 120 2>&1 | tail -2
timeout 100 python tools/attn_ab.py global 64 2>&1 | tail -2
cp paper_2605_17633_b200/_lib/libzstripe_b200_p8.so paper_2605_17633_b200/_lib/libzstripe_b200.so
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "attention_global or large_bias" --timeout 120 2>&1 | tail -2
timeout 100 python tools/attn_ab.py global 64 2>&1 | tail -2
