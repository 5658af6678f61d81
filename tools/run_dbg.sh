timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py tests/test_gpu_relpos.py -q -x -k "attention or attn or win or relpos" --timeout 120 2>&1 | tail -2
L=paper_2605_17633_b200/_lib
timeout 100 python tools/attn_bench.py local 64 2>&1 | grep default
cp $L/libzstripe_b200.so /tmp/new.so; cp $L/libzstripe_b200_old.so $L/libzstripe_b200.so
timeout 100 python tools/attn_bench.py local 64 2>&1 | grep default
cp /tmp/new.so $L/libzstripe_b200.so
timeout 600 python tools/density_sweep.py 16 2>&1 | grep window
