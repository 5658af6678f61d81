# api bench-schema test, window attention timing + timeline (trace build on the box) on one B200
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_api.py -q -x -k "bench_schema" 2>&1 | tail -2
timeout 100 python tools/attn_bench.py local 64 2>&1 | grep default
ZS_BUILD_FLAGS=-DZS_KERNEL_TRACE timeout 200 python -m paper_2605_17633_b200.build --force > /dev/null 2>&1
timeout 60 python tools/win_trace.py 0.4 2>&1 | tail -26
