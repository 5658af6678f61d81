# window kernel timeline (trace build) + untraced timing
timeout 100 python tools/attn_bench.py local 64 2>&1 | grep default
ZS_BUILD_FLAGS=-DZS_KERNEL_TRACE timeout 200 python -m paper_2605_17633_b200.build --force > /dev/null 2>&1
timeout 60 python tools/win_trace.py 0.4 > gpurun_out/wintrace.txt 2>&1; tail -26 gpurun_out/wintrace.txt
