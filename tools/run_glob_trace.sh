# global attention timeline (trace build on the box) on one B200
ZS_BUILD_FLAGS=-DZS_KERNEL_TRACE timeout 200 python -m paper_2605_17633_b200.build --force > /dev/null 2>&1
timeout 100 python tools/glob_trace.py > gpurun_out/globtrace.txt 2>&1; tail -30 gpurun_out/globtrace.txt
