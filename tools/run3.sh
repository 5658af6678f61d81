set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py -q -x -k "attn or attention" 2>&1 | tail -15 > gpurun_out/pytest_attn.log
timeout 300 python tools/gpu_check.py 2>&1 | grep -E "PASS|FAIL|SUMMARY" > gpurun_out/gpu_check3.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-dense > gpurun_out/bench3.log 2>&1
cat gpurun_out/pytest_attn.log gpurun_out/gpu_check3.log; tail -3 gpurun_out/bench3.log
