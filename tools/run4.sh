set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py -q -x -k "attn or attention" 2>&1 | tail -15 > gpurun_out/pytest_attn.log
cat gpurun_out/pytest_attn.log
timeout 300 python tools/gpu_check.py 2>&1 | grep -E "attn|SUMMARY" > gpurun_out/gpu_check4.log
cat gpurun_out/gpu_check4.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-dense > gpurun_out/bench4.log 2>&1
tail -1 gpurun_out/bench4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); [print(k, round(v['ms_per_step'],2), v.get('tflops'), v.get('gbs')) for k,v in d['kernels'].items()]"
