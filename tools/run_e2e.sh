timeout 120 python tools/gemm2_quick.py 2>&1 | tail -6
timeout 900 python -m pytest tests -q -x -m gpu --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d.get('dense_baseline',{}) and d['dense_baseline']['value'], d['roofline']['achieved']); [print(k, round(v['ms_per_step'],2), v.get('tflops'), v.get('gbs')) for k,v in d['kernels'].items()]"
