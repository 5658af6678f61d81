timeout 120 python tools/gemm2_quick.py 2>&1 | tail -2
timeout 120 python tools/gelu_bench.py 2>&1 | tail -3
timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-dense > gpurun_out/bench16.log 2>&1
tail -1 gpurun_out/bench16.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved']); [print(k, round(v['ms_per_step'],2), v.get('tflops'), v.get('gbs')) for k,v in d['kernels'].items()]"
