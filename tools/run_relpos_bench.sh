timeout 900 python -m pytest tests -q -x -m gpu --timeout 200 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
for m in static sam; do
timeout 600 python bench.py --no-cpu --no-dense --rel-pos $m > gpurun_out/bench_$m.log 2>&1; tail -1 gpurun_out/bench_$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['rel_pos'], d['value'], d['ms_per_step'], d['e2e']['value'], d['gpu_launches']); [print(' ', k, round(v['ms_per_step'],2), v.get('tflops'), v.get('gbs')) for k,v in d['kernels'].items()]"
done
