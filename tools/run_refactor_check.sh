# encoder parity tests + default bench (spatial-resident residual stream)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_encoder.py tests/test_gpu_api.py -q -x --timeout 300 2>&1 | tail -3
timeout 600 python bench.py --no-cpu > gpurun_out/bench_refactor.log 2>&1; tail -1 gpurun_out/bench_refactor.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'e2e', d['e2e']['value'], 'clk', d['clocks'], 'launches', d['gpu_launches'])
print({k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
