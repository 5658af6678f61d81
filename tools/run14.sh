timeout 900 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --no-dense > gpurun_out/bench14.log 2>&1
tail -1 gpurun_out/bench14.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['achieved']); [print(k, round(v['ms_per_step'],2), v.get('tflops'), v.get('gbs')) for k,v in d['kernels'].items()]"
timeout 600 ncu --set full --import-source on -k regex:zs_attn -s 1 -c 1 -o gpurun_out/attn_global14 python tools/attn_prof.py global > /dev/null 2>&1
