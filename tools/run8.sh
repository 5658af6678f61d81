timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py -q -x -k "attn or attention" 2>&1 | tail -4
timeout 300 python tools/gpu_check.py 2>&1 | grep -E "perf|SUMMARY"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-dense > gpurun_out/bench8.log 2>&1
tail -1 gpurun_out/bench8.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); [print(k, round(v['ms_per_step'],2), v.get('tflops'), v.get('gbs')) for k,v in d['kernels'].items()]"
timeout 600 ncu --set full --import-source on -k regex:zs_attn -s 1 -c 1 -o gpurun_out/attn_local8 python tools/attn_prof.py local > /dev/null 2>&1
timeout 600 ncu --set full --import-source on -k regex:zs_gemm -s 4 -c 4 -o gpurun_out/gemm8 python tools/gemm_prof.py 8 > /dev/null 2>&1
