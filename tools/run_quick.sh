timeout 300 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_encoder.py -q -x -k "patchify or sam_frame or graph" --timeout 200 2>&1 | tail -2
timeout 600 python bench.py --no-cpu --no-dense --no-e2e > gpurun_out/bench_q.log 2>&1; tail -1 gpurun_out/bench_q.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python bench.py --profile --steps 1 --warmup 1 > /dev/null 2>&1; echo "ncu rc=$?"
