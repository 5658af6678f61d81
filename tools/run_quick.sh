timeout 600 python -m pytest tests -q -x -m gpu -k "sobel or order or saliency or rank" --timeout 200 2>&1 | tail -2
timeout 600 python bench.py --no-cpu --no-dense --no-e2e > gpurun_out/bench_q.log 2>&1; tail -1 gpurun_out/bench_q.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'], d['kernels']['ordering'])"
