for b in 8 64; do
timeout 600 python bench.py --batch $b --no-cpu --no-dense --steps 10 --warmup 5 2>/tmp/err.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$b', round(d['value'],1), round(d['e2e']['value'],1), d['config']['cuda_graph'], d['gpu_launches'], d['clocks']['sm_mhz'])" || tail -5 /tmp/err.log
done
