# per-GPU batch of the 8-GPU split (8 images, CUDA-graph replay) and the SAM rel-pos mode, current build
for a in "--batch 8" "--batch 16" "--rel-pos sam"; do
  timeout 600 python bench.py $a --no-cpu --no-dense --steps 10 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a', round(d['value'],1), round(d['e2e']['value'],1), d['config'].get('cuda_graph'), d['gpu_launches'], d['clocks']['sm_mhz'])"
done
