# BASELINE configs 2 and 3 on one B200 (config 4 is the default bench, config 5 the density sweep)
for args in "--model vit_b --batch 1" "--model vit_b --batch 1 --graph on" "--model vit_l --batch 8 --density 0.4" "--model vit_l --batch 8 --density 0.3" "--model vit_h --batch 64"; do
  timeout 600 python bench.py $args --no-cpu --steps 10 --warmup 5 2>/dev/null | tail -1 > gpurun_out/cfg.json
  cat gpurun_out/cfg.json >> gpurun_out/configs.jsonl
  python -c "import json; d=json.load(open('gpurun_out/cfg.json')); print('$args', round(d['value'],1), round(d['e2e']['value'],1), round(d['dense_baseline']['value'],1), d['gpu_launches'], d['clocks']['sm_mhz'])"
done
