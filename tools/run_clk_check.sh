timeout 600 python bench.py --model vit_b --batch 1 --no-cpu --steps 10 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks'])"
timeout 600 python bench.py --no-cpu --no-dense --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks'])"
