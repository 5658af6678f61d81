# attention kernels alone at the bench shapes (64 images), current build
timeout 300 python tools/attn_bench.py global 64 2>&1 | grep default
timeout 300 python tools/attn_bench.py local 64 2>&1 | grep default
timeout 600 python bench.py --no-cpu --no-dense --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['sm_mhz'])
print({k: (round(v['ms_per_step'],2), round(v.get('frac_bf16_peak',0),3), round(v.get('frac_hbm_peak',0),3)) for k,v in d['kernels'].items()})"
