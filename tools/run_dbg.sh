# paired in-step A/B of the fc2 TMA residual epilogue (default) vs the LSU epilogue (ZS_G2_LSU=1)
for r in 1 2; do
  for v in tma lsu; do
    if [ $v = lsu ]; then export ZS_G2_LSU=1; else unset ZS_G2_LSU; fi
    timeout 600 python bench.py --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('$v', round(d['value'],1), d['clocks']['sm_mhz'], 'fc2', round(k['gemm_fc2']['ms_per_step'],2), 'fc1', round(k['gemm_fc1']['ms_per_step'],2), 'proj', round(k['gemm_proj']['ms_per_step'],2))"
  done
done
