# window attention at high density: sequential-tile mode vs the ping-pong fallback (ZS_WIN_NO_SEQ)
timeout 400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_api.py tests/test_gpu_encoder.py -q -x -k "window or local or attention or dense" --timeout 200 2>&1 | tail -2
for r in 0.7 0.8 0.9 1.0; do
  python - <<PY
import math, torch, sys
sys.path.insert(0, ".")
from paper_2605_17633_b200 import kernels as K
import os
B, H, dh, S, w, tile = 16, 16, 80, 196, 14, 32
U = B * 25; C = H * dh; r = $r
qkv = torch.randn(U * S, 3 * C, device="cuda").bfloat16()
bh = torch.randn(H, S, w, device="cuda") * 0.5; bw = torch.randn(H, S, w, device="cuda") * 0.5
sp = torch.stack([torch.randperm(S, device="cuda") for _ in range(U)]).int()
def run():
    return K.stripe_attn(qkv[:, :C], qkv[:, C:2*C], qkv[:, 2*C:], units=U, heads=H, sq=S, sk=S, dh=dh, bh=bh, bw=bw, q_sp=sp, k_sp=sp, b_row=tile, b_col=tile, prefix=math.floor(r*7), tau=dh**-0.5)
def t():
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): run()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / 10
a = t(); oa = run().float()
os.environ["ZS_WIN_NO_SEQ"] = "1"
b = t(); ob = run().float()
print(f"r={r}: seq {a:.3f} ms, fallback {b:.3f} ms, rel diff {((oa-ob).norm()/ob.norm()).item():.2e}")
PY
done
