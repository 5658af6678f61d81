"""Debug: one fused rel-pos attention call (S, units, heads from argv), synchronized and timed."""
import math
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import kernels as K  # noqa: E402

S, units, heads = (int(a) for a in sys.argv[1:4])
scale = float(sys.argv[4]) if len(sys.argv) > 4 else 0.3
mode = sys.argv[5] if len(sys.argv) > 5 else "fused"
dh, w = 80, int(math.isqrt(S))
tile = 32 if S <= 256 else 128
C = heads * dh
qkv = torch.randn(units * S, 3 * C, device="cuda").bfloat16()
rh = scale * torch.randn(2 * w - 1, dh, device="cuda")
rw = scale * torch.randn(2 * w - 1, dh, device="cuda")
sp = torch.stack([torch.randperm(S, device="cuda") for _ in range(units)]).int()
T = -(-S // tile)
t = time.time()
kw = dict(units=units, heads=heads, sq=S, sk=S, dh=dh, q_sp=sp, k_sp=sp, b_row=tile, b_col=tile,
          prefix=math.floor(0.4 * T), tau=dh ** -0.5)
if mode == "fused":
    o = K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], bh=None, bw=None, rel_pos=(rh, rw), **kw)
else:
    bh, bw = K.relpos_bias(qkv[:, :C], units=units, heads=heads, S=S, dh=dh, rel_pos_h=rh, rel_pos_w=rw, q_sp=sp)
    torch.cuda.synchronize()
    print("tables", float(bh.abs().max()), float(bw.abs().max()), flush=True)
    o = K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], bh=bh, bw=bw, **kw)
torch.cuda.synchronize()
print(f"S={S} units={units} heads={heads} scale={scale} {mode}: ok {time.time() - t:.3f}s finite={bool(o.float().isfinite().all())}",
      flush=True)
