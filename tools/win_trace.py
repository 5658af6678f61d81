"""Dump CTA 0's per-item timeline of the window attention kernel (ZS_WIN_TRACE=1)."""
import ctypes
import math
import os
import sys
from pathlib import Path

os.environ["ZS_WIN_TRACE"] = "1"
import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import _lib  # noqa: E402
from paper_2605_17633_b200 import kernels as K  # noqa: E402

B, H, dh, S, w, tile = 64, 16, 80, 196, 14, 32
r = float(sys.argv[1]) if len(sys.argv) > 1 else 0.4
U = B * 25
C = H * dh
qkv = torch.randn(U * S, 3 * C, device="cuda").bfloat16()
bh = torch.randn(H, S, w, device="cuda") * 0.5
bw = torch.randn(H, S, w, device="cuda") * 0.5
sp = torch.stack([torch.randperm(S, device="cuda") for _ in range(U)]).int()
out = torch.empty(U * S, C, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=U, heads=H, sq=S, sk=S, dh=dh, bh=bh, bw=bw,
                  q_sp=sp, k_sp=sp, b_row=tile, b_col=tile, prefix=math.floor(r * 7), tau=dh ** -0.5, out=out)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * (64 * 32))()
lib.zs_debug_win_trace(buf, 64 * 32)
a = np.array(buf, dtype=np.int64).reshape(64, 32)
t0 = a[0, 0]
names = {0: "ld_qk", 1: "ld_v", 2: "S_A", 3: "PV_B-", 4: "S_B", 5: "PV_A", 8: "bias_op",
         18: "A_s", 19: "A_emit", 20: "A_epi", 21: "A_pfull",
         26: "B_s", 27: "B_emit", 28: "B_epi", 29: "B_pfull"}
cols = sorted(names)
print("item " + " ".join(f"{names[c]:>8s}" for c in cols))
for k in range(24):
    print(f"{k:4d} " + " ".join(f"{(a[k, c] - t0) if a[k, c] else -1:8d}" for c in cols))
