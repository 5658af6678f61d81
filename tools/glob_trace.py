"""Dump CTA 0's per-item timeline of the global attention kernel (ZS_GLOB_TRACE=1)."""
import ctypes
import math
import os
import sys
from pathlib import Path

os.environ["ZS_GLOB_TRACE"] = "1"
import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import _lib  # noqa: E402
from paper_2605_17633_b200 import kernels as K  # noqa: E402

B, H, dh, S, w, tile = 16, 16, 80, 4096, 64, 128
U = B
C = H * dh
qkv = torch.randn(U * S, 3 * C, device="cuda").bfloat16()
bh = torch.randn(H, S, w, device="cuda") * 0.5
bw = torch.randn(H, S, w, device="cuda") * 0.5
sp = torch.stack([torch.randperm(S, device="cuda") for _ in range(U)]).int()
out = torch.empty(U * S, C, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=U, heads=H, sq=S, sk=S, dh=dh, bh=bh, bw=bw,
                  q_sp=sp, k_sp=sp, b_row=tile, b_col=tile, prefix=12, tau=dh ** -0.5, out=out)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * (64 * 16 + 128))()
lib.zs_debug_glob_trace(buf, 64 * 16 + 128)
a = np.array(buf[:1024], dtype=np.int64).reshape(64, 16)
t2 = np.array(buf[1024:], dtype=np.int64).reshape(16, 8)
t0 = a[0, 6]
names = ["c0_s", "c0_p", "wg0_start", "wg1_start", "wg0_done", "wg1_done", "q+bq", "S0", "S1", "S2", "S3", "S4", "S5", "lastP", "epi_go", "PVlast"]
print("item " + " ".join(f"{n:>9s}" for n in names))
for k in range(12):
    print(f"{k:4d} " + " ".join(f"{(a[k, c] - t0) if a[k, c] else -1:9d}" for c in range(16)))

print("item 5, per chunk: S' issued | sees S | P written | PV issued | k_full ok | oh_full ok | OH written | OH start")
base = a[5, 6]
for j in range(16):
    if t2[j].any():
        print(f"  chunk {j:2d} (WG {j % 2}?): " + " ".join(f"{(v - base) if v else -1:7d}" for v in t2[j]))
