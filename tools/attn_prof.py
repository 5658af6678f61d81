"""Run the ViT-H local and global attention once each (for ncu)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import kernels as K  # noqa: E402


def run(kind, B):
    H, dh = 16, 80
    S, w, tile, p = (196, 14, 32, 2) if kind == "local" else (4096, 64, 128, 12)
    U = B * 25 if kind == "local" else B
    C = H * dh
    qkv = torch.randn(U * S, 3 * C, device="cuda").bfloat16()
    bh = torch.randn(H, S, w, device="cuda") * 0.5
    bw = torch.randn(H, S, w, device="cuda") * 0.5
    sp = torch.stack([torch.randperm(S, device="cuda") for _ in range(U)]).int()
    out = torch.empty(U * S, C, device="cuda", dtype=torch.bfloat16)
    for _ in range(2):
        K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=U, heads=H, sq=S, sk=S, dh=dh, bh=bh, bw=bw,
                      q_sp=sp, k_sp=sp, b_row=tile, b_col=tile, prefix=p, tau=dh ** -0.5, out=out)
    torch.cuda.synchronize()


which = sys.argv[1] if len(sys.argv) > 1 else "both"
if which in ("local", "both"):
    run("local", 8)
if which in ("global", "both"):
    run("global", 2)
