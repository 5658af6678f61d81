"""Compare the split-chunk global kernel with the generic one on small shapes (debug)."""
import os
import sys

import torch

sys.path.insert(0, "/root/repo")
from paper_2605_17633_b200 import kernels as K  # noqa: E402


def run(U, H, S, dh, w, prefix, generic):
    if generic:
        os.environ["ZS_ATTN_NO_GLOB"] = "1"
    else:
        os.environ.pop("ZS_ATTN_NO_GLOB", None)
    C = H * dh
    g = torch.Generator().manual_seed(0)
    qkv = torch.randn(U * S, 3 * C, generator=g).bfloat16().cuda()
    bh = (0.5 * torch.randn(H, S, w, generator=g)).cuda()
    bw = (0.5 * torch.randn(H, S, w, generator=g)).cuda()
    sp = torch.stack([torch.randperm(S, generator=g) for _ in range(U)]).int().cuda()
    out = K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=U, heads=H, sq=S, sk=S, dh=dh, bh=bh,
                        bw=bw, q_sp=sp, k_sp=sp, b_row=128, b_col=128, prefix=prefix, tau=dh ** -0.5)
    torch.cuda.synchronize()
    return out.float()


for (U, H, S, dh, w, p) in [(1, 1, 4096, 64, 64, 6), (2, 2, 4096, 64, 64, 6), (1, 1, 4096, 80, 64, 12)]:
    a = run(U, H, S, dh, w, p, False)
    b = run(U, H, S, dh, w, p, True)
    err = ((a - b).norm() / b.norm()).item()
    rows = ((a - b).abs().amax(1) > 0.05).nonzero().flatten()
    print(U, H, S, dh, p, "rel", err, "bad rows", rows.numel(), rows[:10].tolist(), flush=True)
