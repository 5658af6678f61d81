"""Bisect the EPI 3 (TMA residual) GEMM epilogue: one case per process (argv: M N K mode)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import kernels as K  # noqa: E402

M, N, Kd, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn(M, Kd, device="cuda", generator=g).bfloat16()
w = (torch.randn(N, Kd, device="cuda", generator=g) / 20).bfloat16()
x = torch.randn(M, N, device="cuda", generator=g)
x0 = x.clone()
kw = {}
if mode == "mod":
    pos = torch.randn(64, N, device="cuda", generator=g)
    y = K.gemm(a, w, None, epi=K.EPI_F32_RESID, res=pos, res_mod=64)
    ref = a.float() @ w.float().T + pos.repeat((M + 63) // 64, 1)[:M]
else:
    y = K.gemm(a, w, None, epi=K.EPI_F32_RESID, out=x, res=x)
    ref = x0 + a.float() @ w.float().T
torch.cuda.synchronize()
print(sys.argv[1:], "rel", float((y - ref).norm() / ref.norm()))
