"""ViT-H GEMM shapes once each (for ncu): QKV, proj (fp32 residual), fc1 (GELU), fc2 (scatter-add)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import kernels as K  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
C = 1280
R = B * 4900
dev = "cuda"
h = torch.randn(R, C, device=dev).bfloat16()
wqkv = (torch.randn(3 * C, C, device=dev) / 36).bfloat16()
bqkv = torch.zeros(3 * C, device=dev)
wp = (torch.randn(C, C, device=dev) / 36).bfloat16()
x = torch.randn(R, C, device=dev)
n_keep = int(R * 0.34)
hid = torch.randn(n_keep, 4 * C, device=dev).bfloat16()
w1 = (torch.randn(4 * C, C, device=dev) / 36).bfloat16()
w2 = (torch.randn(C, 4 * C, device=dev) / 72).bfloat16()
keep = torch.randperm(R, device=dev)[:n_keep].int()
for _ in range(2):
    qkv = K.gemm(h, wqkv, bqkv)                                               # QKV
    K.gemm(qkv[:, :C].contiguous(), wp, bqkv[:C], epi=K.EPI_F32_RESID, out=x, res=x)  # proj
    K.gemm(h[:n_keep], w1, None, epi=K.EPI_BF16_GELU)                       # fc1
    K.gemm(hid, w2, None, epi=K.EPI_F32_RESID, out=x, res=x, row_map=keep)  # fc2
torch.cuda.synchronize()
