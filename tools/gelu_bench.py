import sys, torch, math
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import kernels as K
dev = "cuda"
M, N, K_ = 107000, 5120, 1280
a = torch.randn(M, K_, device=dev).bfloat16(); w = (torch.randn(N, K_, device=dev) / 36).bfloat16(); b = torch.zeros(N, device=dev)
out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
for epi in (0, 1):
    for _ in range(3): K.gemm(a, w, b, epi=epi, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): K.gemm(a, w, b, epi=epi, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print("epi", epi, ms, 2 * M * N * K_ / ms / 1e9, "TF/s")
y = K.gemm(a[:1000], w, b, epi=1); ref = torch.nn.functional.gelu(a[:1000].float() @ w.float().T + b)
print("gelu rel", ((y.float() - ref).norm() / ref.norm()).item())
