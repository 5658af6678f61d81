import sys, torch, math
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import kernels as K
dev = "cuda"
for M, N, K_ in [(300, 512, 256), (4900, 3840, 1280), (1000, 768, 5120)]:
    a = torch.randn(M, K_, device=dev).bfloat16()
    w = (torch.randn(N, K_, device=dev) / math.sqrt(K_)).bfloat16()
    b = torch.randn(N, device=dev)
    y = K.gemm(a, w, b)
    torch.cuda.synchronize()
    ref = a.float() @ w.float().T + b
    print(M, N, K_, "rel", ((y.float() - ref).norm() / ref.norm()).item(), flush=True)
M, N, K_ = 8 * 4900, 3840, 1280
a = torch.randn(M, K_, device=dev).bfloat16(); w = torch.randn(N, K_, device=dev).bfloat16(); out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
for _ in range(3): K.gemm(a, w, None, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): K.gemm(a, w, None, out=out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("qkv", ms, 2 * M * N * K_ / ms / 1e9, "TF/s")
x = torch.randn(M, 1280, device=dev); wp = torch.randn(1280, 1280, device=dev).bfloat16(); o = a
for _ in range(3): K.gemm(o, wp, None, epi=2, out=x, res=x)
torch.cuda.synchronize(); e0.record()
for _ in range(10): K.gemm(o, wp, None, epi=2, out=x, res=x)
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1) / 10
print("proj", ms, 2 * M * 1280 * 1280 / ms / 1e9, "TF/s")
