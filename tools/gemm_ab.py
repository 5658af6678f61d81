"""A/B timing of zs_gemm_bf16 from two library builds (same box, interleaved): ViT-H shapes."""
import ctypes
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import _lib  # noqa: E402

libs = {name: ctypes.CDLL(str(Path(_lib.LIB_PATH).parent / f)) for name, f in
        [("new", os.environ.get("ZS_AB_NEW", "libzstripe_b200.so")), ("old", "libzstripe_b200_old.so")]}
for l in libs.values():
    l.zs_gemm_bf16.argtypes = _lib.SIGNATURES["zs_gemm_bf16"]
dev = "cuda"
M = (int(sys.argv[1]) if len(sys.argv) > 1 else 16) * 4900
C = 1280
a = torch.randn(M, C, device=dev).bfloat16()
wq = (torch.randn(3 * C, C, device=dev) / 36).bfloat16()
out = torch.empty(M, 3 * C, device=dev, dtype=torch.bfloat16)
wp = (torch.randn(C, C, device=dev) / 36).bfloat16()
x = torch.randn(M, C, device=dev)
Mk = M // 3
w1 = (torch.randn(4 * C, C, device=dev) / 36).bfloat16()
hid = torch.empty(Mk, 4 * C, device=dev, dtype=torch.bfloat16)
w2 = (torch.randn(C, 4 * C, device=dev) / 72).bfloat16()
keep = torch.randperm(M, device=dev)[:Mk].int()
st = torch.cuda.current_stream().cuda_stream
P = lambda t: t.data_ptr() if t is not None else None  # noqa: E731


def call(lib, kind):
    if kind == "qkv":
        lib.zs_gemm_bf16(0, P(a), C, P(wq), C, M, 3 * C, C, None, P(out), 3 * C, None, 0, None, None, 0, None, st)
        return 2.0 * M * 3 * C * C
    if kind == "proj":
        lib.zs_gemm_bf16(2, P(a), C, P(wp), C, M, C, C, None, P(x), C, P(x), C, None, None, 0, None, st)
        return 2.0 * M * C * C
    if kind == "proj16":  # same shape, bf16 output (no fp32 residual traffic)
        lib.zs_gemm_bf16(0, P(a), C, P(wp), C, M, C, C, None, P(out), C, None, 0, None, None, 0, None, st)
        return 2.0 * M * C * C
    if kind == "fc1nogelu":  # fc1 shape, plain bias epilogue
        lib.zs_gemm_bf16(0, P(a), C, P(w1), C, Mk, 4 * C, C, None, P(hid), 4 * C, None, 0, None, None, 0, None, st)
        return 2.0 * Mk * 4 * C * C
    if kind == "fc1":
        lib.zs_gemm_bf16(1, P(a), C, P(w1), C, Mk, 4 * C, C, None, P(hid), 4 * C, None, 0, None, None, 0, None, st)
        return 2.0 * Mk * 4 * C * C
    lib.zs_gemm_bf16(2, P(hid), 4 * C, P(w2), 4 * C, Mk, C, 4 * C, None, P(x), C, P(x), C, P(keep), None, 0, None, st)
    return 2.0 * Mk * 4 * C * C


e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
kinds = sys.argv[2].split(",") if len(sys.argv) > 2 else ("qkv", "proj", "proj16", "fc1", "fc2")
PAIRS = 24  # paired, finely interleaved samples: the power-capped clock drifts between rounds


def batch(lib, kind, n=5):
    e0.record()
    for _ in range(n):
        fl = call(lib, kind)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n, fl


for kind in kinds:
    for lib in libs.values():
        for _ in range(3):
            call(lib, kind)
    torch.cuda.synchronize()
    ratios, tn, to = [], [], []
    for i in range(PAIRS):
        order = ("new", "old") if i % 2 == 0 else ("old", "new")
        t = {}
        for name in order:
            t[name], fl = batch(libs[name], kind)
        ratios.append(t["new"] / t["old"])
        tn.append(t["new"])
        to.append(t["old"])
    ratios.sort()
    tn.sort()
    to.sort()
    med = ratios[len(ratios) // 2]
    print(f"{kind:9s} new/old median {med:.4f} (q1 {ratios[len(ratios) // 4]:.4f} q3 {ratios[3 * len(ratios) // 4]:.4f})"
          f"  new {tn[len(tn) // 2]:.3f} ms  old {to[len(to) // 2]:.3f} ms  new {fl / tn[len(tn) // 2] / 1e9:.0f} TF/s",
          flush=True)
