"""A/B timing of zs_gemm_bf16 from two library builds (same box, interleaved): ViT-H shapes."""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import _lib  # noqa: E402

libs = {name: ctypes.CDLL(str(Path(_lib.LIB_PATH).parent / f)) for name, f in
        [("new", "libzstripe_b200.so"), ("old", "libzstripe_b200_old.so")]}
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
    if kind == "fc1":
        lib.zs_gemm_bf16(1, P(a), C, P(w1), C, Mk, 4 * C, C, None, P(hid), 4 * C, None, 0, None, None, 0, None, st)
        return 2.0 * Mk * 4 * C * C
    lib.zs_gemm_bf16(2, P(hid), 4 * C, P(w2), 4 * C, Mk, C, 4 * C, None, P(x), C, P(x), C, P(keep), None, 0, None, st)
    return 2.0 * Mk * 4 * C * C


e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rnd in range(3):
    for kind in (sys.argv[2].split(",") if len(sys.argv) > 2 else ("qkv", "proj", "proj16", "fc1", "fc2")):
        for name, lib in libs.items():
            for _ in range(2):
                call(lib, kind)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(10):
                fl = call(lib, kind)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            print(f"round {rnd} {kind:5s} {name}: {ms:7.3f} ms {fl / ms / 1e9:7.1f} TF/s", flush=True)
