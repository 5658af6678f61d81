"""Time the stripe-sort attention kernels at ViT-H shapes (CUDA events, inputs > L2).

    python tools/attn_bench.py [local|global|both] [B]

Prints per-launch time, effective TFLOP/s (4*dh*E, skipped tiles not counted) and
algorithmic HBM GB/s (Q, K, V, O bf16 + bias tables), for the default kernel and,
for windows, the previous ping-pong kernel (ZS_ATTN_NO_WIN=1).
"""
import math
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import kernels as K  # noqa: E402
from paper_2605_17633_b200.encoder import attention_elements  # noqa: E402


def run(kind, B, r=0.4, reps=10):
    H, dh = 16, 80
    S, w, tile = (196, 14, 32) if kind == "local" else (4096, 64, 128)
    T = -(-S // tile)
    p = math.floor(r * T)
    U = B * 25 if kind == "local" else B
    C = H * dh
    qkv = torch.randn(U * S, 3 * C, device="cuda").bfloat16()
    bh = torch.randn(H, S, w, device="cuda") * 0.5
    bw = torch.randn(H, S, w, device="cuda") * 0.5
    sp = torch.stack([torch.randperm(S, device="cuda") for _ in range(U)]).int()
    out = torch.empty(U * S, C, device="cuda", dtype=torch.bfloat16)
    E = attention_elements(S, tile, p)
    flops = 4.0 * dh * E * U * H
    byts = U * H * 4 * S * dh * 2 + H * 2 * S * w * 4

    def call():
        K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=U, heads=H, sq=S, sk=S, dh=dh, bh=bh, bw=bw,
                      q_sp=sp, k_sp=sp, b_row=tile, b_col=tile, prefix=p, tau=dh ** -0.5, out=out)

    variants = [("default", None)]
    if kind == "local":
        variants.append(("pingpong", "ZS_ATTN_NO_WIN"))
    for name, env in variants:
        if env:
            os.environ[env] = "1"
        for _ in range(2):
            call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        if env:
            del os.environ[env]
        print(f"{kind:6s} B={B} r={r} {name:9s} {ms:8.3f} ms  {flops / ms / 1e9:7.1f} TF/s  {byts / ms / 1e6:7.1f} GB/s",
              flush=True)


which = sys.argv[1] if len(sys.argv) > 1 else "both"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
prof = "prof" in sys.argv  # one timed launch per kernel (for ncu)
if which in ("local", "both"):
    for r in ((0.4,) if prof else (0.2, 0.4, 0.6)):
        run("local", B, r, reps=1 if prof else 10)
if which in ("global", "both"):
    run("global", B, reps=1 if prof else 10)
