"""BASELINE config 5: density sweep 0.2-1.0 on ViT-H windowed (14x14) and global attention layers
and the RC-MLP, each kernel isolated and timed against the dense library kernels on the same GPU.

    python tools/density_sweep.py [B] [--out profiles/round1_density_sweep.json]

Per density d (attention r = d, MLP keep = d), ViT-H (C 1280, 16 heads, dh 80), B images:
  window attention  our stripe kernel vs F.scaled_dot_product_attention (dense, materialised
                    decomposed rel-pos bias) over all 196 tokens of every (window, head)
  global attention  same over 4096 tokens per (image, head)
  RC-MLP            LN-gather + fc1(GELU) + fc2(scatter-add) on the kept rows vs a dense
                    cuBLAS MLP (F.linear, GELU) over all rows
Effective TFLOP/s count only the work the static schedule requires (4*dh*E for attention,
16*R*C^2 for the MLP); the dense baselines are credited their full dense FLOPs.
CUDA-event timing, 2 warm-up + 5 timed launches, inputs larger than L2.
"""
import json
import math
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import kernels as K  # noqa: E402
from paper_2605_17633_b200.config import RouterConfig  # noqa: E402
from paper_2605_17633_b200.dense import dense_bias  # noqa: E402
from paper_2605_17633_b200.encoder import attention_elements  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 16
OUT = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
H, dh, C = 16, 80, 1280
dev = "cuda"


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def attn_case(kind, d):
    S, w, tile = (196, 14, 32) if kind == "window" else (4096, 64, 128)
    U = B * 25 if kind == "window" else B
    T = -(-S // tile)
    p = math.floor(d * T)
    g = torch.Generator(device=dev).manual_seed(0)
    qkv = torch.randn(U * S, 3 * C, device=dev, generator=g).bfloat16()
    bh = torch.randn(H, S, w, device=dev, generator=g) * 0.5
    bw = torch.randn(H, S, w, device=dev, generator=g) * 0.5
    sp = torch.argsort(torch.rand(U, S, device=dev, generator=g), dim=1).int().contiguous()
    out = torch.empty(U * S, C, device=dev, dtype=torch.bfloat16)
    ms = timed(lambda: K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=U, heads=H, sq=S, sk=S, dh=dh,
                                     bh=bh, bw=bw, q_sp=sp, k_sp=sp, b_row=tile, b_col=tile, prefix=p,
                                     tau=dh ** -0.5, out=out))
    E = attention_elements(S, tile, p)
    eff = 4.0 * dh * E * U * H
    # dense: SDPA with the materialised bias over every (unit, head)
    bias = dense_bias(bh, bw)[None]
    q = qkv.view(U, S, 3, H, dh).permute(2, 0, 3, 1, 4)
    chunk = max(1, min(U, (8 << 30) // (H * S * S * 2 * 4)))  # bound the expanded-mask memory

    def dense():
        for u0 in range(0, U, chunk):
            u1 = min(U, u0 + chunk)
            F.scaled_dot_product_attention(q[0, u0:u1], q[1, u0:u1], q[2, u0:u1],
                                           attn_mask=bias.expand(u1 - u0, -1, -1, -1))
    ms_d = timed(dense)
    full = 4.0 * dh * S * S * U * H
    return dict(kind=kind, density=d, prefix_tiles=p, achieved_density=E / (S * S), units=U, ms=ms,
                eff_tflops=eff / ms / 1e9, dense_ms=ms_d, dense_tflops=full / ms_d / 1e9, speedup=ms_d / ms)


def mlp_case(d):
    S, U = 196, B * 25
    R = U * S
    Kc = RouterConfig(d, "identity").keep_count(S)
    g = torch.Generator(device=dev).manual_seed(1)
    x = torch.randn(R, C, device=dev, generator=g)
    keep, offs = K.unit_span_rows(U, S, 0, Kc, None, dev)
    n = offs[U:U + 1]
    lg, lb = torch.ones(C, device=dev), torch.zeros(C, device=dev)
    w1 = (torch.randn(4 * C, C, device=dev, generator=g) / 36).bfloat16()
    w2 = (torch.randn(C, 4 * C, device=dev, generator=g) / 72).bfloat16()
    b1, b2 = torch.zeros(4 * C, device=dev), torch.zeros(C, device=dev)
    ws = torch.empty(U * Kc * 5 * C, device=dev, dtype=torch.bfloat16)
    ms = timed(lambda: K.rc_mlp(x, keep, ln_g=lg, ln_b=lb, w1=w1, b1=b1, w2=w2, b2=b2, n_keep_dev=n, ws=ws))
    eff = 16.0 * U * Kc * C * C
    xb = x.bfloat16()

    def dense():
        h = F.layer_norm(xb.float(), (C,), lg, lb, 1e-6).bfloat16()
        return F.linear(F.gelu(F.linear(h, w1)), w2)
    ms_d = timed(dense)
    return dict(kind="rc_mlp", density=d, keep_rows=U * Kc, rows=R, ms=ms, eff_tflops=eff / ms / 1e9, dense_ms=ms_d,
                dense_tflops=16.0 * R * C * C / ms_d / 1e9, speedup=ms_d / ms)


res = {"batch": B, "model": "sam_vit_h", "cases": []}
for d in (0.2, 0.3, 0.4, 0.5, 0.6, 0.7, 0.8, 0.9, 1.0):
    for case in (lambda: attn_case("window", d), lambda: attn_case("global", d), lambda: mlp_case(d)):
        r = case()
        res["cases"].append(r)
        print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
if OUT:
    Path(OUT).write_text(json.dumps(res, indent=1) + "\n")
