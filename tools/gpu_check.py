"""Quick on-GPU kernel checks (developer tool; the real gates live in tests/)."""

import math
import sys
import time
import traceback
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2605_17633_b200 import kernels as K  # noqa: E402
from oracle import zs_oracle as O  # noqa: E402

dev = torch.device("cuda:0")
results = []


def check(name):
    def deco(fn):
        t0 = time.time()
        try:
            msg = fn()
            torch.cuda.synchronize()
            results.append((name, "PASS", msg))
        except Exception as e:  # noqa: BLE001
            results.append((name, "FAIL", f"{type(e).__name__}: {e}"))
            traceback.print_exc()
        print(f"[{results[-1][1]}] {name}: {results[-1][2]}  ({time.time() - t0:.1f}s)", flush=True)
        return fn

    return deco


def rel(a, b):
    a = a.float()
    b = b.float()
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


@check("gemm_bf16_small")
def _():
    torch.manual_seed(0)
    out = []
    for M, N, K_ in [(300, 512, 256), (128, 256, 64), (1000, 768, 1280), (77, 3840, 1280)]:
        a = torch.randn(M, K_, device=dev).bfloat16()
        w = torch.randn(N, K_, device=dev).bfloat16()
        b = torch.randn(N, device=dev)
        y = K.gemm(a, w, b)
        ref = a.float() @ w.float().T + b
        e = rel(y, ref)
        out.append(f"{M}x{N}x{K_}:{e:.2e}")
        assert e < 1e-2, out
    return " ".join(out)


@check("gemm_gelu_resid_rowmap")
def _():
    torch.manual_seed(1)
    M, N, K_ = 333, 768, 512
    a = torch.randn(M, K_, device=dev).bfloat16()
    w = torch.randn(N, K_, device=dev).bfloat16() * 0.05
    b = torch.randn(N, device=dev)
    y = K.gemm(a, w, b, epi=K.EPI_BF16_GELU)
    ref = torch.nn.functional.gelu(a.float() @ w.float().T + b)
    e1 = rel(y, ref)
    x = torch.randn(500, N, device=dev)
    x0 = x.clone()
    rm = torch.randperm(500, device=dev)[:M].int()
    zr = (torch.rand(M, device=dev) < 0.2).to(torch.uint8)
    K.gemm(a, w, b, epi=K.EPI_F32_RESID, out=x, res=x, row_map=rm, zero_rows=zr)
    ref2 = x0.clone()
    upd = x0[rm.long()] + a.float() @ w.float().T + b
    upd[zr.bool()] = 0
    ref2[rm.long()] = upd
    e2 = rel(x, ref2)
    mdev = torch.tensor([200], device=dev, dtype=torch.int32)
    y3 = torch.zeros(M, N, device=dev, dtype=torch.bfloat16)
    K.gemm(a, w, b, out=y3, m_dev=mdev)
    e3 = rel(y3[:200], a[:200].float() @ w.float().T + b)
    z3 = y3[200:].float().abs().max().item()
    assert e1 < 1e-2 and e2 < 1e-2 and e3 < 1e-2 and z3 == 0, (e1, e2, e3, z3)
    return f"gelu {e1:.2e} resid {e2:.2e} mdev {e3:.2e}"


def attn_case(units, heads, S, dh, w, tile, r, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    C = heads * dh
    qkv = (torch.randn(units * S, 3 * C, generator=g)).bfloat16().to(dev)
    bh = (0.5 * torch.randn(heads, S, w, generator=g)).to(dev)
    bw = (0.5 * torch.randn(heads, S, w, generator=g)).to(dev)
    sp = torch.stack([torch.randperm(S, generator=g) for _ in range(units)]).int().to(dev)
    T = -(-S // tile)
    p = math.floor(r * T)
    tau = 1.0 / math.sqrt(dh)
    out = K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=units, heads=heads, sq=S, sk=S, dh=dh,
                        bh=bh, bw=bw, q_sp=sp, k_sp=sp, b_row=tile, b_col=tile, prefix=p, tau=tau)
    torch.cuda.synchronize()
    errs = []
    qkvf = qkv.float().cpu().numpy()
    for u in range(min(units, 2)):
        for h in range(heads):
            rows = slice(u * S, (u + 1) * S)
            q = qkvf[rows, h * dh:(h + 1) * dh]
            k = qkvf[rows, C + h * dh:C + (h + 1) * dh]
            v = qkvf[rows, 2 * C + h * dh:2 * C + (h + 1) * dh]
            s = sp[u].cpu().numpy().astype(np.int64)
            ref = O.masked_attention_f64(q, k, v, bh[h].cpu().numpy(), bw[h].cpu().numpy(), s, s, tile, tile, r,
                                         tau)
            got = out[rows, h * dh:(h + 1) * dh].float().cpu().numpy()
            errs.append(np.linalg.norm(got - ref) / np.linalg.norm(ref))
    return max(errs)


@check("attn_local_dh64")
def _():
    e = attn_case(3, 2, 196, 64, 14, 32, 0.4)
    assert e < 2e-2, e
    return f"rel {e:.2e}"


@check("attn_local_dh80")
def _():
    e = attn_case(3, 2, 196, 80, 14, 32, 0.4)
    assert e < 2e-2, e
    return f"rel {e:.2e}"


@check("attn_global_dh80")
def _():
    e = attn_case(1, 2, 4096, 80, 64, 128, 0.4)
    assert e < 2e-2, e
    return f"rel {e:.2e}"


@check("attn_global_dh64_dense")
def _():
    e = attn_case(1, 1, 4096, 64, 64, 128, 1.0)
    assert e < 2e-2, e
    return f"rel {e:.2e}"


@check("ordering_bitexact")
def _():
    x = O.SplitMix(1).normal((64, 64, 96))
    xt = torch.from_numpy(x).to(dev)[None].contiguous()
    sg, sw = K.sobel_saliency(xt, 14)
    ref_g = O.sobel_magnitude(x)
    assert np.array_equal(sg[0].cpu().numpy(), ref_g), "global sobel"
    wins = O.split_windows(O.pad_grid(x, 14), 14)
    for wi in range(25):
        ref_w = O.sobel_magnitude(wins[wi].reshape(14, 14, -1)).reshape(-1)
        assert np.array_equal(sw[0, wi].cpu().numpy(), ref_w), f"window {wi}"
    mg = torch.from_numpy(O.morton_order(64, 64)).int().to(dev)
    mw = torch.from_numpy(O.morton_order(14, 14)).int().to(dev)
    sig_g, _ = K.rank_order(sg.reshape(1, -1), mg)
    sig_w, _ = K.rank_order(sw.reshape(25, -1), mw)
    ref = O.orderings(x, 14)
    assert np.array_equal(sig_g[0].cpu().numpy(), ref["global"]), "sigma global"
    assert np.array_equal(sig_w.cpu().numpy(), ref["local"]), "sigma local"
    return "sobel/sigma bit-exact"


@check("gemm_perf_qkv_vith")
def _():
    M, N, K_ = 8 * 4900, 3840, 1280
    a = torch.randn(M, K_, device=dev).bfloat16()
    w = torch.randn(N, K_, device=dev).bfloat16()
    b = torch.randn(N, device=dev)
    out = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        K.gemm(a, w, b, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 10
    for _ in range(n):
        K.gemm(a, w, b, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    tf = 2 * M * N * K_ / ms / 1e9
    wt = w.t()
    for _ in range(3):
        torch.matmul(a, wt)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        torch.matmul(a, wt)
    e1.record()
    torch.cuda.synchronize()
    ms2 = e0.elapsed_time(e1) / n
    return f"zs {ms:.3f} ms {tf:.0f} TF/s | cublas {ms2:.3f} ms {2 * M * N * K_ / ms2 / 1e9:.0f} TF/s"


@check("attn_perf_global_vith")
def _():
    B, H, S, dh = 8, 16, 4096, 80
    C = H * dh
    qkv = torch.randn(B * S, 3 * C, device=dev).bfloat16()
    bh = torch.randn(H, S, 64, device=dev) * 0.5
    bw = torch.randn(H, S, 64, device=dev) * 0.5
    sp = torch.stack([torch.randperm(S, device=dev) for _ in range(B)]).int()
    out = torch.empty(B * S, C, device=dev, dtype=torch.bfloat16)

    def run():
        K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=B, heads=H, sq=S, sk=S, dh=dh, bh=bh, bw=bw,
                      q_sp=sp, k_sp=sp, b_row=128, b_col=128, prefix=12, tau=dh ** -0.5, out=out)

    for _ in range(2):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    E = 6619136
    fl = 4 * dh * E * B * H
    return f"{ms:.3f} ms  {fl / ms / 1e9:.0f} TF/s effective"


@check("attn_perf_local_vith")
def _():
    B, H, S, dh = 8, 16, 196, 80
    U = B * 25
    C = H * dh
    qkv = torch.randn(U * S, 3 * C, device=dev).bfloat16()
    bh = torch.randn(H, S, 14, device=dev) * 0.5
    bw = torch.randn(H, S, 14, device=dev) * 0.5
    sp = torch.stack([torch.randperm(S, device=dev) for _ in range(U)]).int()
    out = torch.empty(U * S, C, device=dev, dtype=torch.bfloat16)

    def run():
        K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=U, heads=H, sq=S, sk=S, dh=dh, bh=bh, bw=bw,
                      q_sp=sp, k_sp=sp, b_row=32, b_col=32, prefix=2, tau=dh ** -0.5, out=out)

    for _ in range(2):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    byts = U * H * (4 * S * dh * 2) + 2 * H * S * 14 * 4
    return f"{ms:.3f} ms  {byts / ms / 1e6:.0f} GB/s algorithmic"


print("SUMMARY", sum(r[1] == "PASS" for r in results), "/", len(results))
