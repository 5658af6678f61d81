"""SAM decomposed relative-position mode and per-unit bias tables (marker: gpu).

The reference's attention takes static BiasTables (attention.py:28-55); SAM computes them per
query from q and rel_pos_h / rel_pos_w.  Parity is pinned two ways:
  * the tcgen05 rel-pos GEMM (zs_relpos_bias) against an fp32 torch twin of SAM's
    add_decomposed_rel_pos on the same bf16 q (tolerance below);
  * per-unit tables through the reference algorithm: zs_stripe_attn_fwd_unit_bias against the
    float64 oracle of ashape_attention (oracle/zs_oracle.py) unit by unit, and the fused
    zs_stripe_attn_fwd_relpos against the same attention fed the twin's tables.
"""

import math

import numpy as np
import pytest

from oracle import zs_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2605_17633_b200 import kernels as K

DEV = "cuda"


def rel(a, b):
    a = torch.as_tensor(a).double().cpu()
    b = torch.as_tensor(b).double().cpu()
    return float((a - b).norm() / b.norm().clamp_min(1e-300))


def twin_tables(q, sp, rh, rw, heads, dh, w):
    """fp32 twin of SAM add_decomposed_rel_pos as per-unit BiasTables [U, H, S, w] (spatial rows)."""
    U, S = sp.shape
    qf = q.float().reshape(U, S, heads, dh)
    s = sp.long()
    qy, qx = s // w, s % w
    kk = torch.arange(w, device=q.device)
    Rh = rh.float()[qy[:, :, None] - kk + w - 1]  # [U, S, w, dh]
    Rw = rw.float()[qx[:, :, None] - kk + w - 1]
    bh_rows = torch.einsum("ushc,uskc->uhsk", qf, Rh)
    bw_rows = torch.einsum("ushc,uskc->uhsk", qf, Rw)
    bh = torch.empty_like(bh_rows)
    bw = torch.empty_like(bw_rows)
    idx = s[:, None, :, None].expand(U, heads, S, w)
    bh.scatter_(2, idx, bh_rows)
    bw.scatter_(2, idx, bw_rows)
    return bh, bw


def make_case(units, heads, S, dh, w, seed):
    g = torch.Generator().manual_seed(seed)
    C = heads * dh
    qkv = torch.randn(units * S, 3 * C, generator=g).bfloat16().to(DEV)
    rh = (0.3 * torch.randn(2 * w - 1, dh, generator=g)).to(DEV)
    rw = (0.3 * torch.randn(2 * w - 1, dh, generator=g)).to(DEV)
    sp = torch.stack([torch.randperm(S, generator=g) for _ in range(units)]).int().to(DEV)
    return qkv, rh, rw, sp


@pytest.mark.parametrize("units,heads,S,dh,w", [(5, 3, 196, 80, 14), (4, 2, 196, 64, 14), (1, 2, 4096, 80, 64),
                                                (3, 2, 144, 80, 12), (2, 3, 1024, 64, 32)])
def test_relpos_tables_vs_fp32_twin(units, heads, S, dh, w):
    qkv, rh, rw, sp = make_case(units, heads, S, dh, w, seed=S + dh)
    C = heads * dh
    bh, bw = K.relpos_bias(qkv[:, :C], units=units, heads=heads, S=S, dh=dh, rel_pos_h=rh, rel_pos_w=rw, q_sp=sp)
    # exact products of the bf16-rounded tables (the kernel's operands): fp32 accumulation order only
    th, tw = twin_tables(qkv[:, :C], sp, rh.bfloat16().float(), rw.bfloat16().float(), heads, dh, w)
    assert rel(bh, th) < 1e-5 and rel(bw, tw) < 1e-5
    # against the fp32 tables: bf16 rounding of rel_pos only (<= 2^-9 relative per term)
    th, tw = twin_tables(qkv[:, :C], sp, rh, rw, heads, dh, w)
    assert rel(bh, th) < 4e-3 and rel(bw, tw) < 4e-3


def _oracle_unit(qkv, bh, bw, sp, u, h, S, dh, C, tile, r):
    qf = qkv.float().cpu().numpy()
    rows = slice(u * S, (u + 1) * S)
    s = sp[u].cpu().numpy().astype(np.int64)
    return O.masked_attention_f64(qf[rows, h * dh:(h + 1) * dh], qf[rows, C + h * dh:C + (h + 1) * dh],
                                  qf[rows, 2 * C + h * dh:2 * C + (h + 1) * dh], bh[u, h].cpu().numpy(),
                                  bw[u, h].cpu().numpy(), s, s, tile, tile, r)


@pytest.mark.parametrize("S,w,tile,r", [(196, 14, 32, 0.4), (196, 14, 32, 1.0), (4096, 64, 128, 0.4),
                                        (100, 10, 32, 0.4)])
def test_unit_bias_attention_vs_oracle(S, w, tile, r):
    """Per-unit BiasTables through every kernel family (window one-pass, window ping-pong at r=1,
    global) against the float64 oracle of ashape_attention, unit by unit."""
    units = 3 if S > 256 else 6
    heads, dh = 2, 80
    g = torch.Generator().manual_seed(7)
    C = heads * dh
    qkv = torch.randn(units * S, 3 * C, generator=g).bfloat16().to(DEV)
    bh = (0.5 * torch.randn(units, heads, S, w, generator=g)).to(DEV)
    bw = (0.5 * torch.randn(units, heads, S, w, generator=g)).to(DEV)
    sp = torch.stack([torch.randperm(S, generator=g) for _ in range(units)]).int().to(DEV)
    T = -(-S // tile)
    out = K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=units, heads=heads, sq=S, sk=S, dh=dh,
                        bh=bh, bw=bw, q_sp=sp, k_sp=sp, b_row=tile, b_col=tile, prefix=math.floor(r * T),
                        tau=1 / math.sqrt(dh))
    worst = 0.0
    for u in (0, units - 1):
        for h in range(heads):
            ref = _oracle_unit(qkv, bh, bw, sp, u, h, S, dh, C, tile, r)
            worst = max(worst, rel(out[u * S:(u + 1) * S, h * dh:(h + 1) * dh].float(), ref))
    assert worst < 1e-2  # bf16 P / output vs float64 softmax, as test_gpu_kernels.py


@pytest.mark.parametrize("S,w,tile,r,dh", [(196, 14, 32, 0.4, 80), (196, 14, 32, 0.2, 64), (196, 14, 32, 1.0, 80),
                                           (4096, 64, 128, 0.4, 80), (4096, 64, 128, 0.2, 64), (1024, 32, 128, 0.4, 80),
                                           (144, 12, 32, 0.5, 80), (784, 28, 128, 0.6, 64)])
def test_relpos_attention_matches_twin_tables(S, w, tile, r, dh):
    """Fused SAM mode (tables straight into the kernels' fp16 operand rows; r = 1 windows take
    the fp32-table fallback) == the same attention fed the fp32 twin's per-unit tables, and
    within the oracle tolerance of the float64 reference on those tables."""
    units = 2 if S > 256 else 9
    heads = 2
    qkv, rh, rw, sp = make_case(units, heads, S, dh, w, seed=31 + S)
    C = heads * dh
    T = -(-S // tile)
    kw = dict(units=units, heads=heads, sq=S, sk=S, dh=dh, q_sp=sp, k_sp=sp, b_row=tile, b_col=tile,
              prefix=math.floor(r * T), tau=1 / math.sqrt(dh))
    a = K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], bh=None, bw=None, rel_pos=(rh, rw), **kw)
    th, tw = twin_tables(qkv[:, :C], sp, rh, rw, heads, dh, w)
    b = K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], bh=th, bw=tw, **kw)
    assert rel(a.float(), b.float()) < 5e-3
    worst = 0.0
    for u in (0, units - 1):
        for h in range(heads):
            ref = _oracle_unit(qkv, th, tw, sp, u, h, S, dh, C, tile, r)
            worst = max(worst, rel(a[u * S:(u + 1) * S, h * dh:(h + 1) * dh].float(), ref))
    assert worst < 1e-2


def test_relpos_argument_errors():
    qkv, rh, rw, sp = make_case(2, 2, 196, 80, 14, seed=1)
    C = 160
    with pytest.raises(ValueError):
        K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=2, heads=2, sq=196, sk=196, dh=80, bh=None,
                      bw=None, q_sp=sp, k_sp=sp, b_row=32, b_col=32, prefix=2, tau=0.1, rel_pos=(rh[:-1], rw))
    with pytest.raises(ValueError):
        K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=2, heads=2, sq=196, sk=196, dh=80,
                      bh=torch.zeros(3, 2, 196, 14, device=DEV), bw=torch.zeros(3, 2, 196, 14, device=DEV), q_sp=sp,
                      k_sp=sp, b_row=32, b_col=32, prefix=2, tau=0.1)


def _twin_blocks(x, params, cfg):
    """fp32 torch twin of the blocks with SAM decomposed rel-pos, reference pad semantics
    (zero pads before LN1, MLP on padded windows, crop), r = keep = 1."""
    import torch.nn.functional as F

    from paper_2605_17633_b200.dense import sam_rel_pos_bias

    B, Hh, Ww, C = x.shape
    H, win = cfg.heads, cfg.window
    dh = C // H
    Hp, Wp = -(-Hh // win) * win, -(-Ww // win) * win
    for p in params:
        if p.kind == "local":  # zero pads re-created every local block (encoder.py:356), then windows
            xp = F.pad(x, (0, 0, 0, Wp - Ww, 0, Hp - Hh))
            t = xp.view(B, Hp // win, win, Wp // win, win, C).permute(0, 1, 3, 2, 4, 5).reshape(-1, win * win, C)
        else:
            t = x.reshape(B, Hh * Ww, C)
        N, S, _ = t.shape
        h = F.layer_norm(t, (C,), p.ln1_g, p.ln1_b, 1e-6)
        qkv = (h @ p.qkv_w.float().T + p.qkv_b).view(N, S, 3, H, dh).permute(2, 0, 3, 1, 4)
        q, k, v = qkv[0], qkv[1], qkv[2]
        att = (q * dh ** -0.5) @ k.transpose(-1, -2) + sam_rel_pos_bias(q, p.rel_pos_h, p.rel_pos_w)
        o = (att.softmax(-1) @ v).transpose(1, 2).reshape(N, S, C)
        t = t + o @ p.proj_w.float().T + p.proj_b
        hh = F.layer_norm(t, (C,), p.ln2_g, p.ln2_b, 1e-6)
        t = t + F.gelu(hh @ p.w1.float().T + p.b1) @ p.w2.float().T + p.b2
        if p.kind == "local":  # merge windows and crop the pads (encoder.py:366-368)
            x = t.view(B, Hp // win, Wp // win, win, win, C).permute(0, 1, 3, 2, 4, 5).reshape(B, Hp, Wp, C)
            x = x[:, :Hh, :Ww].contiguous()
        else:
            x = t.view(B, Hh, Ww, C)
    return x


@pytest.mark.parametrize("side", [28, 30])
def test_encoder_rel_pos_mode_vs_fp32_twin(side):
    """Whole local + global blocks in SAM rel-pos mode at r = keep = 1 vs the fp32 torch twin
    (tolerance of tests/test_gpu_encoder.py: cos >= 0.999, rel. Frobenius <= 3e-2); side 30
    pads the windows (30 -> 42), exercising the pad-token path (constant K/V rows, dropped
    query rows) with q-dependent biases."""
    import paper_2605_17633_b200 as Z
    from paper_2605_17633_b200.encoder import StripeSortEncoder
    from paper_2605_17633_b200.weights import random_params

    cfg = Z.EncoderConfig(grid=Z.GridShape(side, side), d=320, heads=4, window=14,
                          layout=("local", "global", "local"), r=1.0, keep_fraction=1.0)
    params = random_params(cfg, DEV, seed=4, rel_pos=True, rel_pos_std=0.5)
    assert params[0].bh is None and params[0].rel_pos_h.shape == (27, 80)
    assert params[1].rel_pos_h.shape == (2 * side - 1, 80)
    x = torch.randn(2, side, side, 320, device=DEV)
    got = StripeSortEncoder(cfg, params)(x).double()
    ref = _twin_blocks(x, params, cfg).double()
    cos = float((got * ref).sum() / (got.norm() * ref.norm()))
    assert cos >= 0.999 and rel(got, ref) <= 3e-2, (cos, rel(got, ref))


@pytest.mark.parametrize("S,w,tile", [(196, 14, 32), (4096, 64, 128)])
def test_relpos_attention_concurrent_streams(S, w, tile):
    """the SAM rel-pos path on two streams at once (different rel-pos tables) — every
    call takes its own workspace (caller-owned / stream-ordered allocator), so each result equals
    its sequential run."""
    units, heads, dh = (18 if S <= 256 else 2), 2, 80
    qkv, rh, rw, sp = make_case(units, heads, S, dh, w, seed=77)
    rh2, rw2 = rh.flip(0).contiguous(), (rw * 1.5).contiguous()
    C = heads * dh
    kw = dict(units=units, heads=heads, sq=S, sk=S, dh=dh, q_sp=sp, k_sp=sp, b_row=tile, b_col=tile, prefix=2,
              tau=dh ** -0.5, bh=None, bw=None)
    tabs = [(rh, rw), (rh2, rw2)]
    ref = [K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], rel_pos=t, **kw) for t in tabs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = [torch.empty_like(r) for r in ref]
    for _ in range(3):
        for s_, t, o in zip(streams, tabs, outs):
            s_.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s_):
                K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], rel_pos=t, out=o, **kw)
        torch.cuda.synchronize()
        for o, r in zip(outs, ref):
            assert torch.equal(o, r)
