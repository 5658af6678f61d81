"""Kernel-level parity on the B200 through the C ABI (marker: gpu).

Integer / index / data-movement kernels are checked bit-exactly; float kernels
against fp32 (GEMM, LN) or float64 (attention) oracles on the same bf16
inputs, with the tolerances written in each test.
"""

import math

import numpy as np
import pytest

from conftest import golden
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


# ---------------------------------------------------------------- GEMM
@pytest.mark.parametrize("M,N,K_", [(1, 256, 64), (127, 768, 768), (300, 512, 256), (1000, 3072, 768),
                                    (4900, 3840, 1280), (77, 1280, 5120)])
def test_gemm_bias_bf16(M, N, K_):
    g = torch.Generator(device=DEV).manual_seed(M + N)
    a = torch.randn(M, K_, device=DEV, generator=g).bfloat16()
    w = (torch.randn(N, K_, device=DEV, generator=g) / math.sqrt(K_)).bfloat16()
    b = torch.randn(N, device=DEV, generator=g)
    y = K.gemm(a, w, b)
    ref = a.float() @ w.float().T + b
    assert rel(y, ref) < 5e-3  # bf16 output rounding (2^-9) dominates


def test_gemm_gelu_epilogue():
    g = torch.Generator(device=DEV).manual_seed(3)
    a = torch.randn(333, 512, device=DEV, generator=g).bfloat16()
    w = (torch.randn(2048, 512, device=DEV, generator=g) / 20).bfloat16()
    b = torch.randn(2048, device=DEV, generator=g)
    y = K.gemm(a, w, b, epi=K.EPI_BF16_GELU)
    ref = torch.nn.functional.gelu(a.float() @ w.float().T + b)  # exact-erf GELU
    assert rel(y, ref) < 5e-3


@pytest.mark.parametrize("K_", [512, 2560])  # 2560: the TMA gather4 / scatter4 residual epilogue (long K)
def test_gemm_residual_scatter_zero_rows_and_device_m(K_):
    g = torch.Generator(device=DEV).manual_seed(4)
    M, N = 333, 768
    a = torch.randn(M, K_, device=DEV, generator=g).bfloat16()
    w = (torch.randn(N, K_, device=DEV, generator=g) / 20).bfloat16()
    b = torch.randn(N, device=DEV, generator=g)
    x = torch.randn(500, N, device=DEV, generator=g)
    x0 = x.clone()
    rm = torch.randperm(500, device=DEV, generator=g)[:M].int()
    zr = (torch.rand(M, device=DEV, generator=g) < 0.2).to(torch.uint8)
    mdev = torch.tensor([250], device=DEV, dtype=torch.int32)
    K.gemm(a, w, b, epi=K.EPI_F32_RESID, out=x, res=x, row_map=rm, zero_rows=zr, m_dev=mdev)
    ref = x0.clone()
    live = torch.arange(M, device=DEV) < 250
    upd = x0[rm.long()] + a.float() @ w.float().T + b
    upd[zr.bool()] = 0
    ref[rm.long()[live]] = upd[live]
    assert rel(x, ref) < 1e-5  # fp32 output: accumulation order only
    untouched = torch.ones(500, dtype=torch.bool, device=DEV)
    untouched[rm.long()[live]] = False
    assert torch.equal(x[untouched], x0[untouched])


def test_gemm_residual_scatter_many_tiles_long_k():
    """fc2-shaped residual scatter-add (K = 4C, many tiles per cluster: the TMA epilogue gathers the
    next tile's rows while storing this one's), ragged M, bias."""
    g = torch.Generator(device=DEV).manual_seed(14)
    M, N, K_ = 20011, 1280, 5120
    a = torch.randn(M, K_, device=DEV, generator=g).bfloat16()
    w = (torch.randn(N, K_, device=DEV, generator=g) / 72).bfloat16()
    b = torch.randn(N, device=DEV, generator=g)
    x = torch.randn(25000, N, device=DEV, generator=g)
    x0 = x.clone()
    rm = torch.randperm(25000, device=DEV, generator=g)[:M].int()
    K.gemm(a, w, b, epi=K.EPI_F32_RESID, out=x, res=x, row_map=rm)
    ref = x0.clone()
    ref[rm.long()] = x0[rm.long()] + a.float() @ w.float().T + b
    assert rel(x, ref) < 1e-5
    untouched = torch.ones(25000, dtype=torch.bool, device=DEV)
    untouched[rm.long()] = False
    assert torch.equal(x[untouched], x0[untouched])


@pytest.mark.parametrize("K_", [256, 2560])
def test_gemm_residual_modulo_rows(K_):
    g = torch.Generator(device=DEV).manual_seed(5)
    a = torch.randn(3 * 64, K_, device=DEV, generator=g).bfloat16()
    w = (torch.randn(256, K_, device=DEV, generator=g) / (K_ ** 0.5)).bfloat16()
    pos = torch.randn(64, 256, device=DEV, generator=g)
    y = K.gemm(a, w, None, epi=K.EPI_F32_RESID, res=pos, res_mod=64)
    ref = a.float() @ w.float().T + pos.repeat(3, 1)
    assert rel(y, ref) < 1e-5


def test_gemm_rejects_bad_shapes():
    a = torch.zeros(8, 100, device=DEV, dtype=torch.bfloat16)
    w = torch.zeros(64, 100, device=DEV, dtype=torch.bfloat16)
    with pytest.raises(RuntimeError, match="zs_status -2"):
        K.gemm(a, w)


# ---------------------------------------------------------------- LN / permute / maps
def test_layernorm_rows_gather():
    g = torch.Generator(device=DEV).manual_seed(6)
    x = torch.randn(500, 1280, device=DEV, generator=g) * 3 + 1
    gam = torch.randn(1280, device=DEV, generator=g)
    bet = torch.randn(1280, device=DEV, generator=g)
    rows = torch.randperm(500, device=DEV, generator=g)[:200].int()
    y = K.layernorm_rows(x, gam, bet, rows, out_f32=True)
    ref = O.layernorm(x[rows.long()].cpu().numpy(), gam.cpu().numpy(), bet.cpu().numpy())
    assert rel(y, ref) < 1e-5
    yb = K.layernorm_rows(x, gam, bet, rows)
    assert rel(yb, ref) < 5e-3


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_permute_rows_exact(dtype):
    dt = getattr(torch, dtype)
    src = torch.randn(300, 1280, device=DEV).to(dt)
    mp = torch.randint(-1, 300, (777,), device=DEV, dtype=torch.int32)
    out = K.permute_rows(src, mp)
    ref = torch.zeros(777, 1280, device=DEV, dtype=dt)
    ok = mp >= 0
    ref[ok] = src[mp[ok].long()]
    assert torch.equal(out, ref)


def test_cast_rows_bf16_exact():
    src = torch.randn(300, 256, device=DEV)
    assert torch.equal(K.cast_rows_bf16(src), src.bfloat16())


def test_layout_maps_match_oracle_window_split():
    """Maps reproduce _pad_grid/_split_windows∘sigma and sigma_g exactly (encoder.py:232-254)."""
    rng = np.random.default_rng(0)
    B, H, W, win = 2, 20, 20, 6
    nwin = 16
    sig_l = np.stack([rng.permutation(win * win) for _ in range(B * nwin)]).astype(np.int32)
    sig_g = np.stack([rng.permutation(H * W) for _ in range(B)]).astype(np.int32)
    m = K.layout_maps(torch.from_numpy(sig_g).to(DEV), torch.from_numpy(sig_l).to(DEV), B, H, W, win)
    tok = np.arange(B * H * W).reshape(B, H, W, 1).astype(np.float32)
    exp_l = []
    for b in range(B):
        wins = O.split_windows(O.pad_grid(tok[b] + 1, win), win)  # +1 so pads (0) are distinguishable
        for wi in range(nwin):
            exp_l.append(wins[wi, sig_l[b * nwin + wi], 0] - 1)
    exp_l = np.concatenate(exp_l).astype(np.int64)
    got_l = m["l_from_s"].cpu().numpy()
    assert np.array_equal(got_l, exp_l)
    assert np.array_equal(m["l_is_pad"].cpu().numpy().astype(bool), exp_l < 0)
    exp_g = (sig_g + np.arange(B)[:, None] * H * W).reshape(-1)
    assert np.array_equal(m["g_from_s"].cpu().numpy(), exp_g)
    # round trips: S -> L -> G -> S and S -> G -> L -> S are identities on real tokens
    s = torch.arange(B * H * W, device=DEV, dtype=torch.float32)[:, None].repeat(1, 4).contiguous()
    L = K.permute_rows(s, m["l_from_s"])
    G = K.permute_rows(L, m["g_from_l"])
    assert torch.equal(G, K.permute_rows(s, m["g_from_s"]))
    assert torch.equal(K.permute_rows(G, m["s_from_g"]), s)
    assert torch.equal(K.permute_rows(K.permute_rows(G, m["l_from_g"]), m["s_from_l"]), s)
    assert torch.equal(K.permute_rows(L, m["s_from_l"]), s)


def test_keep_rows_prefix_skips_pads():
    U, S, Kc = 37, 196, 78
    rng = np.random.default_rng(1)
    pad = (rng.random(U * S) < 0.2).astype(np.uint8)
    keep, offs = K.prefix_keep_rows(U, S, Kc, torch.from_numpy(pad).to(DEV))
    n = int(offs[U])
    exp = np.array([u * S + i for u in range(U) for i in range(Kc) if not pad[u * S + i]])
    assert n == exp.size
    assert np.array_equal(keep[:n].cpu().numpy(), exp)
    byp, boff = K.unit_span_rows(U, S, Kc, S, torch.from_numpy(pad).to(DEV))
    expb = np.array([u * S + i for u in range(U) for i in range(Kc, S) if not pad[u * S + i]])
    assert int(boff[U]) == expb.size and np.array_equal(byp[: expb.size].cpu().numpy(), expb)


# ---------------------------------------------------------------- ordering (bit-exact)
def test_sobel_and_orderings_bitexact_small_all_variants():
    g = golden("orders_small")
    x = O.SplitMix(1).normal((20, 20, 24))
    xt = torch.from_numpy(x).to(DEV)[None].contiguous()
    sg, sw = K.sobel_saliency(xt, 6)
    assert np.array_equal(sg[0].cpu().numpy(), g["small_sobel"])
    wins = O.split_windows(O.pad_grid(x, 6), 6)
    for wi in range(wins.shape[0]):
        assert np.array_equal(sw[0, wi].cpu().numpy(), O.sobel_magnitude(wins[wi].reshape(6, 6, -1)).reshape(-1))
    mg = torch.from_numpy(O.morton_order(20, 20)).int().to(DEV)
    mw = torch.from_numpy(O.morton_order(6, 6)).int().to(DEV)
    for gran in ("zgroup", "token"):
        for var in ("full", "no_interleave", "no_sort"):
            s1, _ = K.rank_order(sg.reshape(1, -1), mg, granularity=gran, variant=var)
            s2, _ = K.rank_order(sw.reshape(16, -1), mw, granularity=gran, variant=var)
            assert np.array_equal(s1[0].cpu().numpy(), g[f"small_{gran}_{var}_global"]), (gran, var)
            assert np.array_equal(s2.cpu().numpy(), g[f"small_{gran}_{var}_local"]), (gran, var)


def test_orderings_bitexact_config1():
    """Config 1 input (64x64x768, zstripe.Rng(1)): sigma_global and all 25 sigma_w bit-exact."""
    g = golden("orders_config1")
    x = O.SplitMix(1).normal((64, 64, 768))
    xt = torch.from_numpy(x).to(DEV)[None].contiguous()
    sg, sw = K.sobel_saliency(xt, 14)
    assert np.array_equal(sg[0].cpu().numpy()[::7], g["sobel_rows"])
    s1, _ = K.rank_order(sg.reshape(1, -1), torch.from_numpy(O.morton_order(64, 64)).int().to(DEV))
    s2, _ = K.rank_order(sw.reshape(25, -1), torch.from_numpy(O.morton_order(14, 14)).int().to(DEV))
    assert np.array_equal(s1[0].cpu().numpy(), g["sigma_global"])
    assert np.array_equal(s2.cpu().numpy(), g["sigma_local"])


def test_rank_from_reference_energies_bitexact():
    """Top-K index sets are bit-exact when fed the reference's scores (north star)."""
    g = golden("orders_small")
    e = torch.from_numpy(g["small_energy"]).to(DEV)[None]
    mg = torch.from_numpy(O.morton_order(20, 20)).int().to(DEV)
    sig, _ = K.rank_order(e, mg, variant="no_interleave", scores_are_energy=True)
    assert np.array_equal(sig[0].cpu().numpy(), g["small_pi"])


def test_rank_ties_and_nan_follow_numpy_lexsort():
    # ties -> ascending group index; NaN sorts last (numpy lexsort on -energy)
    e = np.array([1.0, 3.0, 3.0, np.nan, 0.0, 3.0, -0.0, np.nan], np.float32)
    morton = np.arange(32)
    exp = O.order_from_energy(e, morton, 4)
    sig, _ = K.rank_order(torch.from_numpy(e).to(DEV)[None], torch.from_numpy(morton).int().to(DEV),
                          variant="no_interleave", scores_are_energy=True)
    assert np.array_equal(sig[0].cpu().numpy(), exp)


# ---------------------------------------------------------------- attention
def _parity_stripes(S, w, g):
    """σ as the global stripe-sort produces it for G = 4: the four (y % 2, x % 2) classes one after
    the other (stripesort.py:38-62 over 2x2 Morton groups), each in its own order."""
    pos = torch.arange(S)
    cls = ((pos // w) % 2) * 2 + (pos % w) % 2
    return torch.argsort(cls.double() * 2 + torch.rand(S, generator=g, dtype=torch.float64))


def _attn_case(units, heads, S, dh, w, tile, r, seed=0, bscale=0.5, stripes=False):
    g = torch.Generator().manual_seed(seed)
    C = heads * dh
    qkv = torch.randn(units * S, 3 * C, generator=g).bfloat16().to(DEV)
    bh = (bscale * torch.randn(heads, S, w, generator=g)).to(DEV)
    bw = (bscale * torch.randn(heads, S, w, generator=g)).to(DEV)
    if stripes == "shifted":  # class boundaries mid-chunk: parity-pure and mixed chunks in one item
        mk = lambda: torch.roll(_parity_stripes(S, w, g), 64)  # noqa: E731
    else:
        mk = (lambda: _parity_stripes(S, w, g)) if stripes else (lambda: torch.randperm(S, generator=g))
    sp = torch.stack([mk() for _ in range(units)]).int().to(DEV)
    T = -(-S // tile)
    out = K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=units, heads=heads, sq=S, sk=S, dh=dh,
                        bh=bh, bw=bw, q_sp=sp, k_sp=sp, b_row=tile, b_col=tile, prefix=math.floor(r * T),
                        tau=1 / math.sqrt(dh))
    qkvf = qkv.float().cpu().numpy()
    worst = 0.0
    for u in {0, units - 1}:
        for h in range(heads):
            rows = slice(u * S, (u + 1) * S)
            s = sp[u].cpu().numpy().astype(np.int64)
            ref = O.masked_attention_f64(qkvf[rows, h * dh:(h + 1) * dh], qkvf[rows, C + h * dh:C + (h + 1) * dh],
                                         qkvf[rows, 2 * C + h * dh:2 * C + (h + 1) * dh], bh[h].cpu().numpy(),
                                         bw[h].cpu().numpy(), s, s, tile, tile, r)
            worst = max(worst, rel(out[rows, h * dh:(h + 1) * dh].float(), ref))
    return worst


@pytest.mark.parametrize("dh", [64, 80])
@pytest.mark.parametrize("r", [0.0, 0.2, 0.4, 0.6, 0.8, 1.0])
def test_attention_local_window(dh, r):
    # tolerance: bf16 P and bf16 output vs float64 softmax -> ~2e-3 relative
    assert _attn_case(5, 2, 196, dh, 14, 32, r) < 1e-2


@pytest.mark.parametrize("S,w,tile,r", [(100, 10, 32, 0.4), (144, 12, 32, 0.5), (225, 15, 64, 0.3), (64, 8, 32, 1.0),
                                        (121, 11, 32, 0.4), (169, 13, 32, 0.5), (256, 16, 32, 0.4)])
def test_attention_window_shapes(S, w, tile, r):
    """Single-tile windows (S <= 128), a 144-token window, 64-row tiles, odd table widths; partial
    last key groups (32 wide with 25 keys for S = 121, 16 wide with 9 keys for S = 169), which the
    kernel masks with the bias marker column rather than per element; S = 256 (w = 16: no free
    bias column, and no keys past S)."""
    assert _attn_case(7, 3, S, 80, w, tile, r, seed=3) < 1e-2
    assert _attn_case(7, 2, S, 64, w, tile, r, seed=4) < 1e-2


@pytest.mark.parametrize("r", [0.2, 0.4, 0.8])
def test_attention_window_kernels_agree(r, monkeypatch):
    """The one-pass TMEM-P window kernel and the ping-pong window kernel give the same
    softmax (both within bf16 rounding of each other)."""
    g = torch.Generator().manual_seed(11)
    units, heads, S, dh, w = 40, 4, 196, 80, 14
    C = heads * dh
    qkv = torch.randn(units * S, 3 * C, generator=g).bfloat16().to(DEV)
    bh = (0.5 * torch.randn(heads, S, w, generator=g)).to(DEV)
    bw = (0.5 * torch.randn(heads, S, w, generator=g)).to(DEV)
    sp = torch.stack([torch.randperm(S, generator=g) for _ in range(units)]).int().to(DEV)
    kw = dict(units=units, heads=heads, sq=S, sk=S, dh=dh, bh=bh, bw=bw, q_sp=sp, k_sp=sp, b_row=32, b_col=32,
              prefix=math.floor(r * 7), tau=dh ** -0.5)
    a = K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], **kw)
    monkeypatch.setenv("ZS_ATTN_NO_WIN", "1")
    b = K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], **kw)
    assert rel(a.float(), b.float()) < 5e-3


@pytest.mark.parametrize("dh", [64, 80])
@pytest.mark.parametrize("r", [0.0, 0.2, 0.4, 1.0])
def test_attention_global(dh, r):
    assert _attn_case(2, 2, 4096, dh, 64, 128, r) < 1e-2


@pytest.mark.parametrize("dh", [64, 80])
def test_attention_global_partial_tiles(dh):
    """A 30 x 30 grid (S = 900): the last query tile has 4 rows and the last key chunk 4 keys, so
    the kernel's key-range mask and the epilogue warps' row guard are exercised."""
    assert _attn_case(3, 2, 900, dh, 30, 128, 0.4, seed=13) < 1e-2
    assert _attn_case(2, 3, 900, dh, 30, 128, 1.0, seed=14) < 1e-2


@pytest.mark.parametrize("dh", [64, 80])
@pytest.mark.parametrize("r", [0.2, 0.4, 1.0])
def test_attention_global_parity_stripes(dh, r):
    """Stripe-ordered keys as the global stripe sort produces them (every 128-key chunk inside one
    (y % 2, x % 2) class), 4096- and 1024-token grids."""
    assert _attn_case(2, 2, 4096, dh, 64, 128, r, seed=8, stripes=True) < 1e-2
    assert _attn_case(3, 2, 1024, dh, 32, 128, r, seed=9, stripes=True) < 1e-2
    assert _attn_case(2, 2, 4096, dh, 64, 128, r, seed=10, stripes="shifted") < 1e-2


@pytest.mark.parametrize("S,w,tile", [(4096, 64, 128), (196, 14, 32)])
def test_attention_large_bias(S, w, tile):
    """Bias spread far beyond the lazy-rescale threshold (ln 256): rows move their reference max
    on many chunks, so the O rescale runs mid-item, for some rows of a warp only."""
    units = 2 if S > 256 else 8
    assert _attn_case(units, 2, S, 80, w, tile, 0.4, seed=5, bscale=6.0) < 1e-2
    assert _attn_case(units, 2, S, 64, w, tile, 1.0, seed=6, bscale=6.0) < 1e-2


@pytest.mark.parametrize("dh", [64, 80])
def test_attention_many_items_per_cta(dh):
    """More work items than SMs: every persistent CTA walks several (unit, head, block) items,
    so the Q / K / V / metadata rings run across item boundaries."""
    assert _attn_case(300, 3, 196, dh, 14, 32, 0.4, seed=1) < 1e-2
    assert _attn_case(5, 8, 4096, dh, 64, 128, 0.4, seed=2) < 1e-2


@pytest.mark.parametrize("r", [0.2, 0.6, 0.8])
def test_attention_window_variants_many_items(r):
    """The window kernel's three schedules with several items per CTA: Bq rows in TMEM with
    double-buffered key rows (d = 0.2), shared-memory Bq slabs (d = 0.6: S_A + S_B + 2 O fill the
    TMEM columns), tiles in sequence (d = 0.8)."""
    assert _attn_case(300, 2, 196, 80, 14, 32, r, seed=12) < 1e-2


def test_attention_general_tiles_many_items():
    """Tile sizes that are not multiples of 32 take the per-element mask path."""
    g = torch.Generator().manual_seed(9)
    units, heads, S, dh, w = 200, 2, 81, 64, 9
    C = heads * dh
    qkv = torch.randn(units * S, 3 * C, generator=g).bfloat16().to(DEV)
    bh = (0.5 * torch.randn(heads, S, w, generator=g)).to(DEV)
    bw = (0.5 * torch.randn(heads, S, w, generator=g)).to(DEV)
    sp = torch.stack([torch.randperm(S, generator=g) for _ in range(units)]).int().to(DEV)
    for br, bc, r in [(16, 24, 0.4), (7, 5, 0.3), (81, 81, 1.0)]:
        tc = -(-S // bc)
        out = K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], units=units, heads=heads, sq=S, sk=S, dh=dh,
                            bh=bh, bw=bw, q_sp=sp, k_sp=sp, b_row=br, b_col=bc, prefix=math.floor(r * tc), tau=0.125)
        qf = qkv.float().cpu().numpy()
        for u in (0, units - 1):
            rows = slice(u * S, (u + 1) * S)
            s = sp[u].cpu().numpy().astype(np.int64)
            ref = O.masked_attention_f64(qf[rows, :dh], qf[rows, C:C + dh], qf[rows, 2 * C:2 * C + dh],
                                         bh[0].cpu().numpy(), bw[0].cpu().numpy(), s, s, br, bc, r, 0.125)
            assert rel(out[rows, :dh].float(), ref) < 1e-2, (br, bc, r)


def test_im2col3x3_tap_major():
    """Neck 3x3 im2col: tap-major columns (ky, kx, c), zero padding, exact copy."""
    g = torch.Generator().manual_seed(4)
    x = torch.randn(2, 5, 7, 16, generator=g).bfloat16().to(DEV)
    out = K.im2col3x3(x)
    xp = torch.nn.functional.pad(x.permute(0, 3, 1, 2).float(), (1, 1, 1, 1))
    ref = torch.stack([xp[:, :, ky:ky + 5, kx:kx + 7] for ky in range(3) for kx in range(3)], dim=-1)
    ref = ref.permute(0, 2, 3, 4, 1).reshape(2 * 5 * 7, 9 * 16)
    assert torch.equal(out.float(), ref)


@pytest.mark.parametrize("S,w,tile", [(196, 14, 32), (1024, 32, 128)])
def test_attention_output_row_map_and_pad_helpers(S, w, tile):
    """zs_stripe_attn_fwd_rows writes row r of unit u to out[o_rows[u*S+r]] (skips -1) and equals the
    plain layout otherwise (window kernel, and the global kernel whose plain layout leaves through a
    TMA tensor store); invert_rows / fill_flagged_rows (window pad-token skipping)."""
    g = torch.Generator().manual_seed(21)
    units, heads, dh = 6, 2, 80
    C = heads * dh
    qkv = torch.randn(units * S, 3 * C, generator=g).bfloat16().to(DEV)
    bh = (0.5 * torch.randn(heads, S, w, generator=g)).to(DEV)
    bw = (0.5 * torch.randn(heads, S, w, generator=g)).to(DEV)
    sp = torch.stack([torch.randperm(S, generator=g) for _ in range(units)]).int().to(DEV)
    kw = dict(units=units, heads=heads, sq=S, sk=S, dh=dh, bh=bh, bw=bw, q_sp=sp, k_sp=sp, b_row=tile, b_col=tile,
              prefix=2, tau=dh ** -0.5)
    full = K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], **kw)
    keep = (torch.rand(units * S, generator=g) < 0.8).to(DEV)
    rows = keep.nonzero().flatten().int()
    omap = K.invert_rows(rows, units * S)
    assert torch.equal(omap[rows.long()].cpu(), torch.arange(rows.numel(), dtype=torch.int32))
    assert bool((omap[~keep] == -1).all())
    comp = torch.zeros(units * S, C, device=DEV, dtype=torch.bfloat16)
    K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], out=comp, o_rows=omap, **kw)
    n = rows.numel()
    assert torch.equal(comp[:n], full[rows.long()])
    assert bool((comp[n:] == 0).all())
    dst = torch.zeros(10, 24, device=DEV, dtype=torch.bfloat16)
    src = torch.randn(1, 24, generator=g).bfloat16().to(DEV)
    flag = torch.tensor([0, 1, 1, 0, 0, 1, 0, 0, 0, 1], dtype=torch.uint8, device=DEV)
    K.fill_flagged_rows(dst, src, flag)
    assert torch.equal(dst[flag.bool()], src.expand(4, 24))
    assert bool((dst[~flag.bool()] == 0).all())


@pytest.mark.parametrize("S,w,tile", [(196, 14, 32), (4096, 64, 128)])
def test_attention_concurrent_streams(S, w, tile):
    """Two streams run the attention at once with different bias tables: each call's bias-operand
    workspace comes from the stream-ordered caching allocator (the library owns none), so each
    result equals its own sequential run."""
    g = torch.Generator().manual_seed(21)
    units, heads, dh = (40 if S <= 256 else 2), 2, 80
    C = heads * dh
    qkv = torch.randn(units * S, 3 * C, generator=g).bfloat16().to(DEV)
    sp = torch.stack([torch.randperm(S, generator=g) for _ in range(units)]).int().to(DEV)
    tabs = [((0.5 * torch.randn(heads, S, w, generator=g)).to(DEV), (0.5 * torch.randn(heads, S, w, generator=g)).to(DEV))
            for _ in range(2)]
    kw = dict(units=units, heads=heads, sq=S, sk=S, dh=dh, q_sp=sp, k_sp=sp, b_row=tile, b_col=tile, prefix=2,
              tau=dh ** -0.5)
    ref = [K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], bh=bh, bw=bw, **kw) for bh, bw in tabs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = [torch.empty_like(r) for r in ref]
    for _ in range(3):
        for s_, (bh, bw), o in zip(streams, tabs, outs):
            s_.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s_):
                K.stripe_attn(qkv[:, :C], qkv[:, C:2 * C], qkv[:, 2 * C:], bh=bh, bw=bw, out=o, **kw)
        torch.cuda.synchronize()
        for o, r in zip(outs, ref):
            assert torch.equal(o, r)


@pytest.mark.parametrize("B,H,W,P", [(2, 1024, 1024, 16), (1, 64, 96, 16), (2, 48, 40, 8)])
def test_patchify_bit_exact(B, H, W, P):
    """Patch extraction of the SAM patch embed (16x16/16 conv as GEMM rows): bf16 of the same
    pixels in (c, ky, kx) column order, vectorised kernel (P = 16) and generic kernel."""
    img = torch.randn(B, 3, H, W, device=DEV)
    got = K.patchify(img, P)
    ref = (img.view(B, 3, H // P, P, W // P, P).permute(0, 2, 4, 1, 3, 5)
           .reshape(B * (H // P) * (W // P), 3 * P * P).bfloat16())
    assert torch.equal(got, ref)
