"""Typed torch-tensor front-ends for every native entry point.

Each function validates dtypes / devices / contiguity, passes raw device
pointers and the current CUDA stream through the C ABI, and returns new
tensors (or writes the caller-provided ones).  PyTorch is only the
allocator and stream provider here; all arithmetic runs in
``libzstripe_b200.so``.
"""

from __future__ import annotations

import math

import torch

from . import _lib

EPI_BF16, EPI_BF16_GELU, EPI_F32_RESID = 0, 1, 2


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _need(t: torch.Tensor, dtype: torch.dtype, name: str) -> None:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must live on a CUDA device (no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")


# ------------------------------------------------------------------ GEMM
def gemm(
    a: torch.Tensor,
    w: torch.Tensor,
    bias: torch.Tensor | None = None,
    *,
    epi: int = EPI_BF16,
    out: torch.Tensor | None = None,
    res: torch.Tensor | None = None,
    row_map: torch.Tensor | None = None,
    zero_rows: torch.Tensor | None = None,
    res_mod: int = 0,
    m_dev: torch.Tensor | None = None,
) -> torch.Tensor:
    """``a[M,K] @ w[N,K]^T`` on tcgen05 with the fused epilogue ``epi``."""
    _need(a, torch.bfloat16, "a")
    _need(w, torch.bfloat16, "w")
    if a.dim() != 2 or w.dim() != 2 or a.shape[1] != w.shape[1]:
        raise ValueError(f"gemm shapes {tuple(a.shape)} x {tuple(w.shape)}^T")
    if a.stride(1) != 1 or w.stride(1) != 1:
        raise ValueError("gemm operands must be K-contiguous")
    M, K = a.shape
    N = w.shape[0]
    if bias is not None:
        _need(bias, torch.float32, "bias")
    if out is None:
        if epi == EPI_F32_RESID:
            out = torch.empty((M, N), device=a.device, dtype=torch.float32)
        else:
            out = torch.empty((M, N), device=a.device, dtype=torch.bfloat16)
    if epi == EPI_F32_RESID:
        _need(out, torch.float32, "out")
    else:
        _need(out, torch.bfloat16, "out")
    if res is not None:
        _need(res, torch.float32, "res")
    if row_map is not None:
        _need(row_map, torch.int32, "row_map")
    if zero_rows is not None:
        _need(zero_rows, torch.uint8, "zero_rows")
    if m_dev is not None:
        _need(m_dev, torch.int32, "m_dev")
    _lib.call(
        "zs_gemm_bf16", epi, _ptr(a), a.stride(0), _ptr(w), w.stride(0), M, N, K, _ptr(bias), _ptr(out),
        out.stride(0), _ptr(res), 0 if res is None else res.stride(0), _ptr(row_map), _ptr(zero_rows), res_mod,
        _ptr(m_dev), _stream(),
    )
    return out


# ------------------------------------------------------------------ layernorm
def layernorm_rows(
    x: torch.Tensor,
    gamma: torch.Tensor,
    beta: torch.Tensor,
    rows: torch.Tensor | None = None,
    *,
    eps: float = 1e-6,
    out_f32: bool = False,
    out: torch.Tensor | None = None,
    out_rows: torch.Tensor | None = None,
    n_dev: torch.Tensor | None = None,
) -> torch.Tensor:
    _need(x, torch.float32, "x")
    _need(gamma, torch.float32, "gamma")
    _need(beta, torch.float32, "beta")
    n = x.shape[0] if rows is None else rows.shape[0]
    C = x.shape[1]
    if rows is not None:
        _need(rows, torch.int32, "rows")
    if out is None:
        out = torch.empty((n, C), device=x.device, dtype=torch.float32 if out_f32 else torch.bfloat16)
    if n_dev is not None or out_rows is not None:
        _lib.call("zs_layernorm_rows_ex", _ptr(x), x.stride(0), _ptr(rows), _ptr(out_rows), n, _ptr(n_dev), C,
                  _ptr(gamma), _ptr(beta), eps, _ptr(out), out.stride(0), int(out_f32), _stream())
    else:
        _lib.call("zs_layernorm_rows", _ptr(x), x.stride(0), _ptr(rows), n, C, _ptr(gamma), _ptr(beta), eps,
                  _ptr(out), out.stride(0), int(out_f32), _stream())
    return out


# ------------------------------------------------------------------ permute
def permute_rows(src: torch.Tensor, row_map: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """``out[r] = src[map[r]]`` (zeros where ``map[r] < 0``)."""
    _need(row_map, torch.int32, "map")
    if src.dim() != 2 or not src.is_contiguous():
        raise ValueError("src must be a contiguous [rows, C] matrix")
    rows = row_map.numel()
    if out is None:
        out = torch.empty((rows, src.shape[1]), device=src.device, dtype=src.dtype)
    if src.dtype == torch.float32:
        _lib.call("zs_permute_rows_f32", _ptr(src), _ptr(out), _ptr(row_map), rows, src.shape[1], _stream())
    elif src.dtype == torch.bfloat16:
        _lib.call("zs_permute_rows_bf16", _ptr(src), _ptr(out), _ptr(row_map), rows, src.shape[1], _stream())
    else:
        raise TypeError(f"permute_rows supports float32 / bfloat16, got {src.dtype}")
    return out


def cast_rows_bf16(src: torch.Tensor, row_map: torch.Tensor | None = None,
                   out: torch.Tensor | None = None) -> torch.Tensor:
    """bf16 copy of fp32 rows, optionally gathered through ``row_map``."""
    _need(src, torch.float32, "src")
    rows = src.shape[0] if row_map is None else row_map.numel()
    if out is None:
        out = torch.empty((rows, src.shape[1]), device=src.device, dtype=torch.bfloat16)
    _lib.call("zs_permute_rows_f32_bf16", _ptr(src), _ptr(out), _ptr(row_map), rows, src.shape[1], _stream())
    return out


# ------------------------------------------------------------------ ordering
def sobel_saliency(x: torch.Tensor, window: int, *, glob: bool = True, win: bool = True):
    """fp32 ``x[B,H,W,C]`` -> (``sal_glob[B,H,W]`` | None, ``sal_win[B,nwin,window^2]`` | None)."""
    _need(x, torch.float32, "x")
    if x.dim() != 4 or not x.is_contiguous():
        raise ValueError(f"expected contiguous [B, H, W, C], got {tuple(x.shape)}")
    B, H, W, Cc = x.shape
    nwin = math.ceil(H / window) * math.ceil(W / window)
    sg = torch.empty((B, H, W), device=x.device, dtype=torch.float32) if glob else None
    sw = torch.empty((B, nwin, window * window), device=x.device, dtype=torch.float32) if win else None
    _lib.call("zs_sobel_saliency", _ptr(x), B, H, W, Cc, window, _ptr(sg), _ptr(sw), _stream())
    return sg, sw


GRANULARITY = {"zgroup": 0, "token": 1}
VARIANT = {"full": 0, "no_interleave": 1, "no_sort": 2}


def rank_order(
    scores: torch.Tensor,
    morton_fwd: torch.Tensor,
    *,
    granularity: str = "zgroup",
    group_size: int = 4,
    g: int = 4,
    variant: str = "full",
    scores_are_energy: bool = False,
    want_energy: bool = False,
):
    """Per-unit importance order + stripe interleave -> sigma [U, N] int32 (and energies)."""
    _need(scores, torch.float32, "scores")
    _need(morton_fwd, torch.int32, "morton_fwd")
    N = morton_fwd.numel()
    U = scores.numel() // (N // group_size if scores_are_energy else N)
    sigma = torch.empty((U, N), device=scores.device, dtype=torch.int32)
    energy = None
    if want_energy and granularity == "zgroup":
        energy = torch.empty((U, N // group_size), device=scores.device, dtype=torch.float32)
    _lib.call("zs_rank_order", _ptr(scores.contiguous()), int(scores_are_energy), U, N, GRANULARITY[granularity],
              group_size, g, VARIANT[variant], _ptr(morton_fwd), _ptr(sigma), _ptr(energy), _stream())
    return sigma, energy


def layout_maps(sigma_glob: torch.Tensor | None, sigma_loc: torch.Tensor | None, B: int, H: int, W: int,
                window: int) -> dict:
    dev = (sigma_glob if sigma_glob is not None else sigma_loc).device
    nwin = math.ceil(H / window) * math.ceil(W / window)
    nl = B * nwin * window * window
    ng = B * H * W
    i32 = dict(device=dev, dtype=torch.int32)
    m = {}
    if sigma_loc is not None:
        m["l_from_s"] = torch.empty(nl, **i32)
        m["s_from_l"] = torch.empty(ng, **i32)
        m["l_is_pad"] = torch.empty(nl, device=dev, dtype=torch.uint8)
    if sigma_glob is not None:
        m["s_from_g"] = torch.empty(ng, **i32)
        m["g_from_s"] = torch.empty(ng, **i32)
    if sigma_glob is not None and sigma_loc is not None:
        m["g_from_l"] = torch.empty(ng, **i32)
        m["l_from_g"] = torch.empty(nl, **i32)
    _lib.call("zs_layout_maps", _ptr(sigma_glob), _ptr(sigma_loc), B, H, W, window, _ptr(m.get("l_from_s")),
              _ptr(m.get("g_from_l")), _ptr(m.get("l_from_g")), _ptr(m.get("s_from_g")), _ptr(m.get("s_from_l")),
              _ptr(m.get("g_from_s")), _ptr(m.get("l_is_pad")), _stream())
    return m


def unit_span_rows(U: int, S: int, begin: int, end: int, is_pad: torch.Tensor | None, device=None):
    """Rows [begin, end) of every S-row unit (pads skipped) and per-unit offsets (total at [U])."""
    dev = is_pad.device if is_pad is not None else device
    rows = torch.empty(max(U * (end - begin), 1), device=dev, dtype=torch.int32)
    offs = torch.empty(U + 1, device=dev, dtype=torch.int32)
    _lib.call("zs_unit_span_rows", U, S, begin, end, _ptr(is_pad), _ptr(rows), _ptr(offs), _stream())
    return rows[: U * (end - begin)], offs


def prefix_keep_rows(U: int, S: int, K: int, is_pad: torch.Tensor | None, device=None):
    """Kept rows (first K of every S-row unit, pads skipped) and per-unit offsets (total at [U])."""
    return unit_span_rows(U, S, 0, K, is_pad, device)


# ------------------------------------------------------------------ attention
def stripe_attn(
    q: torch.Tensor,
    k: torch.Tensor,
    v: torch.Tensor,
    *,
    units: int,
    heads: int,
    sq: int,
    sk: int,
    dh: int,
    bh: torch.Tensor | None,
    bw: torch.Tensor | None,
    q_sp: torch.Tensor,
    k_sp: torch.Tensor,
    b_row: int,
    b_col: int,
    prefix: int,
    tau: float,
    out: torch.Tensor | None = None,
    q_unit_stride: int | None = None,
    kv_unit_stride: int | None = None,
    o_rows: torch.Tensor | None = None,
    rel_pos: tuple[torch.Tensor, torch.Tensor] | None = None,
    ws: torch.Tensor | None = None,
) -> torch.Tensor:
    """Block-sparse stripe attention.  q/k/v are row-major views ``[units*S, ld]``
    whose head ``h`` lives at columns ``h*dh``; ``out`` is ``[units*sq, heads*dh]``, or, with
    ``o_rows`` (int32 ``[units*sq]``), query row r of unit u goes to ``out[o_rows[u*sq + r]]``
    and is skipped where ``o_rows < 0``.

    Bias: ``bh``/``bw`` fp32 ``[heads, S, w]`` (one table pair, the reference's BiasTables) or
    ``[units, heads, S, w]`` (one pair per unit); or ``rel_pos=(rel_pos_h, rel_pos_w)`` (fp32
    ``[2w-1, dh]``, bh = bw = None): SAM's q-dependent decomposed bias, computed on the fly.

    ``ws``: the caller-owned uint8 workspace (``attn_ws_bytes`` / ``relpos_ws_bytes``); when None
    one is taken from torch's stream-ordered caching allocator for this call (no sync, safe
    across streams, kept alive by a CUDA graph that captures the call)."""
    for t, n in ((q, "q"), (k, "k"), (v, "v")):
        _need(t, torch.bfloat16, n)
        if t.stride(-1) != 1:
            raise ValueError(f"{n} must be column-contiguous")
    _need(q_sp, torch.int32, "q_sp")
    _need(k_sp, torch.int32, "k_sp")
    if out is None:
        out = torch.empty((units * sq, heads * dh), device=q.device, dtype=torch.bfloat16)
    ldq, ldk, ldv = q.stride(0), k.stride(0), v.stride(0)
    qus = q_unit_stride if q_unit_stride is not None else sq * ldq
    kvus = kv_unit_stride if kv_unit_stride is not None else sk * ldk
    if o_rows is not None:
        _need(o_rows, torch.int32, "o_rows")
        if o_rows.numel() < units * sq:
            raise ValueError("o_rows must hold units*sq entries")
    if rel_pos is not None:
        rh, rw = (t.contiguous() for t in rel_pos)
        _need(rh, torch.float32, "rel_pos_h")
        _need(rw, torch.float32, "rel_pos_w")
        bias_w = (rh.shape[0] + 1) // 2
        if sq != sk or rh.shape != (2 * bias_w - 1, dh) or rw.shape != rh.shape:
            raise ValueError("rel_pos tables must be [2w-1, dh] with sq == sk == w*w")
        ws = _workspace(ws, relpos_ws_bytes(units, heads, sq, dh, bias_w), q.device)
        _lib.call(
            "zs_stripe_attn_fwd_relpos", _ptr(q), _ptr(k), _ptr(v), ldq, ldk, ldv, qus, kvus, units, heads, sq, dh,
            _ptr(rh), _ptr(rw), bias_w, _ptr(q_sp), _ptr(k_sp), b_row, b_col, prefix, float(tau), _ptr(out),
            out.stride(0), sq * out.stride(0), _ptr(o_rows) if o_rows is not None else None, _ptr(ws), ws.numel(),
            _stream(),
        )
        return out
    _need(bh, torch.float32, "bh")
    _need(bw, torch.float32, "bw")
    bias_w = bh.shape[-1]
    if bh.dim() == 4:
        if bh.shape[0] != units or bw.shape != bh.shape:
            raise ValueError("per-unit bias tables must be [units, heads, S, w]")
        bh, bw = bh.contiguous(), bw.contiguous()
        ws = _workspace(ws, attn_ws_bytes(units, heads, sq, sk, dh, per_unit=True), q.device)
        _lib.call(
            "zs_stripe_attn_fwd_unit_bias", _ptr(q), _ptr(k), _ptr(v), ldq, ldk, ldv, qus, kvus, units, heads, sq, sk,
            dh, _ptr(bh), _ptr(bw), bh[0].numel(), bias_w, _ptr(q_sp), _ptr(k_sp), b_row, b_col, prefix, float(tau),
            _ptr(out), out.stride(0), sq * out.stride(0), _ptr(o_rows) if o_rows is not None else None, _ptr(ws),
            ws.numel(), _stream(),
        )
        return out
    ws = _workspace(ws, attn_ws_bytes(units, heads, sq, sk, dh), q.device)
    if o_rows is None:
        _lib.call(
            "zs_stripe_attn_fwd", _ptr(q), _ptr(k), _ptr(v), ldq, ldk, ldv, qus, kvus, units, heads, sq, sk, dh,
            _ptr(bh.contiguous()), _ptr(bw.contiguous()), bias_w, _ptr(q_sp), _ptr(k_sp), b_row, b_col, prefix,
            float(tau), _ptr(out), out.stride(0), sq * out.stride(0), _ptr(ws), ws.numel(), _stream(),
        )
    else:
        _lib.call(
            "zs_stripe_attn_fwd_rows", _ptr(q), _ptr(k), _ptr(v), ldq, ldk, ldv, qus, kvus, units, heads, sq, sk, dh,
            _ptr(bh.contiguous()), _ptr(bw.contiguous()), bias_w, _ptr(q_sp), _ptr(k_sp), b_row, b_col, prefix,
            float(tau), _ptr(out), out.stride(0), sq * out.stride(0), _ptr(o_rows), _ptr(ws), ws.numel(), _stream(),
        )
    return out


def attn_ws_bytes(units: int, heads: int, sq: int, sk: int, dh: int, per_unit: bool = False) -> int:
    """Bytes of the attention's caller-owned workspace (zs_stripe_attn_ws_bytes)."""
    return int(_lib.load().zs_stripe_attn_ws_bytes(units, heads, sq, sk, dh, 1 if per_unit else 0))


def relpos_ws_bytes(units: int, heads: int, S: int, dh: int, bias_w: int) -> int:
    """Bytes of the SAM rel-pos path's caller-owned workspace (zs_relpos_ws_bytes)."""
    need = int(_lib.load().zs_relpos_ws_bytes(units, heads, S, dh, bias_w))
    if need <= 0:
        raise ValueError(f"rel-pos shape unsupported (dh={dh}, w={bias_w})")
    return need


def _workspace(ws: torch.Tensor | None, need: int, device) -> torch.Tensor:
    """The caller's workspace if large enough, else a fresh one from the caching allocator
    (allocated on the current stream; its 256-byte alignment is what the library requires)."""
    if ws is not None:
        _need(ws, torch.uint8, "ws")
        if ws.numel() < need:
            raise ValueError(f"workspace has {ws.numel()} bytes, the call needs {need}")
        if ws.data_ptr() % 256:
            raise ValueError("workspace must be 256-byte aligned")
        return ws
    return torch.empty(max(need, 256), dtype=torch.uint8, device=device)


def relpos_bias(q: torch.Tensor, *, units: int, heads: int, S: int, dh: int, rel_pos_h: torch.Tensor,
                rel_pos_w: torch.Tensor, q_sp: torch.Tensor, q_unit_stride: int | None = None):
    """SAM's decomposed rel-pos terms as per-unit BiasTables: (bh, bw) fp32 [units, heads, S, w],
    bh[u, h, s, ky] = q_h(row of s) . rel_pos_h[s // w - ky + w - 1] (unscaled q; s = q_sp[u, row])."""
    _need(q, torch.bfloat16, "q")
    _need(q_sp, torch.int32, "q_sp")
    rh, rw = rel_pos_h.contiguous(), rel_pos_w.contiguous()
    _need(rh, torch.float32, "rel_pos_h")
    _need(rw, torch.float32, "rel_pos_w")
    w = (rh.shape[0] + 1) // 2
    bh = torch.empty((units, heads, S, w), device=q.device, dtype=torch.float32)
    bw = torch.empty_like(bh)
    ws = _workspace(None, relpos_ws_bytes(units, heads, S, dh, w), q.device)
    qus = q_unit_stride if q_unit_stride is not None else S * q.stride(0)
    _lib.call("zs_relpos_bias", _ptr(q), q.stride(0), qus, units, heads, S, dh, w, _ptr(rh), _ptr(rw), _ptr(q_sp),
              _ptr(bh), _ptr(bw), _ptr(ws), ws.numel(), _stream())
    return bh, bw


def invert_rows(rows: torch.Tensor, map_len: int, n_dev: torch.Tensor | None = None,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """``map[rows[i]] = i`` (i < n, n from ``n_dev`` when given), -1 elsewhere; ``map`` has ``map_len`` entries."""
    _need(rows, torch.int32, "rows")
    if n_dev is not None:
        _need(n_dev, torch.int32, "n_dev")
    if out is None:
        out = torch.empty(map_len, device=rows.device, dtype=torch.int32)
    _lib.call("zs_invert_rows", _ptr(rows), rows.numel(), _ptr(n_dev), _ptr(out), map_len, _stream())
    return out


def fill_flagged_rows(dst: torch.Tensor, src_row: torch.Tensor, flag: torch.Tensor) -> torch.Tensor:
    """``dst[r] = src_row`` for every row with ``flag[r] != 0`` (bf16 rows)."""
    _need(dst, torch.bfloat16, "dst")
    _need(src_row, torch.bfloat16, "src_row")
    _need(flag, torch.uint8, "flag")
    if dst.stride(1) != 1 or src_row.numel() < dst.shape[1] or flag.numel() < dst.shape[0]:
        raise ValueError("fill_flagged_rows shapes")
    _lib.call("zs_fill_flagged_rows_bf16", _ptr(dst), dst.stride(0), _ptr(src_row), _ptr(flag), dst.shape[0],
              dst.shape[1], _stream())
    return dst


# ------------------------------------------------------------------ RC-MLP
def rc_mlp(
    x: torch.Tensor,
    keep_rows: torch.Tensor,
    *,
    ln_g: torch.Tensor,
    ln_b: torch.Tensor,
    w1: torch.Tensor,
    b1: torch.Tensor,
    w2: torch.Tensor,
    b2: torch.Tensor,
    n_keep_dev: torch.Tensor | None = None,
    bypass_rows: torch.Tensor | None = None,
    n_bypass_dev: torch.Tensor | None = None,
    ws: torch.Tensor | None = None,
    eps: float = 1e-6,
) -> torch.Tensor:
    """In-place RC-MLP on the fp32 residual stream ``x``; returns ``x``."""
    _need(x, torch.float32, "x")
    _need(keep_rows, torch.int32, "keep_rows")
    C = x.shape[1]
    hidden = w1.shape[0]
    max_keep = keep_rows.numel()
    need = max_keep * (C + hidden)
    if ws is None or ws.numel() < need:
        ws = torch.empty(max(need, 1), device=x.device, dtype=torch.bfloat16)
    nb = 0 if bypass_rows is None else bypass_rows.numel()
    _lib.call("zs_rc_mlp_fwd", _ptr(x), x.stride(0), _ptr(keep_rows), max_keep, _ptr(n_keep_dev), C, hidden,
              _ptr(ln_g), _ptr(ln_b), eps, _ptr(w1), _ptr(b1), _ptr(w2), _ptr(b2), 1 if bypass_rows is not None else 0,
              _ptr(bypass_rows), nb, _ptr(n_bypass_dev), _ptr(ws), _stream())
    return x


# ------------------------------------------------------------------ SAM frame helpers
def patchify(img: torch.Tensor, patch: int) -> torch.Tensor:
    _need(img, torch.float32, "img")
    B, Cin, H, W = img.shape
    out = torch.empty((B * (H // patch) * (W // patch), Cin * patch * patch), device=img.device,
                      dtype=torch.bfloat16)
    _lib.call("zs_patchify", _ptr(img.contiguous()), B, Cin, H, W, patch, _ptr(out), _stream())
    return out


def im2col3x3(x: torch.Tensor) -> torch.Tensor:
    """[B, H, W, C] bf16 -> [B*H*W, 9*C], tap-major columns (ky, kx, c)."""
    _need(x, torch.bfloat16, "x")
    B, H, W, Cc = x.shape
    out = torch.empty((B * H * W, 9 * Cc), device=x.device, dtype=torch.bfloat16)
    _lib.call("zs_im2col3x3", _ptr(x.contiguous()), B, H, W, Cc, _ptr(out), _stream())
    return out
