"""SparseSAM encoder on B200: the block loop of encoder.py:310-385 over device layouts.

Token layouts (rows of the fp32 residual stream, C columns):
  S  spatial   b*HW + y*W + x                       (input / output order)
  L  local     (b*nwin + w)*win^2 + i  = token sigma_w[b,w,i] of window w,
               pad tokens of the zero-padded grid included (kept at zero)
  G  global    b*HW + i                = token sigma_g[b,i]

Because LayerNorm, the projections and the MLP are row-wise, every block runs
directly in its scan-ordered layout: attention sees sigma-ordered Q/K/V rows
without any per-head gather, the RC-MLP keep-set is the first K rows of each
unit, and the residual stream only moves when consecutive blocks change kind
(one ``zs_permute_rows_f32`` per switch).  Local pads are re-zeroed by the
projection epilogue, which is exactly the reference's re-padding at every
local block (encoder.py:356); their MLP rows are skipped (output-exact, since
the crop discards them, encoder.py:366-368).

The orderings come once per image from the fp32 block-0 input
(encoder.py:334): Sobel saliency, z-group energy, stable rank,
stripe interleave — all on device, bit-exact with the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from .config import SAM_NECK, SAM_PATCH, EncoderConfig, RouterConfig
from .trace import NULL
from .weights import BlockParams, FrameParams


def attention_elements(S: int, tile: int, prefix: int) -> int:
    """E = sum_i sum_{j in J_i} |rows_i| * |cols_j|: score elements the static schedule requires."""
    T = -(-S // tile)

    def size(t):
        return min((t + 1) * tile, S) - t * tile

    total = 0
    for i in range(T):
        cols = set(range(min(prefix, T))) | {min(i, T - 1)}
        total += size(i) * sum(size(j) for j in cols)
    return total


def morton_order_np(h: int, w: int) -> np.ndarray:
    """Token index at each Morton rank (x bits even, y bits odd; grid.py:79-104).

    Host-side constant table built once per grid shape."""
    ys, xs = np.divmod(np.arange(h * w, dtype=np.uint64), np.uint64(w))

    def spread(v):
        v = v & np.uint64(0xFFFFFFFF)
        for s, m in ((16, 0x0000FFFF0000FFFF), (8, 0x00FF00FF00FF00FF), (4, 0x0F0F0F0F0F0F0F0F),
                     (2, 0x3333333333333333), (1, 0x5555555555555555)):
            v = (v | (v << np.uint64(s))) & np.uint64(m)
        return v

    codes = spread(xs) | (spread(ys) << np.uint64(1))
    return np.argsort(codes, kind="stable").astype(np.int64)


@dataclass
class Orderings:
    sigma_glob: torch.Tensor | None  # [B, HW] int32
    sigma_loc: torch.Tensor | None  # [B*nwin, win^2] int32
    maps: dict


def _pad_heads(blk: BlockParams, H: int, dh: int, dp: int) -> BlockParams:
    """``blk`` with every head widened from dh to dp columns (zeros): QKV weight rows / bias of
    Q, K and V, the proj weight's input columns and SAM rel-pos tables."""
    import dataclasses

    C = blk.qkv_w.shape[1]
    idx = (torch.arange(H, device=blk.qkv_w.device)[:, None] * dp + torch.arange(dh, device=blk.qkv_w.device)).reshape(-1)
    qkv_w = blk.qkv_w.new_zeros((3 * H * dp, C))
    qkv_b = blk.qkv_b.new_zeros(3 * H * dp)
    for part in range(3):
        qkv_w[part * H * dp + idx] = blk.qkv_w[part * H * dh:(part + 1) * H * dh]
        qkv_b[part * H * dp + idx] = blk.qkv_b[part * H * dh:(part + 1) * H * dh]
    proj_w = blk.proj_w.new_zeros((blk.proj_w.shape[0], H * dp))
    proj_w[:, idx] = blk.proj_w
    extra = {}
    if blk.rel_pos_h is not None:
        extra = dict(rel_pos_h=torch.nn.functional.pad(blk.rel_pos_h, (0, dp - dh)),
                     rel_pos_w=torch.nn.functional.pad(blk.rel_pos_w, (0, dp - dh)))
    return dataclasses.replace(blk, qkv_w=qkv_w, qkv_b=qkv_b, proj_w=proj_w, **extra)


class StripeSortEncoder:
    """Runs the SparseSAM block stack on a batch of fp32 token grids ``[B, H, W, C]``.

    ``mode="sparse"`` uses the per-block r / keep_fraction of ``cfg``;
    ``mode="dense"`` pins r = keep = 1 through the same kernels (the reference's
    dense twin, encoder.py:338-339).
    """

    def __init__(self, cfg: EncoderConfig, params: list[BlockParams], device="cuda"):
        if len(params) != len(cfg.layout):
            raise ValueError(f"{len(params)} weight sets for {len(cfg.layout)} blocks")
        hd = cfg.head_dim
        if hd > 80:
            raise ValueError(f"head dim {hd} > 80 unsupported by the B200 attention kernel")
        if cfg.d % 64:
            raise ValueError("model width must be a multiple of 64 for the tcgen05 GEMMs")
        # heads narrower than the attention kernel's 64 / 80 run zero-padded: Q / K / V columns
        # [h * dp + dh, (h + 1) * dp) are zero (zero QKV weight rows and bias), the proj weight has
        # zero input columns there, tau stays 1 / sqrt(dh) — the same math as the unpadded heads
        self.dh = hd
        self.dp = 64 if hd <= 64 else 80
        self.Cq = cfg.heads * self.dp
        if self.Cq % 64:
            raise ValueError(f"{cfg.heads} heads of {self.dp} (padded) columns: width not a multiple of 64")
        self.cfg = cfg
        self.params = params if self.dp == hd else [_pad_heads(b, cfg.heads, hd, self.dp) for b in params]
        self.device = torch.device(device)
        g = cfg.grid
        self.HW = g.n()
        self.win = cfg.window
        self.S2 = cfg.window**2
        self.nwin = cfg.nwin()
        i32 = dict(device=self.device, dtype=torch.int32)
        self.morton_g = torch.as_tensor(morton_order_np(g.h, g.w)).to(**i32)
        self.morton_w = torch.as_tensor(morton_order_np(cfg.window, cfg.window)).to(**i32)
        self._ws: dict = {}
        self._ws_B = None
        self._pad_rows: dict = {}
        self.has_local = "local" in cfg.layout
        self.has_global = "global" in cfg.layout
        self.tracer = NULL
        # list -> (start, end) CUDA events of every block are appended to it
        self.block_events: list | None = None

    # ------------------------------------------------------------ workspace
    def swap_state(self, state: tuple | None) -> tuple:
        """Install ``state`` (None = fresh, empty) as this encoder's workspaces and return the
        previous ones.  A CUDA graph records raw pointers, so GraphedImageEncoder captures with a
        private state that later eager calls (another batch size, mode="dense", a larger keep
        set) can neither reallocate nor share."""
        old = (self._ws, self._ws_B)
        self._ws, self._ws_B = state if state is not None else ({}, None)
        return old

    def _workspace(self, B: int) -> dict:
        if self._ws_B == B:
            return self._ws
        C = self.cfg.d
        dev = self.device
        RL = B * self.nwin * self.S2 if self.has_local else 0
        RG = B * self.HW
        R = max(RL, RG)
        ws = dict(
            h=torch.empty((R, C), device=dev, dtype=torch.bfloat16),
            qkv=torch.empty((R, 3 * self.Cq), device=dev, dtype=torch.bfloat16),
            o=torch.empty((R, self.Cq), device=dev, dtype=torch.bfloat16),
            mlp=torch.empty((0,), device=dev, dtype=torch.bfloat16),
        )
        self._ws, self._ws_B = ws, B
        return ws

    # ------------------------------------------------------------ ordering
    def orderings(self, x0: torch.Tensor) -> Orderings:
        """sigma_global / sigma_local from the fp32 block-0 input ``x0[B,H,W,C]`` (encoder.py:257-275)."""
        cfg = self.cfg
        B = x0.shape[0]
        sg, sw = K.sobel_saliency(x0, self.win, glob=self.has_global, win=self.has_local)
        kw = dict(granularity=cfg.ordering.granularity, group_size=cfg.ordering.group_size, g=cfg.stripe.g,
                  variant=cfg.stripe.variant)
        sig_g = K.rank_order(sg.reshape(B, self.HW), self.morton_g, **kw)[0] if self.has_global else None
        sig_l = K.rank_order(sw.reshape(B * self.nwin, self.S2), self.morton_w, **kw)[0] if self.has_local else None
        maps = K.layout_maps(sig_g, sig_l, B, cfg.grid.h, cfg.grid.w, self.win)
        return Orderings(sig_g, sig_l, maps)

    def _row_sets(self, B: int, od: Orderings, mode: str) -> dict:
        """Keep-set (σ prefix) and bypass rows per distinct (kind, K), device-side counts."""
        cfg = self.cfg
        sets = {}
        for bi, kind in enumerate(cfg.layout):
            kf = 1.0 if mode == "dense" else cfg.keep_fraction[bi]
            S = self.S2 if kind == "local" else self.HW
            U = B * self.nwin if kind == "local" else B
            Kc = RouterConfig(kf, cfg.bypass_mode).keep_count(S)
            key = (kind, Kc)
            if key in sets:
                continue
            pad = od.maps.get("l_is_pad") if kind == "local" else None
            keep, koff = K.unit_span_rows(U, S, 0, Kc, pad, self.device)
            entry = dict(keep=keep, n_keep=koff[U:U + 1], max_keep=U * Kc)
            if cfg.bypass_mode == "layernorm" and Kc < S:
                byp, boff = K.unit_span_rows(U, S, Kc, S, pad, self.device)
                entry.update(bypass=byp, n_bypass=boff[U:U + 1])
            sets[key] = entry
        need = max(e["max_keep"] for e in sets.values()) * 5 * cfg.d
        ws = self._ws
        if ws["mlp"].numel() < need:
            ws["mlp"] = torch.empty((need,), device=self.device, dtype=torch.bfloat16)
        if self.has_local and "l_is_pad" in od.maps:
            # window pad tokens: LN1 / QKV / proj run on the non-pad rows only (their outputs are
            # cropped, encoder.py:366-368); the pads' K/V rows are the constant QKV row of LN(0)
            U, S = B * self.nwin, self.S2
            rows, offs = K.unit_span_rows(U, S, 0, S, od.maps["l_is_pad"], self.device)
            sets["nonpad"] = dict(rows=rows, n=offs[U:U + 1], max=U * S,
                                  omap=K.invert_rows(rows, U * S, n_dev=offs[U:U + 1]))
        # the residual stream stays in spatial row order for the whole forward: every row set of a
        # block's scan order is composed with that order's spatial row map (slots past the device
        # count hold unused garbage: clamped, never read by the kernels)
        m = od.maps

        def to_spatial(rows_, kind):
            mp = m["l_from_s"] if kind == "local" else m["g_from_s"]
            return mp[rows_.clamp(0, mp.numel() - 1).long()]

        for key, e in sets.items():
            if key == "nonpad":
                e["rows_s"] = to_spatial(e["rows"], "local")
                continue
            e["keep_s"] = to_spatial(e["keep"], key[0])
            if "bypass" in e:
                e["bypass_s"] = to_spatial(e["bypass"], key[0])
        return sets

    def _pad_qkv_row(self, blk: BlockParams) -> torch.Tensor:
        """QKV row of a zero-padded window token: LN(0) = beta exactly, so bf16(beta) @ Wqkv^T + b,
        the same tcgen05 GEMM row the full-width QKV would compute.  Depends on the weights only:
        computed once per block and cached."""
        key = id(blk)
        row = self._pad_rows.get(key)
        if row is None:
            C = self.cfg.d
            hz = K.layernorm_rows(torch.zeros((1, C), device=self.device, dtype=torch.float32), blk.ln1_g, blk.ln1_b)
            row = K.gemm(hz, blk.qkv_w, blk.qkv_b)
            self._pad_rows[key] = row
        return row

    # ------------------------------------------------------------ blocks
    def _block(self, blk: BlockParams, x: torch.Tensor, od: Orderings, B: int, r: float, rows: dict,
               ws: dict, nonpad: dict | None = None) -> None:
        cfg = self.cfg
        C, H, dh, dp, Cq = cfg.d, cfg.heads, self.dh, self.dp, self.Cq
        local = blk.kind == "local"
        S = self.S2 if local else self.HW
        U = B * self.nwin if local else B
        R = U * S
        tile = cfg.tile(blk.kind)
        T = -(-S // tile)
        prefix = math.floor(r * T)
        sig = od.sigma_loc if local else od.sigma_glob
        xs = x  # the spatial residual rows (every access goes through a row map)
        tr = self.tracer
        w = blk.side
        E = attention_elements(S, tile, prefix)
        bias = (dict(bh=None, bw=None, rel_pos=(blk.rel_pos_h, blk.rel_pos_w)) if blk.rel_pos_h is not None
                else dict(bh=blk.bh, bw=blk.bw))
        if nonpad is not None:
            # non-pad rows only (compacted), pad K/V rows = the constant row of LN(0) = beta
            npr, nps, nn, mx = nonpad["rows"], nonpad["rows_s"], nonpad["n"], nonpad["max"]
            with tr.span("layernorm", bytes=(nn, C * 6)):
                h = K.layernorm_rows(xs, blk.ln1_g, blk.ln1_b, nps, out=ws["h"][:mx], n_dev=nn)
            with tr.span("gemm_qkv", flops=(nn, 2.0 * C * 3 * C)):
                qkv = K.gemm(h, blk.qkv_w, blk.qkv_b, out=ws["qkv"][:R], row_map=npr, m_dev=nn)
                # K and V columns only: pad tokens are keys / values of the window, but their own
                # query rows are dropped (o_rows), so their Q part is never needed
                K.fill_flagged_rows(qkv[:, Cq:], self._pad_qkv_row(blk)[0, Cq:], od.maps["l_is_pad"])
            with tr.span(f"attn_{blk.kind}", flops=4.0 * dh * E * U * H,
                         bytes=U * H * 4 * S * dh * 2 + H * 2 * S * w * 4):
                o = K.stripe_attn(qkv[:, :Cq], qkv[:, Cq:2 * Cq], qkv[:, 2 * Cq:], units=U, heads=H, sq=S, sk=S, dh=dp,
                                  q_sp=sig, k_sp=sig, b_row=tile, b_col=tile, prefix=prefix,
                                  tau=1.0 / math.sqrt(dh), out=ws["o"][:R], o_rows=nonpad["omap"], **bias)
            with tr.span("gemm_proj", flops=(nn, 2.0 * C * C)):
                K.gemm(o[:mx], blk.proj_w, blk.proj_b, epi=K.EPI_F32_RESID, out=xs, res=xs, row_map=nps, m_dev=nn)
        else:
            g2s = od.maps["g_from_s"] if not local else od.maps["l_from_s"]  # scan-order row -> spatial row
            with tr.span("layernorm", bytes=R * C * 6):
                h = K.layernorm_rows(xs, blk.ln1_g, blk.ln1_b, g2s, out=ws["h"][:R])
            with tr.span("gemm_qkv", flops=2.0 * R * C * 3 * C, bytes=R * C * 2 + 3 * C * C * 2 + R * 3 * C * 2):
                qkv = K.gemm(h, blk.qkv_w, blk.qkv_b, out=ws["qkv"][:R])
            with tr.span(f"attn_{blk.kind}", flops=4.0 * dh * E * U * H,
                         bytes=U * H * 4 * S * dh * 2 + H * 2 * S * w * 4):
                o = K.stripe_attn(qkv[:, :Cq], qkv[:, Cq:2 * Cq], qkv[:, 2 * Cq:], units=U, heads=H, sq=S, sk=S, dh=dp,
                                  q_sp=sig, k_sp=sig, b_row=tile, b_col=tile, prefix=prefix,
                                  tau=1.0 / math.sqrt(dh), out=ws["o"][:R], **bias)
            with tr.span("gemm_proj", flops=2.0 * R * C * C, bytes=R * C * 2 + C * C * 2 + R * C * 8):
                K.gemm(o, blk.proj_w, blk.proj_b, epi=K.EPI_F32_RESID, out=xs, res=xs, row_map=g2s)
        # RC-MLP (mlp.py:88-114): gather-LN of the kept rows -> fc1 + GELU -> fc2 + scatter-add residual
        nk = rows["n_keep"]
        mk = rows["max_keep"]
        hidden = blk.w1.shape[0]
        hln = ws["mlp"][: mk * C].view(mk, C)
        hid = ws["mlp"][mk * C: mk * (C + hidden)].view(mk, hidden)
        with tr.span("mlp_ln", bytes=(nk, C * 6)):
            K.layernorm_rows(xs, blk.ln2_g, blk.ln2_b, rows["keep_s"], out=hln, n_dev=nk)
        with tr.span("gemm_fc1", flops=(nk, 2.0 * C * hidden)):
            K.gemm(hln, blk.w1, blk.b1, epi=K.EPI_BF16_GELU, out=hid, m_dev=nk)
        with tr.span("gemm_fc2", flops=(nk, 2.0 * C * hidden)):
            K.gemm(hid, blk.w2, blk.b2, epi=K.EPI_F32_RESID, out=xs, res=xs, row_map=rows["keep_s"], m_dev=nk)
        if "bypass" in rows:
            with tr.span("mlp_ln", bytes=(rows["n_bypass"], C * 8)):
                K.layernorm_rows(xs, blk.ln2_g, blk.ln2_b, rows["bypass_s"], out_f32=True, out=xs,
                                 out_rows=rows["bypass_s"], n_dev=rows["n_bypass"])

    def forward_rows(self, x0: torch.Tensor, mode: str = "sparse", orderings: Orderings | None = None,
                     out: torch.Tensor | None = None) -> torch.Tensor:
        """fp32 ``x0[B,H,W,C]`` -> fp32 ``[B*H*W, C]`` spatial rows after every block."""
        if mode not in ("dense", "sparse"):
            raise ValueError(f"mode must be 'dense' or 'sparse', got {mode!r}")
        cfg = self.cfg
        if x0.dim() != 4 or tuple(x0.shape[1:]) != (cfg.grid.h, cfg.grid.w, cfg.d):
            raise ValueError(f"input shape {tuple(x0.shape)} != (B, {cfg.grid.h}, {cfg.grid.w}, {cfg.d})")
        if x0.dtype != torch.float32 or not x0.is_cuda:
            raise ValueError("x0 must be a float32 CUDA tensor")
        x0 = x0.contiguous()
        B = x0.shape[0]
        ws = self._workspace(B)
        if orderings is None:
            with self.tracer.span("ordering", bytes=x0.numel() * 4):
                orderings = self.orderings(x0)
        od = orderings
        rows = self._row_sets(B, od, mode)
        flat = x0.reshape(B * self.HW, cfg.d)
        # the residual stream lives in spatial row order in `out` for the whole forward (every
        # block reads and writes it through its scan order's row maps: no layout permutes);
        # out may be x0 itself (in place, after the orderings were taken from it)
        if out is None:
            out = torch.empty((B * self.HW, cfg.d), device=self.device, dtype=torch.float32)
        if out.data_ptr() != flat.data_ptr():
            out.copy_(flat)
        for bi, blk in enumerate(self.params):
            kind = blk.kind
            if self.block_events is not None:  # per-block device time (CostReport.ms, encoder.py:342,372)
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
                self.block_events.append(ev)
            r = 1.0 if mode == "dense" else cfg.r[bi]
            kf = 1.0 if mode == "dense" else cfg.keep_fraction[bi]
            S = self.S2 if kind == "local" else self.HW
            Kc = RouterConfig(kf, cfg.bypass_mode).keep_count(S)
            self._block(blk, out, od, B, r, rows[(kind, Kc)], ws, rows.get("nonpad") if kind == "local" else None)
            if self.block_events is not None:
                self.block_events[-1][1].record()
        return out

    def __call__(self, x0: torch.Tensor, mode: str = "sparse") -> torch.Tensor:
        B = x0.shape[0]
        return self.forward_rows(x0, mode).reshape(B, self.cfg.grid.h, self.cfg.grid.w, self.cfg.d)


class SparseSAMImageEncoder:
    """SAM ViT image encoder with SparseSAM blocks: 1024² image -> [B, 256, 64, 64].

    patch embed (16x16/16 conv as patchify + tcgen05 GEMM, bias and absolute
    position embedding fused in the epilogue) -> fp32 block-0 input (source of
    the orderings) -> SparseSAM blocks -> neck (1x1 conv GEMM, LN2d, 3x3 conv
    as im2col + GEMM, LN2d).  The frame is SAM's [ext]; parity for it is
    pinned by an fp32 torch twin (tests), the blocks by the reference oracle.
    """

    def __init__(self, cfg: EncoderConfig, params: list[BlockParams], frame: FrameParams, device="cuda"):
        self.cfg = cfg
        self.frame = frame
        self.core = StripeSortEncoder(cfg, params, device)
        self.device = self.core.device
        self._buf_B = None
        # 3x3 neck conv weight [256, 256*9] (c, ky, kx) -> tap-major (ky, kx, c) to match im2col3x3
        self._neck2_tap = (frame.neck2_w.view(SAM_NECK, SAM_NECK, 3, 3).permute(0, 2, 3, 1)
                           .reshape(SAM_NECK, 9 * SAM_NECK).contiguous())

    def swap_state(self, state: tuple | None) -> tuple:
        """Frame buffers + the block stack's workspaces (see StripeSortEncoder.swap_state)."""
        old = (getattr(self, "_bufs_d", None), self._buf_B, self.core.swap_state(None if state is None else state[2]))
        if state is None:
            self._bufs_d, self._buf_B = None, None
        else:
            self._bufs_d, self._buf_B = state[0], state[1]
            # state[2] was installed above
        return old

    def _bufs(self, B: int) -> dict:
        if self._buf_B != B:
            C, HW, dev = self.cfg.d, self.cfg.grid.n(), self.device
            self._bufs_d = dict(
                x0=torch.empty((B * HW, C), device=dev, dtype=torch.float32),
                xb16=torch.empty((B * HW, C), device=dev, dtype=torch.bfloat16),
                n1=torch.empty((B * HW, SAM_NECK), device=dev, dtype=torch.float32),
                n1b=torch.empty((B * HW, SAM_NECK), device=dev, dtype=torch.bfloat16),
                n2=torch.empty((B * HW, SAM_NECK), device=dev, dtype=torch.float32),
                out=torch.empty((B * HW, SAM_NECK), device=dev, dtype=torch.float32),
            )
            self._buf_B = B
        return self._bufs_d

    def embed(self, img: torch.Tensor) -> torch.Tensor:
        """fp32 NCHW image -> fp32 token grid rows [B*HW, C] (patch embed + pos)."""
        B = img.shape[0]
        bufs = self._bufs(B)
        patches = K.patchify(img, SAM_PATCH)
        f = self.frame
        K.gemm(patches, f.pe_w, f.pe_b, epi=K.EPI_F32_RESID, out=bufs["x0"], res=f.pos, res_mod=self.cfg.grid.n())
        return bufs["x0"]

    def neck(self, rows: torch.Tensor, B: int, out: torch.Tensor | None = None) -> torch.Tensor:
        f = self.frame
        bufs = self._bufs(B)
        g = self.cfg.grid
        xb = K.cast_rows_bf16(rows, out=bufs["xb16"])
        K.gemm(xb, f.neck1_w, None, epi=K.EPI_F32_RESID, out=bufs["n1"])
        K.layernorm_rows(bufs["n1"], f.neck_ln1_g, f.neck_ln1_b, out=bufs["n1b"])
        cols = K.im2col3x3(bufs["n1b"].view(B, g.h, g.w, SAM_NECK))  # tap-major (ky, kx, c) columns
        K.gemm(cols, self._neck2_tap, None, epi=K.EPI_F32_RESID, out=bufs["n2"])
        if out is None:
            out = bufs["out"]
        elif tuple(out.shape) not in ((B, g.h, g.w, SAM_NECK), (B * g.h * g.w, SAM_NECK)) or out.dtype != torch.float32:
            raise ValueError(f"out must be float32 [B, {g.h}, {g.w}, {SAM_NECK}]")
        K.layernorm_rows(bufs["n2"], f.neck_ln2_g, f.neck_ln2_b, out_f32=True, out=out.view(B * g.h * g.w, SAM_NECK))
        return out.view(B, g.h, g.w, SAM_NECK)

    def __call__(self, img: torch.Tensor, mode: str = "sparse", out: torch.Tensor | None = None) -> torch.Tensor:
        """[B, 3, 1024, 1024] fp32 -> channels-last embeddings [B, 64, 64, 256] fp32 (into ``out``
        when given, so a caller can double-buffer results while copying the previous ones out)."""
        B = img.shape[0]
        g = self.cfg.grid
        x0 = self.embed(img)
        xo = self.core.forward_rows(x0.view(B, g.h, g.w, self.cfg.d), mode, out=x0)  # in place
        return self.neck(xo, B, out=out)


class GraphedImageEncoder:
    """CUDA-graph replay of a :class:`SparseSAMImageEncoder` forward for a fixed batch size.

    The whole forward (patch embed, orderings, every block's ~9 launches, neck) has no host
    synchronisation (device-side row counts, caller-owned workspaces), so it is captured once into
    a CUDA graph over static input / output buffers and replayed: one graph launch instead of
    ~300 kernel launches from Python per call, which is what bounds small batches (one image).
    The graph owns private workspaces (``swap_state``): eager calls on the same encoder before or
    after the capture never reallocate or share the memory the graph replays into.
    """

    def __init__(self, enc: SparseSAMImageEncoder, batch: int, mode: str = "sparse"):
        g = enc.cfg.grid
        dev = enc.device
        self.enc, self.batch, self.mode = enc, batch, mode
        self.img = torch.zeros((batch, 3, g.h * SAM_PATCH, g.w * SAM_PATCH), device=dev, dtype=torch.float32)
        self.out = torch.empty((batch, g.h, g.w, SAM_NECK), device=dev, dtype=torch.float32)
        # warm-up and capture on the same side stream: the library's scratch is per (device,
        # stream), so everything the captured launches use is allocated before the capture
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        saved = enc.swap_state(None)
        try:
            with torch.cuda.stream(side):
                for _ in range(2):
                    enc(self.img, mode, out=self.out)
            side.synchronize()
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph, stream=side):
                enc(self.img, mode, out=self.out)
        finally:
            self._state = enc.swap_state(saved)  # the graph keeps its buffers alive, enc gets its own back
        torch.cuda.current_stream(dev).wait_stream(side)

    def __call__(self, img: torch.Tensor) -> torch.Tensor:
        """[batch, 3, H, W] fp32 -> the static output buffer [batch, 64, 64, 256] (valid until the
        next call)."""
        if tuple(img.shape) != tuple(self.img.shape):
            raise ValueError(f"graph captured for images of shape {tuple(self.img.shape)}, got {tuple(img.shape)}")
        self.img.copy_(img, non_blocking=True)
        self.graph.replay()
        return self.out
