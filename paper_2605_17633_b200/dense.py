"""Dense cuBLAS / cuDNN SAM encoder on the same B200 — the SPEED baseline.

Same weights and the same decomposed rel-pos bias semantics as the sparse
engine, but every block runs dense through library kernels in bf16:
LayerNorm (torch), QKV / proj / MLP GEMMs (cuBLAS via F.linear),
attention = F.scaled_dot_product_attention with the materialised additive
bias [H, S, S] (cuDNN / memory-efficient backend), SAM-style windowing (pad,
partition, unpartition, crop; MLP on the 4,096 cropped tokens).  It is not
on the product path: it exists so bench.py can report the sparse engine's
speed-up over a dense library encoder on the same GPU (BASELINE north star).
Its parity partner is the reference's ``mode="dense"`` twin; a test checks it
against the sparse engine run at r = keep = 1.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F

from .config import SAM_NECK, SAM_PATCH, EncoderConfig
from .weights import BlockParams, FrameParams


def dense_bias(bh: torch.Tensor, bw: torch.Tensor) -> torch.Tensor:
    """B[h, q, k] = bh[h, q, k // w] + bw[h, q, k % w]  (attention.py:46-55), spatial order."""
    H, S, w = bh.shape
    k = torch.arange(w * w, device=bh.device)
    return (bh[:, :, k // w] + bw[:, :, k % w]).to(torch.bfloat16).contiguous()


def sam_rel_pos_bias(q: torch.Tensor, rel_h: torch.Tensor, rel_w: torch.Tensor) -> torch.Tensor:
    """SAM add_decomposed_rel_pos as an additive mask: q [N, H, S, dh] (unscaled, spatial row-major
    order, S = w * w), rel_h / rel_w [2w - 1, dh] -> [N, H, S, S] bias in q's dtype."""
    N, H, S, dh = q.shape
    w = (rel_h.shape[0] + 1) // 2
    idx = torch.arange(w, device=q.device)
    rel = idx[:, None] - idx[None, :] + w - 1  # [qy, ky] -> table row
    Rh, Rw = rel_h.to(q.dtype)[rel], rel_w.to(q.dtype)[rel]  # [w, w, dh]
    r_q = q.reshape(N, H, w, w, dh)
    bh = torch.einsum("nhyxc,ykc->nhyxk", r_q, Rh)  # [N, H, qy, qx, ky]
    bw = torch.einsum("nhyxc,xkc->nhyxk", r_q, Rw)  # [N, H, qy, qx, kx]
    return (bh[..., :, None] + bw[..., None, :]).reshape(N, H, S, S)


class DenseSAMEncoder:
    def __init__(self, cfg: EncoderConfig, params: list[BlockParams], frame: FrameParams | None = None):
        self.cfg = cfg
        self.params = params
        self.frame = frame
        self.bias = [dense_bias(p.bh, p.bw) if p.rel_pos_h is None else None for p in params]

    def _attn(self, x, p: BlockParams, bias):
        # x [N, S, C] bf16
        N, S, C = x.shape
        H = self.cfg.heads
        dh = C // H
        h = F.layer_norm(x.float(), (C,), p.ln1_g, p.ln1_b, 1e-6).to(torch.bfloat16)
        qkv = F.linear(h, p.qkv_w, p.qkv_b.to(torch.bfloat16)).view(N, S, 3, H, dh).permute(2, 0, 3, 1, 4)
        if bias is None:  # SAM rel-pos mode: q-dependent bias
            mask = sam_rel_pos_bias(qkv[0], p.rel_pos_h, p.rel_pos_w)
        else:
            mask = bias[None].expand(N, -1, -1, -1)
        o = F.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2], attn_mask=mask)
        o = o.transpose(1, 2).reshape(N, S, C)
        return F.linear(o, p.proj_w, p.proj_b.to(torch.bfloat16))

    def _mlp(self, x, p: BlockParams):
        h = F.layer_norm(x.float(), (x.shape[-1],), p.ln2_g, p.ln2_b, 1e-6).to(torch.bfloat16)
        h = F.gelu(F.linear(h, p.w1, p.b1.to(torch.bfloat16)))
        return F.linear(h, p.w2, p.b2.to(torch.bfloat16))

    @torch.no_grad()
    def blocks(self, x: torch.Tensor) -> torch.Tensor:
        """x [B, H, W, C] -> [B, H, W, C]; residual stream kept in fp32."""
        cfg = self.cfg
        B, Hh, Ww, C = x.shape
        win = cfg.window
        hp, wp = -(-Hh // win) * win, -(-Ww // win) * win
        x = x.float()
        for p, bias in zip(self.params, self.bias):
            if p.kind == "global":
                t = x.view(B, Hh * Ww, C)
                t = t + self._attn(t.to(torch.bfloat16), p, bias).float()
                x = t.view(B, Hh, Ww, C)
            else:
                xp = F.pad(x, (0, 0, 0, wp - Ww, 0, hp - Hh))
                wins = xp.view(B, hp // win, win, wp // win, win, C).permute(0, 1, 3, 2, 4, 5).reshape(-1, win * win, C)
                a = self._attn(wins.to(torch.bfloat16), p, bias).float()
                a = a.view(B, hp // win, wp // win, win, win, C).permute(0, 1, 3, 2, 4, 5).reshape(B, hp, wp, C)
                x = x + a[:, :Hh, :Ww]
            x = x + self._mlp(x.to(torch.bfloat16), p).float()
        return x

    @torch.no_grad()
    def __call__(self, img: torch.Tensor) -> torch.Tensor:
        f = self.frame
        cfg = self.cfg
        B = img.shape[0]
        x = F.conv2d(img.to(torch.bfloat16), f.pe_w.view(cfg.d, 3, SAM_PATCH, SAM_PATCH), f.pe_b.to(torch.bfloat16),
                     stride=SAM_PATCH)
        x = x.permute(0, 2, 3, 1).float() + f.pos.view(1, cfg.grid.h, cfg.grid.w, cfg.d)
        x = self.blocks(x)
        t = x.to(torch.bfloat16).permute(0, 3, 1, 2)
        n = F.conv2d(t, f.neck1_w.view(SAM_NECK, cfg.d, 1, 1))
        n = F.layer_norm(n.permute(0, 2, 3, 1).float(), (SAM_NECK,), f.neck_ln1_g, f.neck_ln1_b, 1e-6)
        n = F.conv2d(n.to(torch.bfloat16).permute(0, 3, 1, 2), f.neck2_w.view(SAM_NECK, SAM_NECK, 3, 3), padding=1)
        n = F.layer_norm(n.permute(0, 2, 3, 1).float(), (SAM_NECK,), f.neck_ln2_g, f.neck_ln2_b, 1e-6)
        return n.view(B, cfg.grid.h, cfg.grid.w, SAM_NECK)
