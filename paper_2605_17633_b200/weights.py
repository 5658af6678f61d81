"""Device-resident block parameters in the layouts the B200 kernels consume.

Weight layout: every dense projection is stored nn.Linear-style ``[out, in]``
bf16 (K-major for the tcgen05 GEMM); the reference stores ``[in, out]`` fp32
(encoder.py:112-138, mlp.py:25-57), so conversion transposes once.  Biases,
LN affine parameters and the decomposed bias tables stay fp32; the tables of
all heads are stacked ``[heads, S_attn, w]``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .config import SAM_NECK, SAM_PATCH, EncoderConfig


@dataclass
class BlockParams:
    kind: str
    ln1_g: torch.Tensor
    ln1_b: torch.Tensor
    qkv_w: torch.Tensor  # [3C, C] bf16
    qkv_b: torch.Tensor  # [3C]
    proj_w: torch.Tensor  # [C, C] bf16
    proj_b: torch.Tensor
    bh: torch.Tensor | None  # [H, S_attn, w] fp32 static tables (reference BiasTables), or None
    bw: torch.Tensor | None
    ln2_g: torch.Tensor
    ln2_b: torch.Tensor
    w1: torch.Tensor  # [4C, C] bf16
    b1: torch.Tensor
    w2: torch.Tensor  # [C, 4C] bf16
    b2: torch.Tensor
    # SAM relative-position mode: fp32 [2w - 1, dh] tables shared by the
    # heads; the bias is then q-dependent (SAM add_decomposed_rel_pos) and bh / bw are None
    rel_pos_h: torch.Tensor | None = None
    rel_pos_w: torch.Tensor | None = None

    @property
    def side(self) -> int:
        """Side w of the attention grid (S = w * w)."""
        return int(self.bh.shape[-1]) if self.bh is not None else (int(self.rel_pos_h.shape[0]) + 1) // 2


def _f32(a, dev):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)).to(dev)


def _lin(w_in_out, dev):
    """[in, out] fp32 (reference layout) -> [out, in] bf16 contiguous."""
    return torch.as_tensor(np.ascontiguousarray(np.asarray(w_in_out, np.float32).T)).to(dev).bfloat16().contiguous()


def _get(obj, *names):
    for n in names:
        if hasattr(obj, n):
            return getattr(obj, n)
    raise AttributeError(f"{type(obj).__name__} has none of {names}")


def block_from_reference(blk, kind: str, device) -> BlockParams:
    """Convert one reference ``BlockWeights`` (or an oracle ``Block``) to device parameters.

    Duck-typed over both: reference names (ln_gamma, bias=(BiasTables,...), mlp.ln_gamma)
    and oracle names (g, bh/bw lists, mlp.g).
    """
    if hasattr(blk, "bias"):
        bh = np.stack([b.bh for b in blk.bias])
        bw = np.stack([b.bw for b in blk.bias])
    else:
        bh, bw = np.stack(blk.bh), np.stack(blk.bw)
    m = blk.mlp
    return BlockParams(
        kind=kind,
        ln1_g=_f32(_get(blk, "ln_gamma", "g"), device),
        ln1_b=_f32(_get(blk, "ln_beta", "b"), device),
        qkv_w=_lin(blk.qkv_w, device),
        qkv_b=_f32(blk.qkv_b, device),
        proj_w=_lin(blk.proj_w, device),
        proj_b=_f32(blk.proj_b, device),
        bh=_f32(bh, device),
        bw=_f32(bw, device),
        ln2_g=_f32(_get(m, "ln_gamma", "g"), device),
        ln2_b=_f32(_get(m, "ln_beta", "b"), device),
        w1=_lin(m.w1, device),
        b1=_f32(m.b1, device),
        w2=_lin(m.w2, device),
        b2=_f32(m.b2, device),
    )


def params_from_reference(blocks, cfg: EncoderConfig, device) -> list[BlockParams]:
    return [block_from_reference(b, k, device) for b, k in zip(blocks, cfg.layout)]


def random_params(cfg: EncoderConfig, device, seed: int = 0, rel_pos: bool = False,
                  rel_pos_std: float = 0.05) -> list[BlockParams]:
    """Seeded random weights with the reference's init statistics (encoder.py:192-229),
    drawn on the device (a ViT-H has 0.63 B parameters).  ``rel_pos``: SAM relative-position
    tables N(0, rel_pos_std) [2w - 1, dh] per block instead of the static bias tables."""
    g = torch.Generator(device=device).manual_seed(seed)
    d, hid, H = cfg.d, 4 * cfg.d, cfg.heads
    f32 = dict(device=device, dtype=torch.float32)

    def rn(shape, std):
        return torch.randn(shape, generator=g, **f32) * std

    out = []
    for kind in cfg.layout:
        s_attn, side = (cfg.window**2, cfg.window) if kind == "local" else (cfg.grid.n(), cfg.grid.h)
        out.append(
            BlockParams(
                kind=kind,
                ln1_g=torch.ones(d, **f32),
                ln1_b=torch.zeros(d, **f32),
                qkv_w=rn((3 * d, d), 0.5 / math.sqrt(d)).bfloat16(),
                qkv_b=torch.zeros(3 * d, **f32),
                proj_w=rn((d, d), 1.0 / math.sqrt(d)).bfloat16(),
                proj_b=torch.zeros(d, **f32),
                bh=None if rel_pos else rn((H, s_attn, side), 0.5),
                bw=None if rel_pos else rn((H, s_attn, side), 0.5),
                ln2_g=torch.ones(d, **f32),
                ln2_b=torch.zeros(d, **f32),
                w1=rn((hid, d), 1.0 / math.sqrt(d)).bfloat16(),
                b1=torch.zeros(hid, **f32),
                w2=rn((d, hid), 1.0 / math.sqrt(hid)).bfloat16(),
                b2=torch.zeros(d, **f32),
                rel_pos_h=rn((2 * side - 1, cfg.head_dim), rel_pos_std) if rel_pos else None,
                rel_pos_w=rn((2 * side - 1, cfg.head_dim), rel_pos_std) if rel_pos else None,
            )
        )
    return out


@dataclass
class FrameParams:
    """SAM frame around the blocks: patch embed, absolute position embedding, neck."""

    pe_w: torch.Tensor  # [C, 3*16*16] bf16 (Conv2d weight flattened (c, ky, kx))
    pe_b: torch.Tensor  # [C]
    pos: torch.Tensor  # [64*64, C] fp32
    neck1_w: torch.Tensor  # [256, C] bf16 (1x1 conv)
    neck_ln1_g: torch.Tensor
    neck_ln1_b: torch.Tensor
    neck2_w: torch.Tensor  # [256, 256*9] bf16 (3x3 conv flattened (c, ky, kx))
    neck_ln2_g: torch.Tensor
    neck_ln2_b: torch.Tensor


def random_frame(cfg: EncoderConfig, device, seed: int = 1) -> FrameParams:
    g = torch.Generator(device=device).manual_seed(seed)
    d = cfg.d
    f32 = dict(device=device, dtype=torch.float32)

    def rn(shape, std):
        return torch.randn(shape, generator=g, **f32) * std

    k_pe = 3 * SAM_PATCH * SAM_PATCH
    return FrameParams(
        pe_w=rn((d, k_pe), 1.0 / math.sqrt(k_pe)).bfloat16(),
        pe_b=torch.zeros(d, **f32),
        pos=rn((cfg.grid.n(), d), 0.02),
        neck1_w=rn((SAM_NECK, d), 1.0 / math.sqrt(d)).bfloat16(),
        neck_ln1_g=torch.ones(SAM_NECK, **f32),
        neck_ln1_b=torch.zeros(SAM_NECK, **f32),
        neck2_w=rn((SAM_NECK, SAM_NECK * 9), 1.0 / math.sqrt(SAM_NECK * 9)).bfloat16(),
        neck_ln2_g=torch.ones(SAM_NECK, **f32),
        neck_ln2_b=torch.zeros(SAM_NECK, **f32),
    )
