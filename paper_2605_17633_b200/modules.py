"""PyTorch module API: SparseSAM drop-ins for segment_anything's image-encoder tree.

``SparseSAMImageEncoderViT`` / ``SparseSAMBlock`` / ``StripeSortAttention`` /
``ResidualConsistencyMLP`` have the constructor arguments, submodule names and parameter
shapes of SAM's ``ImageEncoderViT`` / ``Block`` / ``Attention`` / ``MLPBlock``
(``patch_embed.proj``, ``pos_embed``, ``blocks.{i}.norm1 / attn.qkv / attn.proj /
attn.rel_pos_h / attn.rel_pos_w / norm2 / mlp.lin1 / mlp.lin2``, ``neck.{0..3}``), so a SAM
image-encoder ``state_dict`` loads unchanged; the SparseSAM settings (attention density
``density`` = r, MLP ``keep_fraction``, ``bypass_mode``, tile sizes) are extra keyword
arguments.  The forward runs the B200 block engine (``encoder.StripeSortEncoder`` /
``encoder.SparseSAMImageEncoder``: hand-written sm_100a kernels through the C ABI); it is
inference-only (no autograd) and needs CUDA tensors.

Pad tokens: inside ``SparseSAMBlock`` / ``SparseSAMImageEncoderViT`` windows are padded before
norm1 as in the reference (encoder.py:356: a pad token's normalised row is LN(0) = beta); SAM's
own Block pads after norm1, so ``StripeSortAttention`` used inside a SAM Block sees zero rows.

Semantics follow the reference (encoder.py:278-385): stripe-sort
orderings from the encoder input, A-shape block-sparse attention (b_local = 32 /
b_global = 128 tiles, density r), residual-consistency MLP over the σ-prefix keep set.  With
``use_rel_pos`` the bias is SAM's q-dependent decomposed rel-pos, else the
reference's static ``BiasTables`` (buffers ``attn.bias_h`` / ``attn.bias_w``, zeros until set).
At density = keep_fraction = 1 a block computes SAM's dense Block.

The engine parameters are converted from the module tree on the first forward and cached;
any in-place parameter update (``load_state_dict``, optimizer step) bumps the tensors' version
counters and triggers a rebuild on the next forward.
"""

from __future__ import annotations

import math

import torch
from torch import nn

from . import kernels as K
from .config import SAM_NECK, EncoderConfig, GridShape, OrderingConfig, RouterConfig, StripeConfig
from .encoder import SparseSAMImageEncoder, StripeSortEncoder, _pad_heads, morton_order_np
from .weights import BlockParams, FrameParams

__all__ = ["StripeSortAttention", "ResidualConsistencyMLP", "SparseSAMBlock", "LayerNorm2d",
           "SparseSAMImageEncoderViT", "from_sam_image_encoder", "stripe_order"]


def _version_key(mod: nn.Module) -> tuple:
    return tuple((t.data_ptr(), t._version) for t in list(mod.parameters()) + list(mod.buffers()))


def stripe_order(x: torch.Tensor, ordering: OrderingConfig = OrderingConfig(),
                 stripe: StripeConfig = StripeConfig()) -> torch.Tensor:
    """Stripe-sort order σ [U, h*w] (int32) of every unit grid of fp32 ``x[U, h, w, C]`` from its own
    Sobel saliency (saliency.py:62-118, stripesort.py:38-62; zero padding at the unit border)."""
    U, h, w, _ = x.shape
    sal, _ = K.sobel_saliency(x.float().contiguous(), max(h, w), glob=True, win=False)
    morton = torch.as_tensor(morton_order_np(h, w)).to(device=x.device, dtype=torch.int32)
    return K.rank_order(sal.reshape(U, h * w), morton, granularity=ordering.granularity,
                        group_size=ordering.group_size, g=stripe.g, variant=stripe.variant)[0]


class StripeSortAttention(nn.Module):
    """SAM ``Attention`` (qkv / proj Linear, optional rel_pos_h / rel_pos_w) with stripe-sort
    block-sparse attention.  ``input_size`` is the attention grid (window or full grid)."""

    def __init__(self, dim: int, num_heads: int = 8, qkv_bias: bool = True, use_rel_pos: bool = False,
                 rel_pos_zero_init: bool = True, input_size: tuple[int, int] | None = None, *,
                 density: float = 0.4):
        super().__init__()
        if input_size is None or input_size[0] != input_size[1]:
            raise ValueError("StripeSortAttention needs a square input_size (the decomposed bias grid)")
        self.num_heads = num_heads
        head_dim = dim // num_heads
        self.scale = head_dim**-0.5
        self.qkv = nn.Linear(dim, dim * 3, bias=qkv_bias)
        self.proj = nn.Linear(dim, dim)
        self.use_rel_pos = use_rel_pos
        self.input_size = tuple(input_size)
        self.density = float(density)
        w = input_size[0]
        if use_rel_pos:
            self.rel_pos_h = nn.Parameter(torch.zeros(2 * w - 1, head_dim))
            self.rel_pos_w = nn.Parameter(torch.zeros(2 * w - 1, head_dim))
            if not rel_pos_zero_init:
                nn.init.trunc_normal_(self.rel_pos_h, std=0.02)
                nn.init.trunc_normal_(self.rel_pos_w, std=0.02)
        else:
            # the reference's static decomposed bias (BiasTables, attention.py:28-55), one per head
            self.register_buffer("bias_h", torch.zeros(num_heads, w * w, w))
            self.register_buffer("bias_w", torch.zeros(num_heads, w * w, w))
        self.tile = 32 if w * w <= 256 else 128  # the reference's b_local / b_global (encoder.py:57-58)
        self._w = None
        self._key = None

    def _weights(self):
        key = _version_key(self)
        if self._w is None or self._key != key:
            C, H = self.qkv.in_features, self.num_heads
            dh = C // H
            bp = BlockParams(kind="", ln1_g=None, ln1_b=None, qkv_w=self.qkv.weight.detach().to(torch.bfloat16),
                             qkv_b=(self.qkv.bias.detach().float() if self.qkv.bias is not None
                                    else torch.zeros(3 * C, device=self.qkv.weight.device)),
                             proj_w=self.proj.weight.detach().to(torch.bfloat16), proj_b=self.proj.bias.detach().float(),
                             bh=None, bw=None, ln2_g=None, ln2_b=None, w1=None, b1=None, w2=None, b2=None,
                             rel_pos_h=self.rel_pos_h.detach().float() if self.use_rel_pos else None,
                             rel_pos_w=self.rel_pos_w.detach().float() if self.use_rel_pos else None)
            dp = 64 if dh <= 64 else 80
            if dh > 80:
                raise ValueError(f"head dim {dh} > 80 unsupported by the B200 attention kernel")
            if dp != dh:
                bp = _pad_heads(bp, H, dh, dp)
            self._w = (bp, dp)
            self._key = key
        return self._w

    @torch.no_grad()
    def forward(self, x: torch.Tensor, order: torch.Tensor | None = None) -> torch.Tensor:
        """``x[U, h, w, C]`` (windows or whole grids, CUDA) -> ``[U, h, w, C]`` fp32, SAM's
        Attention output computed as stripe-sort attention: rows in σ order (``order`` [U, h*w]
        int32, else from the input's saliency), A-shape schedule at ``density``, output
        scattered back to the spatial rows by the proj GEMM."""
        if x.dim() != 4 or not x.is_cuda or tuple(x.shape[1:3]) != self.input_size:
            raise ValueError(f"expected a CUDA tensor [U, {self.input_size[0]}, {self.input_size[1]}, C]")
        U, h, w, C = x.shape
        S, H = h * w, self.num_heads
        bp, dp = self._weights()
        Cq = H * dp
        rows = x.float().reshape(U * S, C).contiguous()
        sig = stripe_order(x) if order is None else order.to(torch.int32).reshape(U, S).contiguous()
        base = (torch.arange(U, device=x.device, dtype=torch.int32) * S)[:, None]
        sp_rows = (base + sig).reshape(-1).contiguous()  # σ-order row i of unit u -> spatial row
        hq = K.cast_rows_bf16(rows, sp_rows)
        qkv = K.gemm(hq, bp.qkv_w, bp.qkv_b)
        T = -(-S // self.tile)
        bias = (dict(bh=None, bw=None, rel_pos=(bp.rel_pos_h, bp.rel_pos_w)) if self.use_rel_pos
                else dict(bh=self.bias_h.float().contiguous(), bw=self.bias_w.float().contiguous()))
        o = K.stripe_attn(qkv[:, :Cq], qkv[:, Cq:2 * Cq], qkv[:, 2 * Cq:], units=U, heads=H, sq=S, sk=S, dh=dp,
                          q_sp=sig, k_sp=sig, b_row=self.tile, b_col=self.tile, prefix=math.floor(self.density * T),
                          tau=self.scale, **bias)
        y = torch.empty((U * S, C), device=x.device, dtype=torch.float32)
        K.gemm(o, bp.proj_w, bp.proj_b, epi=K.EPI_F32_RESID, out=y, row_map=sp_rows)
        return y.view(U, h, w, C)


class ResidualConsistencyMLP(nn.Module):
    """SAM ``MLPBlock`` parameters (lin1 / lin2, GELU) with residual-consistency routing: only
    the σ-prefix ``keep_fraction`` of each unit's tokens run the MLP (mlp.py:78-114)."""

    def __init__(self, embedding_dim: int, mlp_dim: int, act: type[nn.Module] = nn.GELU, *,
                 keep_fraction: float = 0.4, bypass_mode: str = "identity"):
        super().__init__()
        if act is not nn.GELU:
            raise ValueError("the RC-MLP kernel implements the exact-erf GELU (tensor.py:239-243)")
        self.lin1 = nn.Linear(embedding_dim, mlp_dim)
        self.lin2 = nn.Linear(mlp_dim, embedding_dim)
        self.act = act()
        self.keep_fraction = float(keep_fraction)
        self.bypass_mode = bypass_mode
        self._w = None
        self._key = None

    @torch.no_grad()
    def forward(self, x: torch.Tensor, order: torch.Tensor | None = None) -> torch.Tensor:
        """SAM's ``MLPBlock`` contract (``Block`` adds the result to its residual): ``x[B, H, W, C]``
        (= norm2 of the residual) -> lin2(GELU(lin1(x))) on the σ-prefix ``keep_fraction`` of each
        image's tokens and 0 on the others, i.e. the identity bypass of mlp.py:99-114 once added.
        ``order`` [B, H*W] int32 (else from the input's saliency)."""
        if self.bypass_mode != "identity":
            raise ValueError("as a SAM MLPBlock replacement only the identity bypass is expressible; "
                             "SparseSAMBlock runs the layernorm bypass")
        if x.dim() != 4 or not x.is_cuda:
            raise ValueError("expected a CUDA tensor [B, H, W, C]")
        B, Hh, Ww, C = x.shape
        S = Hh * Ww
        key = _version_key(self)
        if self._w is None or self._key != key:
            self._w = (self.lin1.weight.detach().to(torch.bfloat16), self.lin1.bias.detach().float(),
                       self.lin2.weight.detach().to(torch.bfloat16), self.lin2.bias.detach().float())
            self._key = key
        w1, b1, w2, b2 = self._w
        sig = stripe_order(x) if order is None else order.to(torch.int32).reshape(B, S)
        kc = RouterConfig(self.keep_fraction, "identity").keep_count(S)
        base = (torch.arange(B, device=x.device, dtype=torch.int32) * S)[:, None]
        keep = (base + sig[:, :kc]).reshape(-1).contiguous()
        hk = K.cast_rows_bf16(x.float().reshape(B * S, C).contiguous(), keep)
        hid = K.gemm(hk, w1, b1, epi=K.EPI_BF16_GELU)
        y = torch.zeros((B * S, C), device=x.device, dtype=torch.float32)
        K.gemm(hid, w2, b2, epi=K.EPI_F32_RESID, out=y, row_map=keep)
        return y.view(B, Hh, Ww, C)


class SparseSAMBlock(nn.Module):
    """SAM ``Block``: norm1 -> (window partition) -> attention -> residual -> norm2 -> MLP ->
    residual, as a SparseSAM block (stripe-sort attention + RC-MLP).  ``forward(x[B, H, W, C])``;
    run standalone, the block takes its orderings from its own input (inside
    ``SparseSAMImageEncoderViT`` they come from the encoder input, as in the reference)."""

    def __init__(self, dim: int, num_heads: int, mlp_ratio: float = 4.0, qkv_bias: bool = True,
                 norm_layer: type[nn.Module] = nn.LayerNorm, act_layer: type[nn.Module] = nn.GELU,
                 use_rel_pos: bool = False, rel_pos_zero_init: bool = True, window_size: int = 0,
                 input_size: tuple[int, int] | None = None, *, density: float = 0.4, keep_fraction: float = 0.4,
                 bypass_mode: str = "identity", b_local: int = 32, b_global: int = 128):
        super().__init__()
        self.norm1 = norm_layer(dim, eps=1e-6) if norm_layer is nn.LayerNorm else norm_layer(dim)
        self.attn = StripeSortAttention(dim, num_heads, qkv_bias, use_rel_pos, rel_pos_zero_init,
                                        input_size if window_size == 0 else (window_size, window_size),
                                        density=density)
        self.norm2 = norm_layer(dim, eps=1e-6) if norm_layer is nn.LayerNorm else norm_layer(dim)
        self.mlp = ResidualConsistencyMLP(dim, int(dim * mlp_ratio), act_layer, keep_fraction=keep_fraction,
                                          bypass_mode=bypass_mode)
        self.window_size = window_size
        self.input_size = input_size
        self.b_local, self.b_global = b_local, b_global
        self._engine = None
        self._key = None

    @property
    def kind(self) -> str:
        return "local" if self.window_size > 0 else "global"

    def engine_params(self) -> BlockParams:
        """This block's weights in the engine's layout (bf16 K-major GEMM weights, fp32 rest)."""
        a, m = self.attn, self.mlp
        for ln in (self.norm1, self.norm2):
            if abs(getattr(ln, "eps", 1e-6) - 1e-6) > 1e-12:
                raise ValueError("the engine's LayerNorm uses eps = 1e-6 (SAM's and the reference's)")
        f32 = lambda t: t.detach().float().contiguous()  # noqa: E731
        b16 = lambda t: t.detach().to(torch.bfloat16).contiguous()  # noqa: E731
        dim = a.qkv.in_features
        zeros = lambda n: torch.zeros(n, device=a.qkv.weight.device)  # noqa: E731
        return BlockParams(
            kind=self.kind, ln1_g=f32(self.norm1.weight), ln1_b=f32(self.norm1.bias),
            qkv_w=b16(a.qkv.weight), qkv_b=f32(a.qkv.bias) if a.qkv.bias is not None else zeros(3 * dim),
            proj_w=b16(a.proj.weight), proj_b=f32(a.proj.bias),
            bh=None if a.use_rel_pos else f32(a.bias_h), bw=None if a.use_rel_pos else f32(a.bias_w),
            ln2_g=f32(self.norm2.weight), ln2_b=f32(self.norm2.bias),
            w1=b16(m.lin1.weight), b1=f32(m.lin1.bias), w2=b16(m.lin2.weight), b2=f32(m.lin2.bias),
            rel_pos_h=f32(a.rel_pos_h) if a.use_rel_pos else None, rel_pos_w=f32(a.rel_pos_w) if a.use_rel_pos else None,
        )

    def engine_config(self, grid_h: int, grid_w: int) -> EncoderConfig:
        a = self.attn
        return EncoderConfig(grid=GridShape(grid_h, grid_w), d=a.qkv.in_features, heads=a.num_heads,
                             window=self.window_size if self.window_size > 0 else 14, layout=(self.kind,),
                             r=a.density, keep_fraction=self.mlp.keep_fraction, bypass_mode=self.mlp.bypass_mode,
                             b_local=self.b_local, b_global=self.b_global)

    @torch.no_grad()
    def forward(self, x: torch.Tensor) -> torch.Tensor:
        if x.dim() != 4 or not x.is_cuda:
            raise ValueError("SparseSAMBlock expects a CUDA tensor [B, H, W, C]")
        B, H, W, C = x.shape
        key = (H, W) + _version_key(self)
        if self._engine is None or self._key != key:
            self._engine = StripeSortEncoder(self.engine_config(H, W), [self.engine_params()], x.device)
            self._key = key
        return self._engine(x.float().contiguous())


class LayerNorm2d(nn.Module):
    """SAM's channels-first LayerNorm (neck), eps 1e-6."""

    def __init__(self, num_channels: int, eps: float = 1e-6):
        super().__init__()
        self.weight = nn.Parameter(torch.ones(num_channels))
        self.bias = nn.Parameter(torch.zeros(num_channels))
        self.eps = eps


class _PatchEmbed(nn.Module):
    def __init__(self, kernel_size=(16, 16), stride=(16, 16), in_chans: int = 3, embed_dim: int = 768):
        super().__init__()
        self.proj = nn.Conv2d(in_chans, embed_dim, kernel_size=kernel_size, stride=stride)


class SparseSAMImageEncoderViT(nn.Module):
    """SAM ``ImageEncoderViT`` with SparseSAM blocks: ``forward(x[B, 3, 1024, 1024])`` ->
    ``[B, out_chans, 64, 64]`` (channels-first, as SAM; ``forward_channels_last`` returns the
    engine's [B, 64, 64, out_chans] without the permuted view)."""

    def __init__(self, img_size: int = 1024, patch_size: int = 16, in_chans: int = 3, embed_dim: int = 768,
                 depth: int = 12, num_heads: int = 12, mlp_ratio: float = 4.0, out_chans: int = 256,
                 qkv_bias: bool = True, norm_layer: type[nn.Module] = nn.LayerNorm,
                 act_layer: type[nn.Module] = nn.GELU, use_abs_pos: bool = True, use_rel_pos: bool = False,
                 rel_pos_zero_init: bool = True, window_size: int = 0, global_attn_indexes: tuple[int, ...] = (), *,
                 density: float = 0.4, keep_fraction: float = 0.4, bypass_mode: str = "identity"):
        super().__init__()
        if patch_size != 16 or in_chans != 3 or out_chans != SAM_NECK:
            raise ValueError("the engine's frame is SAM's: 16x16 patches, 3 input channels, 256-channel neck")
        if not use_abs_pos:
            raise ValueError("the engine fuses SAM's absolute position embedding into the patch-embed GEMM")
        self.img_size = img_size
        g = img_size // patch_size
        self.patch_embed = _PatchEmbed((patch_size, patch_size), (patch_size, patch_size), in_chans, embed_dim)
        self.pos_embed = nn.Parameter(torch.zeros(1, g, g, embed_dim))
        self.blocks = nn.ModuleList(
            SparseSAMBlock(embed_dim, num_heads, mlp_ratio, qkv_bias, norm_layer, act_layer, use_rel_pos,
                           rel_pos_zero_init, window_size if i not in global_attn_indexes else 0, (g, g),
                           density=density, keep_fraction=keep_fraction, bypass_mode=bypass_mode)
            for i in range(depth))
        self.neck = nn.Sequential(nn.Conv2d(embed_dim, out_chans, kernel_size=1, bias=False), LayerNorm2d(out_chans),
                                  nn.Conv2d(out_chans, out_chans, kernel_size=3, padding=1, bias=False),
                                  LayerNorm2d(out_chans))
        windows = {b.window_size for b in self.blocks if b.window_size > 0}
        if len(windows) > 1:
            raise ValueError("one window size for all local blocks")
        self._window = windows.pop() if windows else 14
        self._engine = None
        self._key = None

    def engine_config(self) -> EncoderConfig:
        g = self.img_size // 16
        b0 = self.blocks[0]
        return EncoderConfig(grid=GridShape(g, g), d=b0.attn.qkv.in_features, heads=b0.attn.num_heads,
                             window=self._window, layout=tuple(b.kind for b in self.blocks),
                             r=tuple(b.attn.density for b in self.blocks),
                             keep_fraction=tuple(b.mlp.keep_fraction for b in self.blocks),
                             bypass_mode=b0.mlp.bypass_mode)

    def engine_frame(self) -> FrameParams:
        C = self.pos_embed.shape[-1]
        pe = self.patch_embed.proj
        n0, ln1, n2, ln2 = self.neck
        return FrameParams(
            pe_w=pe.weight.detach().reshape(C, -1).to(torch.bfloat16).contiguous(),
            pe_b=(pe.bias.detach().float() if pe.bias is not None else torch.zeros(C, device=pe.weight.device)),
            pos=self.pos_embed.detach().reshape(-1, C).float().contiguous(),
            neck1_w=n0.weight.detach().reshape(SAM_NECK, C).to(torch.bfloat16).contiguous(),
            neck_ln1_g=ln1.weight.detach().float(), neck_ln1_b=ln1.bias.detach().float(),
            neck2_w=n2.weight.detach().reshape(SAM_NECK, SAM_NECK * 9).to(torch.bfloat16).contiguous(),
            neck_ln2_g=ln2.weight.detach().float(), neck_ln2_b=ln2.bias.detach().float(),
        )

    def engine(self) -> SparseSAMImageEncoder:
        """The engine instance for the current parameters (rebuilt after any in-place update)."""
        key = _version_key(self)
        if self._engine is None or self._key != key:
            dev = self.pos_embed.device
            self._engine = SparseSAMImageEncoder(self.engine_config(), [b.engine_params() for b in self.blocks],
                                                 self.engine_frame(), dev)
            self._key = key
        return self._engine

    @torch.no_grad()
    def forward_channels_last(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if x.dim() != 4 or x.shape[1] != 3 or x.shape[2] != self.img_size or x.shape[3] != self.img_size:
            raise ValueError(f"expected [B, 3, {self.img_size}, {self.img_size}] images, got {tuple(x.shape)}")
        if not x.is_cuda:
            raise ValueError("SparseSAMImageEncoderViT runs on CUDA tensors (the B200 engine)")
        return self.engine()(x.float().contiguous(), out=out)

    @torch.no_grad()
    def forward(self, x: torch.Tensor) -> torch.Tensor:
        return self.forward_channels_last(x).permute(0, 3, 1, 2)


def from_sam_image_encoder(sam_encoder: nn.Module, *, density: float = 0.4, keep_fraction: float = 0.4,
                           bypass_mode: str = "identity") -> SparseSAMImageEncoderViT:
    """A SparseSAM encoder with the configuration and weights of a segment_anything
    ``ImageEncoderViT`` instance (duck-typed: its attributes and state_dict)."""
    b0 = sam_encoder.blocks[0]
    g = sam_encoder.pos_embed.shape[1]
    gidx = tuple(i for i, b in enumerate(sam_encoder.blocks) if b.window_size == 0)
    win = next((b.window_size for b in sam_encoder.blocks if b.window_size > 0), 0)
    dim = b0.attn.qkv.in_features
    enc = SparseSAMImageEncoderViT(
        img_size=g * 16, embed_dim=dim, depth=len(sam_encoder.blocks), num_heads=b0.attn.num_heads,
        mlp_ratio=b0.mlp.lin1.out_features / dim, qkv_bias=b0.attn.qkv.bias is not None,
        use_rel_pos=b0.attn.use_rel_pos, window_size=win, global_attn_indexes=gidx, density=density,
        keep_fraction=keep_fraction, bypass_mode=bypass_mode).to(sam_encoder.pos_embed.device)
    enc.load_state_dict(sam_encoder.state_dict(), strict=False)
    return enc
