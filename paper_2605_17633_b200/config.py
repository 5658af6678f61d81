"""Configuration types mirroring the reference's frozen dataclasses.

Same names, fields, defaults and ``ValueError`` behaviour as the reference
(grid.py:19-29, stripesort.py:26-35, saliency.py:44-59, attention.py:58-74,
mlp.py:60-75, encoder.py:38-109), so code written against ``zstripe`` reads
the same against this package.  ``sam_config`` adds the SAM ViT-B/L/H
layouts the benchmark is quoted on.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

BLOCK_KINDS = ("local", "global")
STRIPE_VARIANTS = ("full", "no_interleave", "no_sort")


@dataclass(frozen=True)
class GridShape:
    h: int
    w: int

    def __post_init__(self):
        if self.h < 1 or self.w < 1:
            raise ValueError(f"grid extents must be >= 1, got {self.h}x{self.w}")

    def n(self) -> int:
        return self.h * self.w


@dataclass(frozen=True)
class StripeConfig:
    g: int = 4
    variant: str = "full"

    def __post_init__(self):
        if self.g < 1:
            raise ValueError("group count must be >= 1")
        if self.variant not in STRIPE_VARIANTS:
            raise ValueError(f"variant must be one of {STRIPE_VARIANTS}, got {self.variant!r}")


@dataclass(frozen=True)
class OrderingConfig:
    granularity: str = "zgroup"
    group_size: int = 4

    def __post_init__(self):
        if self.granularity not in ("token", "zgroup"):
            raise ValueError(f"unknown granularity {self.granularity!r}")
        if self.group_size < 1:
            raise ValueError("group_size must be >= 1")


@dataclass(frozen=True)
class AShapeConfig:
    """Static sparsity schedule: tile sizes, density ratio, softmax scale (None = 1/sqrt(d))."""

    b_row: int = 32
    b_col: int = 32
    r: float = 1.0
    tau: float | None = None

    def __post_init__(self):
        if self.b_row < 1 or self.b_col < 1:
            raise ValueError("tile sizes must be >= 1")
        if not 0.0 <= self.r <= 1.0:
            raise ValueError(f"density ratio must be in [0, 1], got {self.r}")

    def prefix_tiles(self, t_col: int) -> int:
        """floor(r * T_col) evaluated in double, as attention.py:98."""
        return math.floor(self.r * t_col)


@dataclass(frozen=True)
class RouterConfig:
    keep_fraction: float = 1.0
    bypass_mode: str = "identity"

    def __post_init__(self):
        if not 0.0 < self.keep_fraction <= 1.0:
            raise ValueError(f"keep_fraction must be in (0, 1], got {self.keep_fraction}")
        if self.bypass_mode not in ("identity", "layernorm"):
            raise ValueError(f"unknown bypass_mode {self.bypass_mode!r}")

    def keep_count(self, n: int) -> int:
        """K = round(keep_fraction * N) clamped to [1, N]; Python's half-to-even round (mlp.py:73-75)."""
        return min(max(round(self.keep_fraction * n), 1), n)


def _per_block(value, n: int, name: str) -> tuple[float, ...]:
    if isinstance(value, (int, float)):
        return (float(value),) * n
    vals = tuple(float(v) for v in value)
    if len(vals) != n:
        raise ValueError(f"{name} needs 1 or {n} values, got {len(vals)}")
    return vals


@dataclass(frozen=True)
class EncoderConfig:
    grid: GridShape
    d: int = 64
    heads: int = 4
    window: int = 14
    layout: tuple = ("local", "local", "global")
    r: float | tuple = 0.25
    keep_fraction: float | tuple = 0.5
    stripe: StripeConfig = field(default_factory=StripeConfig)
    ordering: OrderingConfig = field(default_factory=OrderingConfig)
    bypass_mode: str = "identity"
    b_local: int = 32
    b_global: int = 128
    seed: int = 0

    def __post_init__(self):
        if self.d < 1 or self.heads < 1 or self.d % self.heads:
            raise ValueError(f"width {self.d} must be a positive multiple of heads={self.heads}")
        if self.window < 1:
            raise ValueError("window must be >= 1")
        if self.b_local < 1 or self.b_global < 1:
            raise ValueError("tile sizes must be >= 1")
        layout = tuple(self.layout)
        if not layout:
            raise ValueError("layout must name at least one block")
        for k in layout:
            if k not in BLOCK_KINDS:
                raise ValueError(f"unknown block kind {k!r}, expected one of {BLOCK_KINDS}")
        object.__setattr__(self, "layout", layout)
        object.__setattr__(self, "r", _per_block(self.r, len(layout), "r"))
        object.__setattr__(self, "keep_fraction", _per_block(self.keep_fraction, len(layout), "keep_fraction"))
        for v in self.r:
            if not 0.0 <= v <= 1.0:
                raise ValueError(f"density ratio must be in [0, 1], got {v}")
        for v in self.keep_fraction:
            if not 0.0 < v <= 1.0:
                raise ValueError(f"keep_fraction must be in (0, 1], got {v}")
        if self.bypass_mode not in ("identity", "layernorm"):
            raise ValueError(f"unknown bypass_mode {self.bypass_mode!r}")
        if "global" in layout:
            if self.grid.h != self.grid.w:
                raise ValueError("global blocks need a square token grid")
            if self.grid.n() % self.stripe.g:
                raise ValueError(f"stripe count {self.stripe.g} must divide N={self.grid.n()} for global blocks")
        if "local" in layout and (self.window * self.window) % self.stripe.g:
            raise ValueError(f"stripe count {self.stripe.g} must divide window^2={self.window * self.window}")

    @property
    def head_dim(self) -> int:
        return self.d // self.heads

    def tile(self, kind: str) -> int:
        return self.b_local if kind == "local" else self.b_global

    def nwin(self) -> int:
        return math.ceil(self.grid.h / self.window) * math.ceil(self.grid.w / self.window)


# SAM image-encoder geometry (public segment_anything ImageEncoderViT)
SAM_MODELS = {
    "vit_b": dict(d=768, depth=12, heads=12, global_idx=(2, 5, 8, 11)),
    "vit_l": dict(d=1024, depth=24, heads=16, global_idx=(5, 11, 17, 23)),
    "vit_h": dict(d=1280, depth=32, heads=16, global_idx=(7, 15, 23, 31)),
}
SAM_IMG = 1024
SAM_PATCH = 16
SAM_NECK = 256


def sam_config(model: str, density: float = 0.4, seed: int = 0, **kw) -> EncoderConfig:
    """EncoderConfig of a SAM ViT encoder (64x64 tokens, window 14) at attention r = keep = density."""
    m = SAM_MODELS[model]
    layout = tuple("global" if i in m["global_idx"] else "local" for i in range(m["depth"]))
    return EncoderConfig(grid=GridShape(64, 64), d=m["d"], heads=m["heads"], window=14, layout=layout, r=density,
                         keep_fraction=density, seed=seed, **kw)
