"""Reference-compatible functional API over the B200 kernels.

Drop-in counterparts of the reference entry points on the hot path, with the
same names, argument meaning, return shapes and ``ValueError`` behaviour:

  sobel_magnitude   saliency.py:62-82        importance_order  saliency.py:99-118
  group_energy      saliency.py:85-96        stripe_sort       stripesort.py:38-62
  morton_order      grid.py:97-104           build_active_set  attention.py:88-104
  ashape_attention  attention.py:167-221     dense_attention   attention.py:138-164
  mlp_forward       mlp.py:78-85             route_mlp         mlp.py:88-114
  encoder_forward   encoder.py:310-385

Inputs may be numpy arrays (returned as numpy, like the reference) or CUDA
tensors (returned as CUDA tensors).  All arithmetic runs in the sm_100a
library; the host code here only validates, packs and unpacks.  The kernels
compute in bf16 with fp32 accumulation, so float outputs match the fp32
reference within the tolerances stated in DESIGN.md, while orderings,
permutations, active sets and keep-sets are bit-exact.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import kernels as K
from .config import AShapeConfig, EncoderConfig, GridShape, OrderingConfig, RouterConfig, StripeConfig
from .encoder import StripeSortEncoder, morton_order_np
from .weights import BlockParams, params_from_reference

# ---------------------------------------------------------------- plumbing


def _dev() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the SparseSAM B200 kernels need a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(a, dtype=torch.float32) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=_dev(), dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a)).to(device=_dev(), dtype=dtype).contiguous()


def _like(t: torch.Tensor, ref):
    return t if isinstance(ref, torch.Tensor) else t.cpu().numpy()


def _as_index(p) -> np.ndarray:
    f = p.forward if hasattr(p, "forward") else p
    if isinstance(f, torch.Tensor):
        f = f.cpu().numpy()
    return np.asarray(f, dtype=np.int64)


@dataclass(frozen=True)
class Permutation:
    """Validated bijection over [0, N): forward[i] = token at rank i (grid.py:32-69)."""

    forward: np.ndarray
    inverse: np.ndarray = field(default=None)  # type: ignore[assignment]

    def __post_init__(self):
        f = np.ascontiguousarray(np.asarray(self.forward, dtype=np.int64))
        if f.ndim != 1:
            raise ValueError("forward must be 1-d")
        n = f.size
        if n and (f.min() < 0 or f.max() >= n):
            raise ValueError("forward entries must lie in [0, N)")
        seen = np.zeros(n, bool)
        seen[f] = True
        if not seen.all():
            raise ValueError("forward is not a bijection on [0, N)")
        inv = np.empty(n, np.int64)
        inv[f] = np.arange(n)
        if self.inverse is not None and not np.array_equal(np.asarray(self.inverse, np.int64), inv):
            raise ValueError("inverse does not match forward")
        object.__setattr__(self, "forward", f)
        object.__setattr__(self, "inverse", inv)

    def __len__(self) -> int:
        return int(self.forward.size)

    @staticmethod
    def identity(n: int) -> "Permutation":
        return Permutation(np.arange(n, dtype=np.int64))


@dataclass(frozen=True)
class SaliencyMap:
    shape: GridShape
    values: np.ndarray

    def flat(self):
        return self.values.reshape(-1)


def morton_order(shape: GridShape) -> Permutation:
    return Permutation(morton_order_np(shape.h, shape.w))


# ---------------------------------------------------------------- ordering
def sobel_magnitude(x) -> SaliencyMap:
    """Sobel gradient magnitude of [H, W, D] features, bit-exact with the reference."""
    if np.ndim(x) != 3:
        raise ValueError(f"expected [H, W, D], got shape {tuple(np.shape(x))}")
    xt = _to_dev(x)
    h, w, _ = xt.shape
    sal, _ = K.sobel_saliency(xt[None], window=max(h, w), glob=True, win=False)
    return SaliencyMap(GridShape(h, w), _like(sal[0], x))


def group_energy(m: SaliencyMap, morton: Permutation, group_size: int):
    n = m.shape.n()
    if len(morton) != n:
        raise ValueError("permutation size does not match grid")
    if group_size < 1 or n % group_size:
        raise ValueError(f"group_size {group_size} must divide N={n}")
    vals = _to_dev(m.values).reshape(1, -1)
    _, e = K.rank_order(vals, _to_dev(morton.forward, torch.int32), group_size=group_size, g=1,
                        variant="no_interleave", want_energy=True)
    return _like(e[0], m.values)


def importance_order(m: SaliencyMap, cfg: OrderingConfig = OrderingConfig()) -> Permutation:
    n = m.shape.n()
    if cfg.granularity == "zgroup" and n % cfg.group_size:
        raise ValueError(f"group_size {cfg.group_size} must divide N={n}")
    mo = _to_dev(morton_order_np(m.shape.h, m.shape.w), torch.int32)
    sig, _ = K.rank_order(_to_dev(m.values).reshape(1, -1), mo, granularity=cfg.granularity,
                          group_size=cfg.group_size, g=1, variant="no_interleave")
    return Permutation(sig[0].cpu().numpy())


def importance_order_from_energy(energy, morton: Permutation, group_size: int = 4) -> Permutation:
    """Rank pre-computed z-group energies (the 'fed the reference's scores' path)."""
    sig, _ = K.rank_order(_to_dev(energy).reshape(1, -1), _to_dev(morton.forward, torch.int32),
                          group_size=group_size, g=1, variant="no_interleave", scores_are_energy=True)
    return Permutation(sig[0].cpu().numpy())


def stripe_sort(pi: Permutation, cfg: StripeConfig = StripeConfig(), morton: Permutation | None = None) -> Permutation:
    """sigma = flatten(reshape(pi, (N/G, G))^T); ``no_sort`` interleaves ``morton`` instead."""
    n = len(pi)
    if n % cfg.g:
        raise ValueError(f"group count {cfg.g} must divide N={n}")
    if cfg.variant == "no_interleave":
        return Permutation(pi.forward.copy())
    if cfg.variant == "no_sort":
        if morton is None:
            raise ValueError("variant 'no_sort' needs the morton base order")
        if len(morton) != n:
            raise ValueError("morton permutation size mismatch")
        base = morton.forward
    else:
        base = pi.forward
    # the stripe interleave is the last stage of the device rank kernel; feeding it the
    # base order as "energies" of singleton groups in rank order reproduces it exactly
    keys = -np.arange(n, dtype=np.float32)  # strictly decreasing -> rank == position
    sig, _ = K.rank_order(_to_dev(keys).reshape(1, -1), _to_dev(base, torch.int32), group_size=1, g=cfg.g,
                          variant="full", scores_are_energy=True)
    return Permutation(sig[0].cpu().numpy())


# ---------------------------------------------------------------- attention
@dataclass(frozen=True)
class BiasTables:
    bh: np.ndarray
    bw: np.ndarray

    def __post_init__(self):
        bh = np.ascontiguousarray(np.asarray(self.bh, dtype=np.float32))
        bw = np.ascontiguousarray(np.asarray(self.bw, dtype=np.float32))
        if bh.ndim != 2 or bh.shape != bw.shape:
            raise ValueError(f"bias tables must share shape [S_q, w], got {bh.shape} / {bw.shape}")
        object.__setattr__(self, "bh", bh)
        object.__setattr__(self, "bw", bw)

    @property
    def w(self) -> int:
        return int(self.bh.shape[1])


@dataclass(frozen=True)
class ActiveSet:
    t_col: int
    tiles: tuple

    def size(self) -> int:
        return sum(len(j) for j in self.tiles)


def build_active_set(t_row: int, t_col: int, r: float) -> ActiveSet:
    """J_i = {0..floor(r*Tc)-1} ∪ {min(i, Tc-1)}: the static schedule the kernel's chunk plan encodes."""
    if t_row < 1 or t_col < 1:
        raise ValueError("tile counts must be >= 1")
    p = math.floor(r * t_col)
    return ActiveSet(t_col, tuple(tuple(sorted(set(range(p)) | {min(i, t_col - 1)})) for i in range(t_row)))


def achieved_density(t_row: int, t_col: int, r: float) -> float:
    return build_active_set(t_row, t_col, r).size() / (t_row * t_col)


def _check_attn(q, k, v, bias, sq_perm, sk_perm):
    for a, n in ((q, "q"), (k, "k"), (v, "v")):
        if np.ndim(a) != 2:
            raise ValueError("q, k, v must be 2-d")
    sq, d = q.shape
    sk = k.shape[0]
    if k.shape[1] != d:
        raise ValueError(f"k width {k.shape[1]} != q width {d}")
    if tuple(v.shape) != (sk, d):
        raise ValueError(f"v shape {tuple(v.shape)} != [{sk}, {d}]")
    if len(sq_perm) != sq or len(sk_perm) != sk:
        raise ValueError("permutation sizes must match S_q / S_k")
    bh = bias.bh
    if bh.shape[0] != sq:
        raise ValueError(f"bias tables have {bh.shape[0]} rows, expected {sq}")
    w = bh.shape[1]
    if w * w != sk:
        raise ValueError(f"bias grid {w}^2 != S_k={sk}")
    return sq, sk, d, w


def ashape_attention(q, k, v, bias: BiasTables, sq_perm, sk_perm, cfg: AShapeConfig):
    """Blocked A-shape attention (attention.py:167-221) on the tcgen05 kernel.

    Head dims up to 80 run natively (zero-padded to 64 / 80 with tau kept at
    1/sqrt(d)); wider heads raise ValueError.
    """
    sq, sk, d, w = _check_attn(q, k, v, bias, sq_perm, sk_perm)
    if d > 80:
        raise ValueError(f"head dim {d} > 80 is not supported by the B200 kernel")
    dpad = 64 if d <= 64 else 80
    tau = (1.0 / math.sqrt(d)) if cfg.tau is None else float(cfg.tau)
    # pack q | k | v into one padded bf16 buffer per operand
    qb = torch.zeros((sq, dpad), device=_dev(), dtype=torch.bfloat16)
    kb = torch.zeros((sk, dpad), device=_dev(), dtype=torch.bfloat16)
    vb = torch.zeros((sk, dpad), device=_dev(), dtype=torch.bfloat16)
    qb[:, :d] = _to_dev(q)
    kb[:, :d] = _to_dev(k)
    vb[:, :d] = _to_dev(v)
    tc = -(-sk // cfg.b_col)
    out = K.stripe_attn(qb, kb, vb, units=1, heads=1, sq=sq, sk=sk, dh=dpad, bh=_to_dev(bias.bh)[None],
                        bw=_to_dev(bias.bw)[None], q_sp=_to_dev(_as_index(sq_perm), torch.int32),
                        k_sp=_to_dev(_as_index(sk_perm), torch.int32), b_row=cfg.b_row, b_col=cfg.b_col,
                        prefix=cfg.prefix_tiles(tc), tau=tau)
    return _like(out[:, :d].float(), q)


def dense_attention(q, k, v, bias: BiasTables, sq_perm, sk_perm, tau=None):
    """Full-matrix attention (the dense twin, attention.py:138-164): one tile spanning all columns."""
    sq, sk, _, _ = _check_attn(q, k, v, bias, sq_perm, sk_perm)
    return ashape_attention(q, k, v, bias, sq_perm, sk_perm, AShapeConfig(b_row=sq, b_col=sk, r=1.0, tau=tau))


# ---------------------------------------------------------------- MLP
@dataclass(frozen=True)
class MlpWeights:
    w1: np.ndarray  # [d, h]
    b1: np.ndarray
    w2: np.ndarray  # [h, d]
    b2: np.ndarray
    ln_gamma: np.ndarray
    ln_beta: np.ndarray

    def __post_init__(self):
        for n in ("w1", "b1", "w2", "b2", "ln_gamma", "ln_beta"):
            object.__setattr__(self, n, np.ascontiguousarray(np.asarray(getattr(self, n), dtype=np.float32)))
        if self.w1.ndim != 2 or self.w2.ndim != 2:
            raise ValueError("w1 and w2 must be 2-d")
        d, h = self.w1.shape
        if d < 1 or h < 1:
            raise ValueError("weight extents must be >= 1")
        if self.w2.shape != (h, d):
            raise ValueError(f"w2 shape {self.w2.shape} != [{h}, {d}]")
        for n, e in (("b1", h), ("b2", d), ("ln_gamma", d), ("ln_beta", d)):
            if getattr(self, n).shape != (e,):
                raise ValueError(f"{n} must have shape [{e}]")

    @property
    def d(self) -> int:
        return int(self.w1.shape[0])

    @property
    def h(self) -> int:
        return int(self.w1.shape[1])


def _pad64(n: int) -> int:
    return -(-n // 64) * 64


def _mlp_device(w: MlpWeights):
    """Zero-padded device weights: widths rounded up to the GEMM's 64-column granule."""
    d, h = w.d, w.h
    dp, hp = _pad64(d), _pad64(h)
    dev = _dev()
    w1 = torch.zeros((hp, dp), device=dev, dtype=torch.bfloat16)
    w1[:h, :d] = _to_dev(w.w1).T
    w2 = torch.zeros((dp, hp), device=dev, dtype=torch.bfloat16)
    w2[:d, :h] = _to_dev(w.w2).T
    b1 = torch.zeros(hp, device=dev)
    b1[:h] = _to_dev(w.b1)
    b2 = torch.zeros(dp, device=dev)
    b2[:d] = _to_dev(w.b2)
    return w1, b1, w2, b2, dp


def _rows_mlp(x, w: MlpWeights, keep: np.ndarray, bypass: np.ndarray | None):
    n, d = x.shape
    w1, b1, w2, b2, dp = _mlp_device(w)
    xt = torch.zeros((n, dp), device=_dev(), dtype=torch.float32)
    xt[:, :d] = _to_dev(x)
    g, b = _to_dev(w.ln_gamma), _to_dev(w.ln_beta)
    keep_t = _to_dev(keep, torch.int32)
    if dp == d:
        K.rc_mlp(xt, keep_t, ln_g=g, ln_b=b, w1=w1, b1=b1, w2=w2, b2=b2,
                 bypass_rows=None if bypass is None else _to_dev(bypass, torch.int32))
    else:
        # narrow widths (tests / toy configs): LN on the exact width, then the padded GEMM pair
        xn = K.layernorm_rows(_to_dev(x), g, b, rows=keep_t)
        hpad = torch.zeros((keep.size, dp), device=_dev(), dtype=torch.bfloat16)
        hpad[:, :d] = xn
        hid = K.gemm(hpad, w1, b1, epi=K.EPI_BF16_GELU)
        K.gemm(hid, w2, b2, epi=K.EPI_F32_RESID, out=xt, res=xt, row_map=keep_t)
        if bypass is not None and bypass.size:
            bt = _to_dev(bypass, torch.int32)
            ln = K.layernorm_rows(_to_dev(x), g, b, rows=bt, out_f32=True)
            xt[bt.long(), :d] = ln
    return xt[:, :d]


def mlp_forward(x, w: MlpWeights):
    """(x + delta, delta) with delta = MLP(LN(x)) (mlp.py:78-85)."""
    if np.ndim(x) != 2 or x.shape[1] != w.d:
        raise ValueError(f"x must be [N, {w.d}], got {tuple(np.shape(x))}")
    n = x.shape[0]
    y = _rows_mlp(x, w, np.arange(n), None)
    xt = _to_dev(x)
    return _like(y, x), _like(y - xt, x)


def route_mlp(x, w: MlpWeights, sigma, cfg: RouterConfig):
    """MLP on the K leading-rank tokens of sigma only (mlp.py:88-114)."""
    if np.ndim(x) != 2 or x.shape[1] != w.d:
        raise ValueError(f"x must be [N, {w.d}], got {tuple(np.shape(x))}")
    n = x.shape[0]
    if len(sigma) != n:
        raise ValueError(f"permutation sized {len(sigma)} != N={n}")
    order = _as_index(sigma)
    kc = cfg.keep_count(n)
    keep, rest = order[:kc], order[kc:]
    y = _rows_mlp(x, w, keep, rest if cfg.bypass_mode == "layernorm" else None)
    return _like(y, x)


# ---------------------------------------------------------------- encoder
@dataclass(frozen=True)
class BlockCost:
    kind: str
    tile_pairs: int
    tile_pairs_total: int
    mlp_rows: int
    mlp_rows_total: int
    ms: float

    @property
    def attn_density(self) -> float:
        return self.tile_pairs / self.tile_pairs_total

    @property
    def mlp_fraction(self) -> float:
        return self.mlp_rows / self.mlp_rows_total


COST_COLUMNS = "block,kind,tile_pairs,tile_pairs_total,attn_density,mlp_rows,mlp_rows_total,mlp_fraction,ms"


@dataclass(frozen=True)
class CostReport:
    blocks: tuple

    def total_ms(self) -> float:
        return sum(b.ms for b in self.blocks)

    def attn_density(self) -> float:
        return sum(b.tile_pairs for b in self.blocks) / sum(b.tile_pairs_total for b in self.blocks)

    def csv(self, with_ms: bool = True) -> str:
        lines = [COST_COLUMNS]
        for i, b in enumerate(self.blocks):
            ms = f"{b.ms:.3f}" if with_ms else ""
            lines.append(f"{i},{b.kind},{b.tile_pairs},{b.tile_pairs_total},{b.attn_density!r},"
                         f"{b.mlp_rows},{b.mlp_rows_total},{b.mlp_fraction!r},{ms}")
        return "\r\n".join(lines) + "\r\n"


def cost_report(cfg: EncoderConfig, mode: str = "sparse", ms=None) -> CostReport:
    """Work accounting per block, identical to encoder.py:372-384."""
    out = []
    for bi, kind in enumerate(cfg.layout):
        r = 1.0 if mode == "dense" else cfg.r[bi]
        kf = 1.0 if mode == "dense" else cfg.keep_fraction[bi]
        if kind == "global":
            units, s = 1, cfg.grid.n()
        else:
            units, s = cfg.nwin(), cfg.window**2
        tile = cfg.tile(kind)
        t = -(-s // tile)
        a = build_active_set(t, t, r)
        out.append(BlockCost(kind, units * cfg.heads * a.size(), units * cfg.heads * t * t,
                             units * RouterConfig(kf, cfg.bypass_mode).keep_count(s), units * s,
                             0.0 if ms is None else float(ms[bi])))
    return CostReport(tuple(out))


def encoder_forward(x, weights, cfg: EncoderConfig, mode: str = "sparse"):
    """Run every block over [H, W, D] (or a batch [B, H, W, D]); returns (output, CostReport).

    ``weights`` are reference-layout block weights (``BlockWeights`` / oracle
    blocks) or already-converted ``BlockParams``.  ``CostReport.ms`` holds each
    block's device time (CUDA events around its launches).

    Shape envelope of the B200 block engine: d a multiple of 64 and head dim
    d / heads <= 80; heads narrower than 64 (e.g. the reference's default d = 64
    with 4 heads, dh = 16) run zero-padded to 64 columns with tau = 1/sqrt(dh)
    (``encoder._pad_heads``), other widths raise ValueError.  The per-op entry
    points (``ashape_attention``, ``route_mlp``) zero-pad heads up to 80 and take
    any width.
    """
    if mode not in ("dense", "sparse"):
        raise ValueError(f"mode must be 'dense' or 'sparse', got {mode!r}")
    single = np.ndim(x) == 3
    shape = (cfg.grid.h, cfg.grid.w, cfg.d)
    if tuple(np.shape(x))[-3:] != shape or np.ndim(x) not in (3, 4):
        raise ValueError(f"input shape {tuple(np.shape(x))} != {shape}")
    if len(weights) != len(cfg.layout):
        raise ValueError(f"{len(weights)} weight sets for {len(cfg.layout)} blocks")
    dev = _dev()
    params = weights if isinstance(weights[0], BlockParams) else params_from_reference(weights, cfg, dev)
    enc = StripeSortEncoder(cfg, params, dev)
    xt = _to_dev(x)
    if single:
        xt = xt[None]
    # per-block device time from CUDA events around each block's launches (the reference's
    # per-block wall clock, encoder.py:342,372; the orderings are outside every block)
    enc.block_events = []
    y = enc(xt, mode)
    torch.cuda.synchronize()
    per = [s.elapsed_time(e) for s, e in enc.block_events]
    enc.block_events = None
    y = y[0] if single else y
    return _like(y, x), cost_report(cfg, mode, per)


# ---------------------------------------------------------------- benchmarks (encoder.py:388-444, cli.py:96-130)
@dataclass(frozen=True)
class BenchRow:
    density: float
    achieved_density: float
    median_ms: float
    speedup: float


BENCH_COLUMNS = "density,achieved_density,median_ms,speedup"


def _median(v):
    s = sorted(v)
    n = len(s)
    return s[n // 2] if n % 2 else 0.5 * (s[n // 2 - 1] + s[n // 2])


def _time_ms(fn, repeats: int) -> list:
    """Device time of fn() per repeat (CUDA events on the current stream, one warm-up call)."""
    fn()
    out = []
    for _ in range(repeats):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    return out


def bench(cfg: EncoderConfig, densities, repeats: int = 3, x=None, weights=None) -> list:
    """Median sparse-mode encoder time per density against the dense twin (encoder.py:399-436).

    The reference times ``encoder_forward`` on the host; this times the same block engine on the
    device (CUDA events, one warm-up call per configuration): the sparse encoder at each
    density and the SAME engine in ``mode="dense"`` (r = keep = 1, encoder.py:416-419) as the
    dense twin, so ``speedup`` is dense-twin median over sparse median exactly as the reference
    defines it.  ``x`` defaults to a seeded normal image [H, W, D] (torch generator seeded with
    cfg.seed + 1, not the reference's splitmix stream); ``weights`` (reference-layout blocks or
    ``BlockParams``) default to ``weights.random_params(cfg, seed=cfg.seed)`` — the values do not
    change the timing.  A batch [B, H, W, D] is accepted too.
    """
    import dataclasses

    from .weights import random_params

    if repeats < 1:
        raise ValueError("repeats must be >= 1")
    dev = _dev()
    if x is None:
        g = torch.Generator(device=dev).manual_seed(cfg.seed + 1)
        xt = torch.randn((cfg.grid.h, cfg.grid.w, cfg.d), generator=g, device=dev)
    else:
        xt = _to_dev(x)
    if xt.dim() == 3:
        xt = xt[None]
    if tuple(xt.shape[-3:]) != (cfg.grid.h, cfg.grid.w, cfg.d):
        raise ValueError(f"input shape {tuple(xt.shape)} != {(cfg.grid.h, cfg.grid.w, cfg.d)}")
    if weights is None:
        params = random_params(cfg, dev, seed=cfg.seed)
    elif isinstance(weights[0], BlockParams):
        params = list(weights)
    else:
        params = params_from_reference(weights, cfg, dev)
    dense_enc = StripeSortEncoder(cfg, params, dev)
    dense_ms = _median(_time_ms(lambda: dense_enc(xt, "dense"), repeats))
    rows = []
    for density in densities:
        cfg_r = dataclasses.replace(cfg, r=float(density))
        enc = StripeSortEncoder(cfg_r, params, dev)
        med = _median(_time_ms(lambda: enc(xt, "sparse"), repeats))
        rows.append(BenchRow(density=float(density), achieved_density=cost_report(cfg_r).attn_density(),
                             median_ms=med, speedup=dense_ms / med))
    return rows


def bench_csv(rows) -> str:
    """BENCH_COLUMNS table, CRLF line ends, the reference's number formats (encoder.py:439-444)."""
    lines = [BENCH_COLUMNS]
    for r in rows:
        lines.append(f"{r.density!r},{r.achieved_density!r},{r.median_ms:.3f},{r.speedup:.4f}")
    return "\r\n".join(lines) + "\r\n"


def attn_bench(n: int = 4096, d: int = 64, densities=(0.25, 0.5, 1.0), repeats: int = 20, tile: int = 128,
               seed: int = 0) -> str:
    """``zstripe attn-bench`` (cli.py:96-130) on the tcgen05 attention kernel: one head of n tokens
    (a perfect square: the w x w bias grid), identity permutations, tile x tile blocks; median
    device time per distinct density, speedup against r = 1.0; returns the BENCH_COLUMNS CSV
    (CRLF).  Inputs are seeded torch normals (bias tables std 0.5, as the reference), staged on the
    device before timing; head widths d <= 80 run zero-padded to 64 / 80 with tau = 1/sqrt(d)."""
    w = math.isqrt(n)
    if w * w != n:
        raise ValueError(f"--n must be a perfect square for the 2D bias grid, got {n}")
    densities = [float(r) for r in densities]
    if not densities:
        raise ValueError("--densities must name at least one density")
    if d > 80 or d < 1:
        raise ValueError(f"head dim {d} outside the B200 kernel's 1..80")
    dev = _dev()
    g = torch.Generator(device=dev).manual_seed(seed)
    dpad = 64 if d <= 64 else 80
    qkv = [torch.zeros((n, dpad), device=dev, dtype=torch.bfloat16) for _ in range(3)]
    for t in qkv:
        t[:, :d] = torch.randn((n, d), generator=g, device=dev).bfloat16()
    bh = torch.randn((1, n, w), generator=g, device=dev) * 0.5
    bw = torch.randn((1, n, w), generator=g, device=dev) * 0.5
    ident = torch.arange(n, device=dev, dtype=torch.int32)
    out = torch.empty((n, dpad), device=dev, dtype=torch.bfloat16)
    ws = torch.empty(max(K.attn_ws_bytes(1, 1, n, n, dpad), 256), device=dev, dtype=torch.uint8)
    t_tiles = -(-n // tile)
    tau = 1.0 / math.sqrt(d)

    def run(r: float) -> float:
        prefix = AShapeConfig(b_row=tile, b_col=tile, r=r).prefix_tiles(t_tiles)
        return _median(_time_ms(lambda: K.stripe_attn(qkv[0], qkv[1], qkv[2], units=1, heads=1, sq=n, sk=n, dh=dpad,
                                                      bh=bh, bw=bw, q_sp=ident, k_sp=ident, b_row=tile, b_col=tile,
                                                      prefix=prefix, tau=tau, out=out, ws=ws), repeats))

    medians = {r: run(r) for r in dict.fromkeys(densities)}
    baseline = medians.get(1.0)
    if baseline is None:
        baseline = run(1.0)
    lines = [BENCH_COLUMNS]
    for r in densities:
        lines.append(f"{r!r},{achieved_density(t_tiles, t_tiles, r)!r},{medians[r]:.3f},{baseline / medians[r]:.4f}")
    return "\r\n".join(lines) + "\r\n"
