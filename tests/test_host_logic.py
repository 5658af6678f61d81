"""Host-side logic (CPU): config validation mirrors the reference, SAM layouts,
the attention kernel's chunk plan covers exactly the static active set, the
host Morton tables, image sharding and the CostReport accounting."""

import math

import numpy as np
import pytest

from conftest import golden
from oracle import zs_oracle as O
from paper_2605_17633_b200 import config as C
from paper_2605_17633_b200.encoder import morton_order_np
from paper_2605_17633_b200.parallel import shard_bounds, shard_counts


def test_config_validation_mirrors_reference():
    # encoder.py:60-100 error cases
    g = C.GridShape(8, 8)
    with pytest.raises(ValueError):
        C.EncoderConfig(grid=g, d=10, heads=4)
    with pytest.raises(ValueError):
        C.EncoderConfig(grid=g, layout=("local", "bogus"))
    with pytest.raises(ValueError):
        C.EncoderConfig(grid=g, r=(0.1, 0.2))
    with pytest.raises(ValueError):
        C.EncoderConfig(grid=C.GridShape(8, 6), layout=("global",))
    with pytest.raises(ValueError):
        C.EncoderConfig(grid=g, window=5, layout=("local",))
    with pytest.raises(ValueError):
        C.EncoderConfig(grid=g, keep_fraction=0.0)
    with pytest.raises(ValueError):
        C.GridShape(0, 3)
    with pytest.raises(ValueError):
        C.StripeConfig(variant="nope")
    with pytest.raises(ValueError):
        C.OrderingConfig(granularity="pixel")
    cfg = C.EncoderConfig(grid=g, d=64, heads=4, window=4, layout=("local", "global"), r=(0.2, 0.9))
    assert cfg.r == (0.2, 0.9) and cfg.keep_fraction == (0.5, 0.5) and cfg.head_dim == 16


def test_keep_count_half_to_even():
    rc = C.RouterConfig
    assert [rc(0.5).keep_count(7), rc(0.5).keep_count(9), rc(0.01).keep_count(10)] == [4, 4, 1]
    g = golden("mlp_cases")
    for fm, n, k in g["keep_counts"].tolist():
        assert C.RouterConfig(fm / 1000).keep_count(n) == k


@pytest.mark.parametrize("model,glob", [("vit_b", (2, 5, 8, 11)), ("vit_l", (5, 11, 17, 23)),
                                        ("vit_h", (7, 15, 23, 31))])
def test_sam_layouts(model, glob):
    cfg = C.sam_config(model, 0.4)
    assert tuple(i for i, k in enumerate(cfg.layout) if k == "global") == glob
    assert cfg.grid.n() == 4096 and cfg.window == 14 and cfg.nwin() == 25
    assert cfg.head_dim == (80 if model == "vit_h" else 64)


def test_host_morton_tables_match_oracle():
    for h, w in [(64, 64), (14, 14), (20, 20), (6, 10)]:
        assert np.array_equal(morton_order_np(h, w), O.morton_order(h, w))


def _needed_chunks(sq, sk, br, bc, p, mb, BKC=128):
    """Python restatement of attn::ChunkPlan::needed (csrc/zs_attn.cu)."""
    tc = -(-sk // bc)
    row0 = mb * 128
    qlo, qhi = row0 // br, min(row0 + 127, sq - 1) // br
    dlo, dhi = min(qlo, tc - 1), min(qhi, tc - 1)
    out = []
    for cj in range(-(-sk // BKC)):
        klo = (cj * BKC) // bc
        khi = min((cj * BKC + BKC - 1) // bc, tc - 1)
        if klo < p or not (dhi < klo or dlo > khi):
            out.append(cj)
    return out


@pytest.mark.parametrize("sq,sk,br,bc", [(196, 196, 32, 32), (4096, 4096, 128, 128), (100, 81, 32, 32),
                                         (130, 144, 128, 128), (70, 81, 16, 24), (300, 49, 7, 5)])
@pytest.mark.parametrize("r", [0.0, 0.2, 0.4, 0.77, 1.0])
def test_chunk_plan_covers_active_set(sq, sk, br, bc, r):
    """Every active (row, col) of J_i lies in a visited chunk, and every visited chunk holds one."""
    tr, tc = -(-sq // br), -(-sk // bc)
    J = O.active_set(tr, tc, r)
    p = math.floor(r * tc)
    for mb in range(-(-sq // 128)):
        need = set(_needed_chunks(sq, sk, br, bc, p, mb))
        rows = range(mb * 128, min(mb * 128 + 128, sq))
        active_chunks = set()
        for row in rows:
            for j in J[row // br]:
                for c in range(j * bc, min((j + 1) * bc, sk)):
                    active_chunks.add(c // 128)
        assert active_chunks <= need
        assert need <= active_chunks


def test_shard_bounds_partition():
    for n in (0, 1, 7, 64):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(shard_counts(n, world)) - min(shard_counts(n, world)) <= 1
    assert shard_counts(64, 8) == [8] * 8


def test_bench_csv_bytes_match_reference():
    """api.bench_csv writes the reference's bytes (encoder.py:439-444); the expected string is the
    output of the reference's own bench_csv on these rows (generated with zstripe.encoder)."""
    from paper_2605_17633_b200 import api

    rows = [api.BenchRow(0.25, 0.3125, 1.23456, 2.5), api.BenchRow(1.0, 1.0, 10.0, 1.0)]
    assert api.bench_csv(rows) == ("density,achieved_density,median_ms,speedup\r\n0.25,0.3125,1.235,2.5000\r\n"
                                   "1.0,1.0,10.000,1.0000\r\n")


def test_module_api_mirrors_sam_parameter_tree():
    """modules.SparseSAMImageEncoderViT has SAM ImageEncoderViT's parameter names and shapes (ViT-B
    constructor arguments of segment_anything build_sam_vit_b), so SAM state_dicts load."""
    from paper_2605_17633_b200 import modules as M

    enc = M.SparseSAMImageEncoderViT(depth=12, embed_dim=768, img_size=1024, mlp_ratio=4, num_heads=12,
                                     qkv_bias=True, use_rel_pos=True, global_attn_indexes=(2, 5, 8, 11),
                                     window_size=14, out_chans=256)
    sd = enc.state_dict()
    assert sd["patch_embed.proj.weight"].shape == (768, 3, 16, 16) and sd["pos_embed"].shape == (1, 64, 64, 768)
    assert sd["blocks.0.attn.qkv.weight"].shape == (2304, 768) and sd["blocks.0.attn.rel_pos_h"].shape == (27, 64)
    assert sd["blocks.2.attn.rel_pos_w"].shape == (127, 64) and sd["blocks.3.mlp.lin1.weight"].shape == (3072, 768)
    assert sd["neck.0.weight"].shape == (256, 768, 1, 1) and sd["neck.2.weight"].shape == (256, 256, 3, 3)
    assert sd["neck.3.bias"].shape == (256,)
    assert [b.kind for b in enc.blocks].count("global") == 4
    assert len(sd) == 3 + 12 * 14 + 6  # SAM vit_b image encoder: 177 entries


def test_from_sam_image_encoder_copies_config_and_weights():
    """modules.from_sam_image_encoder reads a SAM ImageEncoderViT's configuration from its attributes
    (duck-typed; here a module with SAM's tree) and loads its state_dict."""
    import torch

    from paper_2605_17633_b200 import modules as M

    torch.manual_seed(0)
    src = M.SparseSAMImageEncoderViT(img_size=320, embed_dim=128, depth=3, num_heads=2, window_size=6,
                                     global_attn_indexes=(1,), use_rel_pos=True, rel_pos_zero_init=False)
    dst = M.from_sam_image_encoder(src, density=0.3, keep_fraction=0.5)
    assert [b.kind for b in dst.blocks] == ["local", "global", "local"]
    assert dst.blocks[0].window_size == 6 and dst.blocks[0].attn.density == 0.3
    assert dst.blocks[2].mlp.keep_fraction == 0.5
    for k, v in src.state_dict().items():
        assert torch.equal(dst.state_dict()[k], v), k
