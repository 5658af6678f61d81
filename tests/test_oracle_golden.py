"""Pin the oracle (oracle/zs_oracle.py) against the reference's own golden vectors.

Two sources: (1) the reference's known-answer tests (quoted with file:line),
(2) outputs of the reference itself, committed under tests/golden/ by
tests/golden/make_golden.py.  CPU only.
"""

import math

import numpy as np
import pytest

from conftest import golden
from oracle import zs_oracle as O


# ---------------------------------------------------------------- known answers (reference tests)
def test_morton_known_answers():
    # test_grid.py:37-39: morton_encode(2, 3) == 14 ; test_grid.py:61-64: first quad of 4x4 is [0,1,4,5]
    codes = O.morton_codes(4, 4)
    assert int(codes[3 * 4 + 2]) == 14
    assert O.morton_order(4, 4)[:4].tolist() == [0, 1, 4, 5]


def test_morton_aligned_quads_on_window_and_grid():
    # Morton groups of 4 are aligned 2x2 cells for 64x64 and 14x14
    for n in (64, 14):
        mo = O.morton_order(n, n).reshape(-1, 4)
        ys, xs = np.divmod(mo, n)
        assert (ys.max(1) - ys.min(1) == 1).all() and (xs.max(1) - xs.min(1) == 1).all()
        assert (ys.min(1) % 2 == 0).all() and (xs.min(1) % 2 == 0).all()


def test_stripe_known_answer():
    # test_stripesort.py:27-31
    assert O.stripe_sort(np.arange(8), 4).tolist() == [0, 4, 1, 5, 2, 6, 3, 7]


def test_sobel_step_edge_known_answer():
    # test_saliency.py:54-63: a vertical step edge of height 1 gives magnitude 4 on the edge columns
    x = np.zeros((6, 6, 1), np.float32)
    x[:, 3:] = 1.0
    m = O.sobel_magnitude(x)
    assert m[2, 2] == 4.0 and m[2, 3] == 4.0


def test_group_energy_known_answer():
    # test_saliency.py:117-122: a single salient token in the first quad
    sal = np.zeros(16, np.float32)
    sal[5] = 5.0
    e = O.group_energy(sal, O.morton_order(4, 4), 4)
    assert e.tolist() == [5.0, 0.0, 0.0, 0.0]


def test_active_set_known_answers():
    # test_attention.py:94-112
    assert O.active_set(8, 8, 0.25)[5] == (0, 1, 5)
    assert O.active_set(4, 4, 0.0) == [(0,), (1,), (2,), (3,)]
    assert O.active_set(6, 3, 0.0) == [(0,), (1,), (2,), (2,), (2,), (2,)]


def test_achieved_density_known_answers():
    # test_attention.py:132-135
    def dens(t, r):
        return sum(len(j) for j in O.active_set(t, t, r)) / (t * t)

    assert dens(8, 0.25) == 22 / 64
    assert dens(32, 0.25) == 0.2734375


def test_keep_count_known_answers():
    # test_mlp.py:122-126 (banker's rounding)
    assert [O.keep_count(0.5, 8), O.keep_count(0.5, 7), O.keep_count(0.01, 10), O.keep_count(0.25, 10)] == [4, 4, 1, 2]
    assert O.keep_count(0.4, 196) == 78 and O.keep_count(0.4, 4096) == 1638


# ---------------------------------------------------------------- golden vectors (reference outputs)
def test_splitmix_matches_reference_stream():
    # tests/golden/config1 orderings were produced from zstripe.Rng(1).normal((64,64,768));
    # the oracle regenerates the same input and must reproduce those orderings
    x = O.SplitMix(1).normal((64, 64, 768))
    g = golden("orders_config1")
    assert np.array_equal(O.sobel_magnitude(x)[::7], g["sobel_rows"])


def test_morton_orders_golden():
    g = golden("orders_small")
    for h, w in [(4, 4), (14, 14), (6, 10), (64, 64)]:
        assert np.array_equal(O.morton_order(h, w), g[f"morton_{h}x{w}"])
        assert np.array_equal(O.morton_codes(h, w).astype(np.int64), g[f"codes_{h}x{w}"])


@pytest.mark.parametrize("gran", ["zgroup", "token"])
@pytest.mark.parametrize("var", ["full", "no_interleave", "no_sort"])
def test_orderings_small_golden(gran, var):
    g = golden("orders_small")
    x = O.SplitMix(1).normal((20, 20, 24))
    o = O.orderings(x, 6, cfg=O.OrderCfg(4, var, gran, 4))
    assert np.array_equal(o["global"], g[f"small_{gran}_{var}_global"])
    assert np.array_equal(o["local"], g[f"small_{gran}_{var}_local"])


def test_sobel_energy_pi_small_golden():
    g = golden("orders_small")
    x = O.SplitMix(1).normal((20, 20, 24))
    sal = O.sobel_magnitude(x)
    assert np.array_equal(sal, g["small_sobel"])
    assert np.array_equal(O.group_energy(sal.reshape(-1), O.morton_order(20, 20), 4), g["small_energy"])
    assert np.array_equal(O.importance_order(sal.reshape(-1), 20, 20), g["small_pi"])


def test_orderings_config1_golden():
    g = golden("orders_config1")
    x = O.SplitMix(1).normal((64, 64, 768))
    o = O.orderings(x, 14)
    assert np.array_equal(o["global"], g["sigma_global"])
    assert np.array_equal(o["local"], g["sigma_local"])


def test_attention_golden():
    g = golden("attention_cases")
    for ci in range(5):
        sq, w, dh, br, bc = g[f"c{ci}_shape"].tolist()
        for r in (0.0, 0.25, 0.4, 1.0):
            out = O.ashape_attention(g[f"c{ci}_q"], g[f"c{ci}_k"], g[f"c{ci}_v"], g[f"c{ci}_bh"], g[f"c{ci}_bw"],
                                     g[f"c{ci}_sp"], g[f"c{ci}_kp"], br, bc, r, mm=O.matmul_fixed)
            ref = g[f"c{ci}_r{int(r * 100)}"]
            np.testing.assert_allclose(out, ref, rtol=0, atol=2e-6)


def test_active_sets_golden():
    g = golden("attention_cases")
    for key in [k for k in g if k.startswith("active_")]:
        tr, tc, rm = map(int, key.split("_")[1:])
        r = rm / 1000
        flat = [(i, j) for i, js in enumerate(O.active_set(tr, tc, r)) for j in js]
        assert np.array_equal(np.array(flat), g[key]), key


def test_route_mlp_golden():
    g = golden("mlp_cases")
    for ci in range(4):
        n, dm, fm, byp = g[f"c{ci}_meta"].tolist()
        p = O.Mlp(g[f"c{ci}_w1"], g[f"c{ci}_b1"], g[f"c{ci}_w2"], g[f"c{ci}_b2"], g[f"c{ci}_g"], g[f"c{ci}_b"])
        out = O.route_mlp(g[f"c{ci}_x"], p, g[f"c{ci}_sig"], fm / 1000, "layernorm" if byp else "identity",
                          mm=O.matmul_fixed)
        np.testing.assert_allclose(out, g[f"c{ci}_out"], rtol=0, atol=1e-6)
    for fm, n, k in g["keep_counts"].tolist():
        assert O.keep_count(fm / 1000, n) == k


def _small_cfg():
    return O.EncCfg(h=20, w=20, d=128, heads=2, window=6, layout=("local", "global", "local", "local"),
                    r=(0.4,) * 4, keep=(0.4,) * 4, seed=5)


@pytest.mark.parametrize("mode", ["sparse", "dense"])
def test_encoder_small_golden_bitexact(mode):
    g = golden("encoder_small")
    cfg = _small_cfg()
    x = O.SplitMix(3).normal((20, 20, 128))
    y = O.encoder_forward(x, O.init_weights(cfg), cfg, mode=mode, mm=O.matmul_fixed)
    assert np.array_equal(y, g[mode])


def test_config1_local_block_golden():
    """Config 1 (one ViT-B local block, density 0.4) — the oracle with BLAS matmul vs the reference."""
    g = golden("config1_blocks")
    cfg = O.EncCfg(layout=("local",), r=(0.4,), keep=(0.4,))
    x = O.SplitMix(1).normal((64, 64, 768))
    y = O.encoder_forward(x, O.init_weights(cfg), cfg).reshape(4096, 768)
    np.testing.assert_allclose(y[g["rows"]], g["local_rows"], rtol=0, atol=1e-4)
    np.testing.assert_allclose(y.sum(1), g["local_rowsum"], rtol=0, atol=2e-3)


def test_reference_sparse_equals_dense_at_full_density():
    # test_encoder.py:205-213: sparse(r=1, keep=1) == dense, bit-exact
    cfg = O.EncCfg(h=12, w=12, d=64, heads=2, window=6, layout=("local", "global"), r=(1.0, 1.0), keep=(1.0, 1.0))
    x = O.SplitMix(9).normal((12, 12, 64))
    w = O.init_weights(cfg)
    assert np.array_equal(O.encoder_forward(x, w, cfg, "sparse", mm=O.matmul_fixed),
                          O.encoder_forward(x, w, cfg, "dense", mm=O.matmul_fixed))


def test_schedule_table_survey_8d():
    # SURVEY §8(d) static schedule per density (local T=7 / global T=32)
    table = {0.2: (1, 6, 39, 819), 0.3: (2, 9, 59, 1229), 0.4: (2, 12, 78, 1638), 0.5: (3, 16, 98, 2048),
             0.6: (4, 19, 118, 2458), 0.7: (4, 22, 137, 2867), 0.8: (5, 25, 157, 3277), 0.9: (6, 28, 176, 3686),
             1.0: (7, 32, 196, 4096)}
    for d, (pl, pg, kl, kg) in table.items():
        assert math.floor(d * 7) == pl and math.floor(d * 32) == pg
        assert O.keep_count(d, 196) == kl and O.keep_count(d, 4096) == kg


def _global_case(g, ci):
    dh, rm, seed = g[f"g{ci}_meta"].tolist()
    rng = O.SplitMix(seed)
    q, k, v = rng.normal((4096, dh)), rng.normal((4096, dh)), rng.normal((4096, dh))
    bh, bw = rng.normal((4096, 64), std=0.5), rng.normal((4096, 64), std=0.5)
    return q, k, v, bh, bw, g[f"g{ci}_sp"].astype(np.int64), rm / 1000, g[f"g{ci}_out"]


@pytest.mark.parametrize("ci", [0, 1])
def test_global_attention_golden(ci):
    """SAM global-attention shape (S = 4096, tile 128, dh 80 / 64): the oracle's streaming
    attention (BLAS matmul) vs the reference's own output."""
    q, k, v, bh, bw, sp, r, ref = _global_case(golden("attention_global"), ci)
    out = O.ashape_attention(q, k, v, bh, bw, sp, sp, 128, 128, r)
    np.testing.assert_allclose(out, ref, rtol=0, atol=2e-5)


def test_masked_attention_f64_pinned_to_reference():
    """The float64 masked-softmax checker the 4096-token / ViT-H GPU tests use is itself pinned to
    the reference's outputs: every attention golden (5 small cases x 4 densities, 2 global heads)."""
    g = golden("attention_cases")
    for ci in range(5):
        sq, w, dh, br, bc = g[f"c{ci}_shape"].tolist()
        for r in (0.0, 0.25, 0.4, 1.0):
            out = O.masked_attention_f64(g[f"c{ci}_q"], g[f"c{ci}_k"], g[f"c{ci}_v"], g[f"c{ci}_bh"], g[f"c{ci}_bw"],
                                         g[f"c{ci}_sp"], g[f"c{ci}_kp"], br, bc, r)
            np.testing.assert_allclose(out, g[f"c{ci}_r{int(r * 100)}"], rtol=0, atol=5e-6)
    gg = golden("attention_global")
    for ci in range(2):
        q, k, v, bh, bw, sp, r, ref = _global_case(gg, ci)
        out = O.masked_attention_f64(q, k, v, bh, bw, sp, sp, 128, 128, r)
        np.testing.assert_allclose(out, ref, rtol=0, atol=2e-5)
