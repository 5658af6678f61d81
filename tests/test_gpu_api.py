"""Reference-API parity: the functional API of paper_2605_17633_b200 vs the reference's own outputs.

These read like the reference's tests (pkg/tests/test_attention.py, test_mlp.py,
test_saliency.py, test_stripesort.py) but run the B200 kernels and compare with
golden outputs produced by the reference itself (tests/golden/).
"""

import numpy as np
import pytest

from conftest import golden
from oracle import zs_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2605_17633_b200 as Z
    from paper_2605_17633_b200 import api


def test_sobel_importance_stripe_bitexact():
    g = golden("orders_small")
    x = O.SplitMix(1).normal((20, 20, 24))
    sal = api.sobel_magnitude(x)
    assert isinstance(sal.values, np.ndarray) and np.array_equal(sal.values, g["small_sobel"])
    mo = api.morton_order(Z.GridShape(20, 20))
    assert np.array_equal(api.group_energy(sal, mo, 4), g["small_energy"])
    pi = api.importance_order(sal, Z.OrderingConfig())
    assert np.array_equal(pi.forward, g["small_pi"])
    sig = api.stripe_sort(pi, Z.StripeConfig(4, "full"), morton=mo)
    assert np.array_equal(sig.forward, g["small_zgroup_full_global"])
    assert np.array_equal(api.stripe_sort(pi, Z.StripeConfig(4, "no_sort"), morton=mo).forward,
                          g["small_zgroup_no_sort_global"])
    assert np.array_equal(api.importance_order(sal, Z.OrderingConfig("token")).forward,
                          g["small_token_no_interleave_global"])
    assert np.array_equal(api.importance_order_from_energy(g["small_energy"], mo).forward, g["small_pi"])


def test_stripe_sort_known_answer_and_errors():
    assert api.stripe_sort(api.Permutation(np.arange(8)), Z.StripeConfig(4)).forward.tolist() == [0, 4, 1, 5, 2, 6,
                                                                                                    3, 7]
    with pytest.raises(ValueError):
        api.stripe_sort(api.Permutation(np.arange(6)), Z.StripeConfig(4))
    with pytest.raises(ValueError):
        api.stripe_sort(api.Permutation(np.arange(8)), Z.StripeConfig(4, "no_sort"))


@pytest.mark.parametrize("ci", range(5))
@pytest.mark.parametrize("r", [0.0, 0.25, 0.4, 1.0])
def test_ashape_attention_vs_reference(ci, r):
    """Reference ashape_attention outputs (fp32) vs the bf16 tcgen05 kernel.

    Tolerance: relative Frobenius error <= 1e-2 and max-abs <= 3e-2 (bf16 q/k/v
    and P with fp32 accumulation; measured ~2-4e-3 relative).
    """
    g = golden("attention_cases")
    sq, w, dh, br, bc = g[f"c{ci}_shape"].tolist()
    out = api.ashape_attention(g[f"c{ci}_q"], g[f"c{ci}_k"], g[f"c{ci}_v"], api.BiasTables(g[f"c{ci}_bh"],
                               g[f"c{ci}_bw"]), api.Permutation(g[f"c{ci}_sp"]), api.Permutation(g[f"c{ci}_kp"]),
                               Z.AShapeConfig(br, bc, r))
    ref = g[f"c{ci}_r{int(r * 100)}"]
    assert out.shape == ref.shape and out.dtype == np.float32
    err = np.linalg.norm(out - ref) / np.linalg.norm(ref)
    assert err < 1e-2 and np.abs(out - ref).max() < 3e-2, (err, np.abs(out - ref).max())


def test_attention_input_checks_raise_valueerror():
    q = np.zeros((16, 64), np.float32)
    k = np.zeros((16, 64), np.float32)
    b = api.BiasTables(np.zeros((16, 4), np.float32), np.zeros((16, 4), np.float32))
    p = api.Permutation.identity(16)
    with pytest.raises(ValueError):
        api.ashape_attention(q, k[:, :32], k, b, p, p, Z.AShapeConfig())
    with pytest.raises(ValueError):
        api.ashape_attention(q, k, k[:8], b, p, p, Z.AShapeConfig())
    with pytest.raises(ValueError):
        api.ashape_attention(q, k, k, api.BiasTables(np.zeros((16, 3), np.float32), np.zeros((16, 3), np.float32)), p,
                             p, Z.AShapeConfig())
    with pytest.raises(ValueError):
        Z.AShapeConfig(r=1.5)


def test_dense_attention_is_single_tile_ashape():
    g = golden("attention_cases")
    ci = 1
    args = (g[f"c{ci}_q"], g[f"c{ci}_k"], g[f"c{ci}_v"], api.BiasTables(g[f"c{ci}_bh"], g[f"c{ci}_bw"]),
            api.Permutation(g[f"c{ci}_sp"]), api.Permutation(g[f"c{ci}_kp"]))
    dense = api.dense_attention(*args)
    ref = g[f"c{ci}_r100"]
    assert np.linalg.norm(dense - ref) / np.linalg.norm(ref) < 1e-2


@pytest.mark.parametrize("ci", range(4))
def test_route_mlp_vs_reference(ci):
    """Kept rows within bf16 tolerance; bypassed rows bit-identical (identity) / LN (layernorm)."""
    g = golden("mlp_cases")
    n, dm, fm, byp = g[f"c{ci}_meta"].tolist()
    w = api.MlpWeights(g[f"c{ci}_w1"], g[f"c{ci}_b1"], g[f"c{ci}_w2"], g[f"c{ci}_b2"], g[f"c{ci}_g"], g[f"c{ci}_b"])
    cfg = Z.RouterConfig(fm / 1000, "layernorm" if byp else "identity")
    x = g[f"c{ci}_x"]
    out = api.route_mlp(x, w, api.Permutation(g[f"c{ci}_sig"]), cfg)
    ref = g[f"c{ci}_out"]
    kc = cfg.keep_count(n)
    keep = g[f"c{ci}_sig"][:kc]
    rest = g[f"c{ci}_sig"][kc:]
    e = np.linalg.norm(out[keep] - ref[keep]) / np.linalg.norm(ref[keep])
    assert e < 1e-2, e
    if byp:
        np.testing.assert_allclose(out[rest], ref[rest], rtol=0, atol=1e-5)
    else:
        assert np.array_equal(out[rest], x[rest])


def test_route_mlp_checks():
    w = api.MlpWeights(np.zeros((64, 256)), np.zeros(256), np.zeros((256, 64)), np.zeros(64), np.ones(64),
                       np.zeros(64))
    with pytest.raises(ValueError):
        api.route_mlp(np.zeros((10, 32), np.float32), w, api.Permutation.identity(10), Z.RouterConfig(0.5))
    with pytest.raises(ValueError):
        api.route_mlp(np.zeros((10, 64), np.float32), w, api.Permutation.identity(9), Z.RouterConfig(0.5))
    with pytest.raises(ValueError):
        Z.RouterConfig(0.0)


def test_cost_report_matches_reference_accounting():
    """CostReport columns (minus wall time) equal the reference's (encoder.py:372-384)."""
    g = golden("encoder_small")
    cfg = Z.EncoderConfig(grid=Z.GridShape(20, 20), d=128, heads=2, window=6,
                          layout=("local", "global", "local", "local"), r=0.4, keep_fraction=0.4, seed=5)
    ref = bytes(g["cost_csv"]).decode().split("\r\n")
    mine = api.cost_report(cfg).csv(with_ms=False).split("\r\n")
    assert mine[0] == ref[0]
    for a, b in zip(mine[1:], ref[1:]):
        assert a.rsplit(",", 1)[0] == b.rsplit(",", 1)[0]


@pytest.mark.parametrize("ci", [0, 1])
def test_global_attention_vs_reference_golden(ci):
    """S = 4096 global heads (dh 80 / 64, tile 128) straight against the reference's own output
    (tests/golden/attention_global.npz), not only the oracle."""
    from test_oracle_golden import _global_case

    q, k, v, bh, bw, sp, r, ref = _global_case(golden("attention_global"), ci)
    got = api.ashape_attention(q, k, v, api.BiasTables(bh, bw), sp, sp, Z.AShapeConfig(b_row=128, b_col=128, r=r))
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel <= 1e-2 and np.abs(got - ref).max() <= 3e-2, (rel, np.abs(got - ref).max())


@pytest.mark.gpu
def test_bench_schema_matches_reference():
    """api.bench / bench_csv / attn_bench: the reference's columns, number formats and speedup
    definition (encoder.py:388-444, cli.py:96-130), timed on the device."""
    import re

    from paper_2605_17633_b200 import api
    from paper_2605_17633_b200.config import EncoderConfig, GridShape

    cfg = EncoderConfig(grid=GridShape(64, 64), d=768, heads=12, window=14, layout=("local", "global"), r=0.4,
                        keep_fraction=0.4, seed=3)
    rows = api.bench(cfg, [0.25, 1.0], repeats=2)
    assert [r.density for r in rows] == [0.25, 1.0]
    assert all(r.median_ms > 0 and r.speedup > 0 for r in rows)
    assert rows[1].achieved_density == 1.0
    assert rows[0].achieved_density == api.cost_report(__import__("dataclasses").replace(cfg, r=0.25)).attn_density()
    csv = api.bench_csv(rows)
    lines = csv.split("\r\n")
    assert lines[0] == api.BENCH_COLUMNS == "density,achieved_density,median_ms,speedup" and lines[-1] == ""
    assert re.fullmatch(r"0\.25,[0-9.e-]+,\d+\.\d{3},\d+\.\d{4}", lines[1])
    ab = api.attn_bench(n=1024, d=64, densities=(0.25, 0.5, 0.25), repeats=3, tile=128)
    al = ab.split("\r\n")
    assert al[0] == api.BENCH_COLUMNS and len(al) == 5 and al[-1] == ""
    assert al[1].startswith("0.25,0.") and al[3].startswith("0.25,")
    with pytest.raises(ValueError):
        api.attn_bench(n=1000)
