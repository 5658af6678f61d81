"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (where /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
The GPU box has no /root/reference; tests read only the .npz files written here.
Inputs are regenerated in the tests from (seed, shape) with the oracle's
splitmix64 restatement (bit-exact with zstripe.Rng), so only outputs and
small inputs are stored.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import zstripe as Z  # noqa: E402

OUT = Path(__file__).resolve().parent


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz ({(OUT / f'{name}.npz').stat().st_size} B)")


def grid_and_orders():
    d = {}
    for h, w in [(4, 4), (14, 14), (6, 10), (64, 64)]:
        d[f"morton_{h}x{w}"] = Z.morton_order(Z.GridShape(h, w)).forward
        d[f"codes_{h}x{w}"] = Z.morton_codes(Z.GridShape(h, w)).astype(np.int64)
    # orderings on a small grid, all variants / granularities
    x = Z.Rng(1).normal((20, 20, 24))
    for gran in ("zgroup", "token"):
        for var in ("full", "no_interleave", "no_sort"):
            cfg = Z.EncoderConfig(grid=Z.GridShape(20, 20), d=24, heads=2, window=6, layout=("local", "global"),
                                  stripe=Z.StripeConfig(4, var), ordering=Z.OrderingConfig(gran, 4))
            o = Z.encoder._orderings(x, cfg)
            d[f"small_{gran}_{var}_global"] = o["global"].forward
            d[f"small_{gran}_{var}_local"] = np.stack([s.forward for s in o["local"]])
    d["small_sobel"] = Z.sobel_magnitude(x).values
    # group energies and their order (the "fed the reference's scores" gate)
    sal = Z.sobel_magnitude(x)
    mo = Z.morton_order(sal.shape)
    d["small_energy"] = Z.group_energy(sal, mo, 4)
    d["small_pi"] = Z.importance_order(sal, Z.OrderingConfig()).forward
    save("orders_small", **d)


def config1_orders():
    x = Z.Rng(1).normal((64, 64, 768))
    cfg = Z.EncoderConfig(grid=Z.GridShape(64, 64), d=768, heads=12, window=14, layout=("local", "global"))
    t = time.time()
    o = Z.encoder._orderings(x, cfg)
    print("config-1 orderings", time.time() - t)
    sal = Z.sobel_magnitude(x).values
    save("orders_config1", sigma_global=o["global"].forward.astype(np.int32),
         sigma_local=np.stack([s.forward for s in o["local"]]).astype(np.int32),
         sobel_rows=sal[::7].copy())


def attention_cases():
    rng = np.random.default_rng(20240821)
    d = {}
    cases = [(100, 9, 64, 32, 32), (196, 14, 64, 32, 32), (196, 14, 80, 32, 32), (130, 12, 64, 128, 128),
             (70, 9, 80, 16, 24)]
    for ci, (sq, w, dh, br, bc) in enumerate(cases):
        sk = w * w
        q = rng.standard_normal((sq, dh)).astype(np.float32)
        k = rng.standard_normal((sk, dh)).astype(np.float32)
        v = rng.standard_normal((sk, dh)).astype(np.float32)
        bh = (0.5 * rng.standard_normal((sq, w))).astype(np.float32)
        bw = (0.5 * rng.standard_normal((sq, w))).astype(np.float32)
        sp, kp = rng.permutation(sq), rng.permutation(sk)
        d.update({f"c{ci}_q": q, f"c{ci}_k": k, f"c{ci}_v": v, f"c{ci}_bh": bh, f"c{ci}_bw": bw, f"c{ci}_sp": sp,
                  f"c{ci}_kp": kp, f"c{ci}_shape": np.array([sq, w, dh, br, bc])})
        for r in (0.0, 0.25, 0.4, 1.0):
            out = Z.ashape_attention(q, k, v, Z.BiasTables(bh, bw), Z.Permutation(sp), Z.Permutation(kp),
                                     Z.AShapeConfig(br, bc, r))
            d[f"c{ci}_r{int(r * 100)}"] = out
    # active sets / achieved density known answers
    sets = []
    for tr, tc, r in [(8, 8, 0.25), (4, 4, 0.0), (3, 5, 1.0), (6, 3, 0.0), (7, 7, 0.4), (32, 32, 0.4), (7, 7, 0.3),
                      (32, 32, 0.2), (13, 9, 0.77)]:
        a = Z.build_active_set(tr, tc, r)
        flat = [(i, j) for i, js in enumerate(a.tiles) for j in js]
        sets.append(np.array([[tr, tc, int(r * 1000), len(flat)]]))
        d[f"active_{tr}_{tc}_{int(r * 1000)}"] = np.array(flat, dtype=np.int64)
        d[f"density_{tr}_{tc}_{int(r * 1000)}"] = np.array(Z.achieved_density(tr, tc, r))
    save("attention_cases", **d)


def mlp_cases():
    rng = np.random.default_rng(7)
    d = {}
    for ci, (n, dm, f, byp) in enumerate([(50, 64, 0.4, "identity"), (196, 128, 0.4, "layernorm"),
                                         (77, 64, 1.0, "identity"), (33, 64, 0.05, "identity")]):
        x = rng.standard_normal((n, dm)).astype(np.float32)
        hid = 4 * dm
        w = Z.MlpWeights(w1=(rng.standard_normal((dm, hid)) / np.sqrt(dm)).astype(np.float32),
                         b1=(0.1 * rng.standard_normal(hid)).astype(np.float32),
                         w2=(rng.standard_normal((hid, dm)) / np.sqrt(hid)).astype(np.float32),
                         b2=(0.1 * rng.standard_normal(dm)).astype(np.float32),
                         ln_gamma=(1 + 0.1 * rng.standard_normal(dm)).astype(np.float32),
                         ln_beta=(0.1 * rng.standard_normal(dm)).astype(np.float32))
        sig = rng.permutation(n)
        out = Z.route_mlp(x, w, Z.Permutation(sig), Z.RouterConfig(f, byp))
        d.update({f"c{ci}_x": x, f"c{ci}_w1": w.w1, f"c{ci}_b1": w.b1, f"c{ci}_w2": w.w2, f"c{ci}_b2": w.b2,
                  f"c{ci}_g": w.ln_gamma, f"c{ci}_b": w.ln_beta, f"c{ci}_sig": sig, f"c{ci}_out": out,
                  f"c{ci}_meta": np.array([n, dm, int(f * 1000), int(byp == "layernorm")])})
    kc = []
    for f, n in [(0.5, 8), (0.5, 7), (0.5, 9), (0.01, 10), (0.4, 196), (0.4, 4096), (0.3, 196), (0.25, 10),
                 (0.75, 6)]:
        kc.append([int(f * 1000), n, Z.RouterConfig(f).keep_count(n)])
    d["keep_counts"] = np.array(kc)
    save("mlp_cases", **d)


def encoder_small():
    """Small multi-block encoder (pads, local + global, both modes)."""
    x = Z.Rng(3).normal((20, 20, 128))
    cfg = Z.EncoderConfig(grid=Z.GridShape(20, 20), d=128, heads=2, window=6,
                          layout=("local", "global", "local", "local"), r=0.4, keep_fraction=0.4, seed=5)
    w = Z.init_weights(cfg)
    ys, rep = Z.encoder_forward(x, w, cfg, mode="sparse")
    yd, _ = Z.encoder_forward(x, w, cfg, mode="dense")
    save("encoder_small", sparse=ys, dense=yd, cost_csv=np.frombuffer(rep.csv().encode(), dtype=np.uint8))


def config1_blocks():
    """Config 1: one ViT-B block (64x64, 768, 12 heads, density 0.4), local and global."""
    x = Z.Rng(1).normal((64, 64, 768))
    rows = np.arange(0, 4096, 32)
    out = {}
    for kind in ("local", "global"):
        cfg = Z.EncoderConfig(grid=Z.GridShape(64, 64), d=768, heads=12, window=14, layout=(kind,), r=0.4,
                              keep_fraction=0.4, seed=0)
        w = Z.init_weights(cfg)
        t = time.time()
        y, rep = Z.encoder_forward(x, w, cfg, mode="sparse")
        print(f"config-1 {kind} block: {time.time() - t:.1f} s")
        flat = y.reshape(4096, 768)
        out[f"{kind}_rows"] = flat[rows]
        out[f"{kind}_rowsum"] = flat.sum(axis=1)
        out[f"{kind}_seconds"] = np.array(time.time() - t)
    out["rows"] = rows
    save("config1_blocks", **out)


def attention_global():
    """Global-attention shapes of SAM ViT-B/H (S = 4096 = 64x64, tile 128): one head each, the
    reference's own ashape_attention output.  Inputs come from zstripe.Rng(seed) (regenerated in
    the tests by the oracle's bit-exact SplitMix), only the key permutation and outputs are stored."""
    d = {}
    for ci, (dh, r, seed) in enumerate([(80, 0.4, 31), (64, 0.25, 32)]):
        g = Z.Rng(seed)
        q, k, v = g.normal((4096, dh)), g.normal((4096, dh)), g.normal((4096, dh))
        bh, bw = g.normal((4096, 64), std=0.5), g.normal((4096, 64), std=0.5)
        sp = np.random.default_rng(seed).permutation(4096)
        t = time.time()
        out = Z.ashape_attention(q, k, v, Z.BiasTables(bh, bw), Z.Permutation(sp), Z.Permutation(sp),
                                 Z.AShapeConfig(128, 128, r))
        print(f"global attention dh={dh} r={r}: {time.time() - t:.1f} s")
        d.update({f"g{ci}_meta": np.array([dh, int(r * 1000), seed]), f"g{ci}_sp": sp.astype(np.int16),
                  f"g{ci}_out": out})
    save("attention_global", **d)


def sptn_files():
    """SPTN files written by the reference (tensor.py:65-84, grid.py:122-127) for the reader/writer gate."""
    d = OUT / "sptn"
    d.mkdir(exist_ok=True)
    Z.tensor_write(np.array([3.0], dtype=np.float32), d / "scalar.sptn")
    Z.tensor_write(Z.Rng(7).normal((3, 5, 4)), d / "rank3.sptn")
    Z.tensor_write(Z.sobel_magnitude(Z.Rng(1).normal((6, 10, 8))).values, d / "sobel_6x10.sptn")
    Z.permutation_write(Z.morton_order(Z.GridShape(6, 10)), d / "morton_6x10.sptn")
    print("wrote", sorted(p.name for p in d.iterdir()))


if __name__ == "__main__":
    which = sys.argv[1:] or ["grid", "c1orders", "attn", "mlp", "enc", "c1blocks", "sptn", "attn_global"]
    if "sptn" in which:
        sptn_files()
    if "grid" in which:
        grid_and_orders()
    if "c1orders" in which:
        config1_orders()
    if "attn" in which:
        attention_cases()
    if "mlp" in which:
        mlp_cases()
    if "enc" in which:
        encoder_small()
    if "c1blocks" in which:
        config1_blocks()
    if "attn_global" in which:
        attention_global()
