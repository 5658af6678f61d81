"""A/B timing of zs_stripe_attn_fwd from two library builds on the same box (interleaved rounds).

    python tools/attn_ab.py [local|global] [B]   (needs _lib/libzstripe_b200_old.so next to the library)
"""
import ctypes
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import _lib  # noqa: E402

import os  # noqa: E402
# ZS_AB_LIBS="a.so,b.so,...": variants in _lib/ timed against the first (default: new vs _old)
_names = os.environ.get("ZS_AB_LIBS", "libzstripe_b200.so,libzstripe_b200_old.so").split(",")
libs = {("new" if i == 0 else ("old" if i == 1 else f)): ctypes.CDLL(str(Path(_lib.LIB_PATH).parent / f))
        for i, f in enumerate(_names)}
for l in libs.values():
    l.zs_stripe_attn_fwd.argtypes = _lib.SIGNATURES["zs_stripe_attn_fwd"]
    l.zs_stripe_attn_fwd_rows.argtypes = _lib.SIGNATURES["zs_stripe_attn_fwd_rows"]
ROWS = "rows" in sys.argv  # compacted output rows (the encoder's pad-skipping path): 16 % of rows dropped
kind = sys.argv[1] if len(sys.argv) > 1 else "local"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
H, dh = 16, 80
S, w, tile = (196, 14, 32) if kind == "local" else (4096, 64, 128)
U = B * 25 if kind == "local" else B
C = H * dh
p = math.floor(0.4 * (-(-S // tile)))
qkv = torch.randn(U * S, 3 * C, device="cuda").bfloat16()
bh = torch.randn(H, S, w, device="cuda") * 0.5
bw = torch.randn(H, S, w, device="cuda") * 0.5
sp = torch.argsort(torch.rand(U, S, device="cuda"), dim=1).int().contiguous()
if "stripes" in sys.argv:  # σ made of the 4 (y % 2, x % 2) parity classes, each shuffled (global stripes)
    pos = torch.arange(S, device="cuda")
    cls = ((pos // w) % 2) * 2 + (pos % w) % 2
    key = cls[None, :].float() * 2 + torch.rand(U, S, device="cuda")
    sp = torch.argsort(key, dim=1).int().contiguous()
outs = {n: torch.empty(U * S, C, device="cuda", dtype=torch.bfloat16) for n in libs}
wsn = _lib.load().zs_stripe_attn_ws_bytes(U, H, S, S, dh, 0)
ws = {n: torch.empty(wsn, device="cuda", dtype=torch.uint8) for n in libs}
st = torch.cuda.current_stream().cuda_stream


orows = None
if ROWS:
    keep = torch.rand(U * S, device="cuda") > 0.16
    orows = torch.where(keep, torch.cumsum(keep.int(), 0) - 1, torch.full_like(keep, -1, dtype=torch.long)).int()


def call(lib, out, name):
    q = qkv
    if ROWS:
        rc = lib.zs_stripe_attn_fwd_rows(q.data_ptr(), q.data_ptr() + 2 * C, q.data_ptr() + 4 * C, 3 * C, 3 * C,
                                         3 * C, S * 3 * C, S * 3 * C, U, H, S, S, dh, bh.data_ptr(), bw.data_ptr(), w,
                                         sp.data_ptr(), sp.data_ptr(), tile, tile, p, dh ** -0.5, out.data_ptr(), C,
                                         S * C, orows.data_ptr(), ws[name].data_ptr(), wsn, st)
        assert rc == 0, rc
        return
    rc = lib.zs_stripe_attn_fwd(q.data_ptr(), q.data_ptr() + 2 * C, q.data_ptr() + 4 * C, 3 * C, 3 * C, 3 * C,
                                S * 3 * C, S * 3 * C, U, H, S, S, dh, bh.data_ptr(), bw.data_ptr(), w, sp.data_ptr(),
                                sp.data_ptr(), tile, tile, p, dh ** -0.5, out.data_ptr(), C, S * C, ws[name].data_ptr(),
                                wsn, st)
    assert rc == 0, rc


e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
PAIRS = 20  # paired, finely interleaved samples: the power-capped clock drifts between rounds


def batch(name, n=4):
    e0.record()
    for _ in range(n):
        call(libs[name], outs[name], name)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for name in libs:
    for _ in range(2):
        call(libs[name], outs[name], name)
torch.cuda.synchronize()
names = list(libs)
times = {n: [] for n in names}
for i in range(PAIRS):
    order = names if i % 2 == 0 else names[::-1]
    for name in order:
        times[name].append(batch(name))
m = PAIRS // 2
ref = sorted(times["old"])[m]
for name in names:
    r = sorted(a / b for a, b in zip(times[name], times["old"]))
    print(f"{kind} {name:>28s}: median {sorted(times[name])[m]:.3f} ms  vs old {r[m]:.4f} "
          f"(q1 {r[PAIRS // 4]:.4f} q3 {r[3 * PAIRS // 4]:.4f})", flush=True)
    d = (outs[name].float() - outs["old"].float()).norm() / outs["old"].float().norm()
    print(f"   rel diff vs old: {d.item():.3e}")
