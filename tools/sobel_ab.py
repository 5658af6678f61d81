"""A/B of zs_sobel_saliency between the current library and _old (bit-exact outputs, timing), ViT-H grid."""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import _lib  # noqa: E402

libs = {n: ctypes.CDLL(str(Path(_lib.LIB_PATH).parent / f)) for n, f in
        [("new", "libzstripe_b200.so"), ("old", "libzstripe_b200_old.so")]}
for l in libs.values():
    l.zs_sobel_saliency.argtypes = _lib.SIGNATURES["zs_sobel_saliency"]
B, H, W, C, win = 64, 64, 64, 1280, 14
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.randn(B, H, W, C, device="cuda", generator=g)
x[0, 3, 5, 7] = float("inf")  # non-finite inputs follow the reference's rules too
x[1, 10, 13, 0] = float("nan")
Hp = -(-H // win) * win
out = {n: (torch.empty(B, H * W, device="cuda"), torch.empty(B, Hp * Hp, device="cuda")) for n in libs}
st = torch.cuda.current_stream().cuda_stream
for n, l in libs.items():
    assert l.zs_sobel_saliency(x.data_ptr(), B, H, W, C, win, out[n][0].data_ptr(), out[n][1].data_ptr(), st) == 0
torch.cuda.synchronize()
for i in range(2):
    a, b = out["new"][i], out["old"][i]
    same = torch.equal(a.view(torch.int32), b.view(torch.int32))
    print("map", i, "bit-identical" if same else f"DIFFER {(a != b).sum().item()}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    for n, l in libs.items():
        e0.record()
        for _ in range(10):
            l.zs_sobel_saliency(x.data_ptr(), B, H, W, C, win, out[n][0].data_ptr(), out[n][1].data_ptr(), st)
        e1.record()
        torch.cuda.synchronize()
        print(n, f"{e0.elapsed_time(e1) / 10:.3f} ms")
