"""A/B timing of zs_layernorm_rows_ex (gathered rows, bf16 out) from two library builds (same box)."""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200 import _lib  # noqa: E402

libs = {name: ctypes.CDLL(str(Path(_lib.LIB_PATH).parent / f)) for name, f in
        [("new", "libzstripe_b200.so"), ("old", "libzstripe_b200_old.so")]}
for l in libs.values():
    l.zs_layernorm_rows_ex.argtypes = _lib.SIGNATURES["zs_layernorm_rows_ex"]
C, R = 1280, 64 * 4900
x = torch.randn(R, C, device="cuda")
keep = torch.rand(R, device="cuda") > 0.164
rows = torch.nonzero(keep).int().flatten()
n = rows.numel()
out = torch.empty(n, C, device="cuda", dtype=torch.bfloat16)
g, b = torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")
st = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rnd in range(3):
    for name, lib in libs.items():
        call = lambda: lib.zs_layernorm_rows_ex(x.data_ptr(), C, rows.data_ptr(), None, n, None, C, g.data_ptr(),  # noqa
                                                b.data_ptr(), 1e-6, out.data_ptr(), C, 0, st)
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"round {rnd} ln {name}: {ms:.3f} ms {n * C * 6 / ms / 1e6:.0f} GB/s", flush=True)
