"""INTEGRATION.md's ctypes stub (the binding a zstripe maintainer would paste) runs as written:
on CPU it binds every symbol it names and its workspace query answers; on the GPU it reproduces
``api.ashape_attention`` (same kernel) bit for bit."""

import math
import os
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2605_17633_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def _stub() -> dict:
    text = (ROOT / "INTEGRATION.md").read_text()
    m = re.search(r"```python\n(# zstripe/_b200\.py\n.*?)```", text, re.S)
    assert m, "INTEGRATION.md lost its ctypes stub"
    os.environ["ZSTRIPE_B200_LIB"] = str(_lib.LIB_PATH)
    ns: dict = {}
    exec(compile(m.group(1), "INTEGRATION.md:_b200.py", "exec"), ns)  # noqa: S102
    return ns


def test_stub_binds_and_sizes_workspace():
    ns = _stub()
    assert ns["attn_ws_bytes"](196, 80) == (196 + 196) * 32 * 2
    assert ns["attn_ws_bytes"](4096, 64) == 4096 * 128 * 2
    with pytest.raises(ValueError, match="workspace"):
        fake = 0x1000
        ns["ashape_attention_dev"](fake, fake, fake, 196, 64, fake, fake, 14, fake, fake, 32, 32, 2, 0.125, fake,
                                   None, 0)


@pytest.mark.gpu
@pytest.mark.parametrize("S,w,tile,d", [(196, 14, 32, 64), (4096, 64, 128, 80)])
def test_stub_matches_api_on_device(S, w, tile, d):
    import torch

    from oracle import zs_oracle as O
    from paper_2605_17633_b200 import api
    from paper_2605_17633_b200.config import AShapeConfig

    ns = _stub()
    rng = O.SplitMix(11)
    q, k, v = (rng.normal((S, d)) for _ in range(3))
    bh, bw = rng.normal((S, w), 0.5), rng.normal((S, w), 0.5)
    sig = np.random.default_rng(0).permutation(S)
    cfg = AShapeConfig(b_row=tile, b_col=tile, r=0.4)
    ref = api.ashape_attention(q, k, v, api.BiasTables(bh, bw), sig, sig, cfg)
    dev = torch.device("cuda")
    qt, kt, vt = (torch.as_tensor(a).to(dev).bfloat16().contiguous() for a in (q, k, v))
    bht, bwt = (torch.as_tensor(a).to(dev).contiguous() for a in (bh, bw))
    sp = torch.as_tensor(sig).to(dev).int()
    out = torch.empty((S, d), device=dev, dtype=torch.bfloat16)
    n = ns["attn_ws_bytes"](S, d)
    ws = torch.empty(n, device=dev, dtype=torch.uint8)
    prefix = math.floor(0.4 * -(-S // tile))
    ns["ashape_attention_dev"](qt.data_ptr(), kt.data_ptr(), vt.data_ptr(), S, d, bht.data_ptr(), bwt.data_ptr(), w,
                               sp.data_ptr(), sp.data_ptr(), tile, tile, prefix, 1.0 / math.sqrt(d), out.data_ptr(),
                               ws.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(out.float().cpu().numpy(), ref)
