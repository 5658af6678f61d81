"""Small-batch latency of the image encoder: eager (one Python launch per kernel) vs one CUDA graph.

    python tools/graph_latency.py [model] [B...]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2605_17633_b200 as Z  # noqa: E402
from paper_2605_17633_b200.encoder import GraphedImageEncoder, SparseSAMImageEncoder  # noqa: E402
from paper_2605_17633_b200.weights import random_frame, random_params  # noqa: E402

model = sys.argv[1] if len(sys.argv) > 1 else "vit_h"
Bs = [int(b) for b in sys.argv[2:]] or [1, 4]
cfg = Z.sam_config(model, 0.4)
enc = SparseSAMImageEncoder(cfg, random_params(cfg, "cuda", seed=0), random_frame(cfg, "cuda", seed=1))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for B in Bs:
    img = torch.randn(B, 3, 1024, 1024, device="cuda")
    t_eager = timed(lambda: enc(img))
    gr = GraphedImageEncoder(enc, B)
    t_graph = timed(lambda: gr(img))
    print(f"{model} B={B}: eager {t_eager:.2f} ms ({B / t_eager * 1e3:.1f} img/s)  graph {t_graph:.2f} ms "
          f"({B / t_graph * 1e3:.1f} img/s)", flush=True)
