"""One bench step (SAM image encoder forward at the bench config) inside a cudaProfilerStart/Stop
region, after two warm-up forwards: run under `ncu --profile-from-start off` to capture exactly
the bench's own launches (launch list or --set full of selected kernels).

    python tools/prof_step.py [--model vit_h] [--batch 64] [--density 0.4]
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_17633_b200.config import sam_config  # noqa: E402
from paper_2605_17633_b200.encoder import SparseSAMImageEncoder  # noqa: E402
from paper_2605_17633_b200.weights import random_frame, random_params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="vit_h")
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--density", type=float, default=0.4)
a = ap.parse_args()
dev = torch.device("cuda", 0)
cfg = sam_config(a.model, a.density)
enc = SparseSAMImageEncoder(cfg, random_params(cfg, dev, seed=0), random_frame(cfg, dev, seed=1), dev)
imgs = torch.randn((a.batch, 3, 1024, 1024), device=dev, generator=torch.Generator(device=dev).manual_seed(100))
with torch.no_grad():
    for _ in range(2):
        enc(imgs)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    enc(imgs)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
print("profiled one forward:", a.model, a.batch, a.density)
