"""bench.py — SAM ViT-H SparseSAM encoder throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one forward pass of this rank's shard of a 64-image batch of
synthetic 1024x1024 images through the full SAM ViT-H image encoder (patch
embed -> 32 SparseSAM blocks at density 0.4 -> neck), random-init weights of
that architecture.  N>1 ranks (torchrun, NCCL) split the 64 images
(strong scaling, no collective on the hot path; the all_gather of the
embeddings runs after the timed region, as in parallel.run_sharded).

Reported (rank 0, one JSON line): whole-job images/s from CUDA events over
exactly K steps bracketed by barrier + synchronize, max over ranks; the
end-to-end rate through the public API with pinned-host inputs (H2D + D2H in
the timed region); the dominant kernel's roofline from per-launch CUDA events
recorded on the launching stream inside the timed region; the dense
cuBLAS/cuDNN encoder on the same GPU; the oracle port on the host cores;
SM clocks sampled during the timed region.

--impl reference times the reference algorithm's CPU implementation (the
oracle port in oracle/, pinned to the reference in tests/) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SAM ViT-H encoder images/s at density 0.4 vs dense; kernel % of BF16 peak"
UNIT = "images/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="vit_h")
    ap.add_argument("--density", type=float, default=0.4)
    ap.add_argument("--batch", type=int, default=64, help="global batch (images), split across ranks")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense cuBLAS/cuDNN baseline leg")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no side legs)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="run each step's forward as one CUDA-graph replay (encoder.GraphedImageEncoder): "
                         "removes the per-kernel Python launches that bound small per-GPU batches; auto = on "
                         "when the per-GPU batch is <= 16 (the default 64 is GPU-bound either way)")
    ap.add_argument("--rel-pos", default="static", choices=["static", "sam"],
                    help="static: the reference's BiasTables (the headline config); sam: SAM's q-dependent "
                         "decomposed rel-pos (rel_pos_h / rel_pos_w tables, bias computed per query)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------------------- CPU (oracle) legs
def cpu_sample_image_seconds(model: str, density: float, reps: int = 1) -> tuple[float, str, int]:
    """Seconds per image of the oracle port (BLAS matmul, all host cores) extrapolated from one
    local block + one global block + the orderings of one image (SURVEY §8(d) plan)."""
    import numpy as np

    from oracle import zs_oracle as O
    from paper_2605_17633_b200.config import sam_config

    cfg = sam_config(model, density)
    n_loc = sum(k == "local" for k in cfg.layout)
    n_glob = len(cfg.layout) - n_loc
    x = O.SplitMix(1).normal((64, 64, cfg.d))
    t0 = time.perf_counter()
    orders = O.orderings(x, 14)
    t_ord = time.perf_counter() - t0
    res = {}
    for kind in ("local", "global"):
        oc = O.EncCfg(d=cfg.d, heads=cfg.heads, layout=(kind,), r=(density,), keep=(density,))
        w = O.init_weights(oc)
        best = math.inf
        for _ in range(reps):
            t0 = time.perf_counter()
            O.encoder_forward(x, w, oc, orders=orders)
            best = min(best, time.perf_counter() - t0)
        res[kind] = best
    per_image = t_ord + n_loc * res["local"] + n_glob * res["global"]
    sample = (f"1 image {model} d={density}: orderings {t_ord:.2f}s + {n_loc} x local block {res['local']:.2f}s + "
              f"{n_glob} x global block {res['global']:.2f}s (blocks timed, total extrapolated)")
    cores = os.cpu_count() or 1
    return per_image, sample, cores


def run_reference(args):
    world, rank, _ = dist_env()
    if world > 1 and rank != 0:
        return 0
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    for _ in range(args.warmup if args.warmup < 1 else 1):
        pass
    times = []
    sample = ""
    cores = os.cpu_count() or 1
    for i in range(max(1, args.warmup) + args.steps):
        per_image, sample, cores = cpu_sample_image_seconds(args.model, args.density)
        if i >= max(1, args.warmup):
            times.append(per_image)
        if i == 0 and args.steps + args.warmup > 3:
            # one step is ~10-20 s of CPU work; cap the run at a few minutes
            args.steps = min(args.steps, 4)
            args.warmup = 1
    v = 1.0 / (sum(times) / len(times))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": len(times),
        "warmup": max(1, args.warmup), "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"SAM {args.model} encoder, density {args.density}, 1024x1024 images",
                   "global_batch": args.batch, "parallelism": "host cores (BLAS threads)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, idx: int):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        self.idx = idx

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            self.f.close()

    def summary(self) -> dict:
        try:
            rows = [r.split(", ") for r in Path(self.path).read_text().strip().splitlines() if r.strip()]
        except Exception:  # noqa: BLE001
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[1]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.strip() == "Active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][2]), "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2605_17633_b200.config import sam_config
    from paper_2605_17633_b200.encoder import SparseSAMImageEncoder
    from paper_2605_17633_b200.parallel import shard_bounds
    from paper_2605_17633_b200.trace import Tracer
    from paper_2605_17633_b200.weights import random_frame, random_params

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.warmup < 3 and not args.profile:
        args.warmup = 3

    cfg = sam_config(args.model, args.density)
    params = random_params(cfg, dev, seed=0, rel_pos=args.rel_pos == "sam")
    frame = random_frame(cfg, dev, seed=1)
    enc = SparseSAMImageEncoder(cfg, params, frame, dev)
    a, b = shard_bounds(args.batch, world, rank)
    nloc = b - a
    g = torch.Generator(device=dev).manual_seed(100 + rank)
    imgs = torch.randn((nloc, 3, 1024, 1024), device=dev, generator=g)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with torch.no_grad():
        for _ in range(args.warmup):
            enc(imgs)
        torch.cuda.synchronize()

        from paper_2605_17633_b200 import _lib

        use_graph = args.graph == "on" or (args.graph == "auto" and nloc <= 16)
        step = enc
        graphs = None
        if use_graph:
            from paper_2605_17633_b200.encoder import GraphedImageEncoder

            # two captures over separate static buffers: the e2e loop double-buffers them
            graphs = [GraphedImageEncoder(enc, nloc) for _ in range(2)]
            step = graphs[0]
            for _ in range(2):
                step(imgs)
        launches0 = _lib.launch_count
        enc(imgs)  # one eager step: launches per step (a graph replay launches the same kernels)
        launches = _lib.launch_count - launches0
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            barrier()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(args.steps):
                step(imgs)
            e1.record()
            torch.cuda.synchronize()
            barrier()
        ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        clocks = clk.summary()
        # per-kernel breakdown from separate traced steps (the CUDA events of the spans add host
        # work per kernel, which would inflate the timed steps of small batches)
        tracer = Tracer()
        enc.core.tracer = tracer
        for _ in range(args.steps):
            enc(imgs)
        torch.cuda.synchronize()
        enc.core.tracer = __import__("paper_2605_17633_b200.trace", fromlist=["NULL"]).NULL
        kern = tracer.summary()

        # ---- end to end through the public API: pinned host in, embeddings out
        e2e = None
        if not args.no_e2e and not args.profile:
            # every step: H2D of its images from pinned host memory, the forward through the
            # public module, D2H of its embeddings.  Copies run on a side stream, double-buffered
            # on the device, so step i's transfers overlap steps i-1 / i+1's compute (each step's
            # copies are still inside the timed region, which ends after the last D2H).
            host_in = [imgs.cpu().pin_memory() for _ in range(2)]
            host_out = [torch.empty((nloc, 64, 64, 256), dtype=torch.float32).pin_memory() for _ in range(2)]
            if graphs:
                dimg = [gr.img for gr in graphs]
                dout = [gr.out for gr in graphs]
            else:
                dimg = [torch.empty_like(imgs) for _ in range(2)]
                dout = [torch.empty((nloc, 64, 64, 256), device=dev, dtype=torch.float32) for _ in range(2)]
            comp = torch.cuda.current_stream()
            copy = torch.cuda.Stream(device=dev)
            ev_in = [torch.cuda.Event() for _ in range(2)]
            ev_done = [torch.cuda.Event() for _ in range(2)]
            ev_out = [torch.cuda.Event() for _ in range(2)]
            barrier()
            torch.cuda.synchronize()
            e0.record(comp)
            with torch.cuda.stream(copy):
                dimg[0].copy_(host_in[0], non_blocking=True)
                ev_in[0].record(copy)
            for s in range(args.steps):
                b = s & 1
                if s + 1 < args.steps:  # next step's images while this step computes
                    with torch.cuda.stream(copy):
                        if s >= 1:
                            copy.wait_event(ev_done[b ^ 1])  # its buffer's previous forward finished
                        dimg[b ^ 1].copy_(host_in[b ^ 1], non_blocking=True)
                        ev_in[b ^ 1].record(copy)
                comp.wait_event(ev_in[b])
                if s >= 2:
                    comp.wait_event(ev_out[b])  # dout[b] copied out two steps ago
                if graphs:
                    graphs[b].graph.replay()  # forward of dimg[b] into dout[b]
                else:
                    enc(dimg[b], out=dout[b])
                ev_done[b].record(comp)
                with torch.cuda.stream(copy):
                    copy.wait_event(ev_done[b])
                    host_out[b].copy_(dout[b], non_blocking=True)
                    ev_out[b].record(copy)
            comp.wait_stream(copy)
            e1.record(comp)
            torch.cuda.synchronize()
            barrier()
            ms_e2e = max_over_ranks(e0.elapsed_time(e1) / args.steps)
            e2e = {"value": args.batch / (ms_e2e / 1e3), "unit": UNIT,
                   "h2d_bytes_per_step": host_in[0].numel() * 4, "d2h_bytes_per_step": host_out[0].numel() * 4,
                   "ms_per_step": ms_e2e, "copies": "side stream, double-buffered (overlap compute)"}

        # ---- dense cuBLAS/cuDNN encoder on the same GPU (rank 0, N=1 only)
        dense = None
        if world == 1 and not args.no_dense and not args.profile:
            from paper_2605_17633_b200.dense import DenseSAMEncoder

            den = DenseSAMEncoder(cfg, params, frame)
            for _ in range(2):
                den(imgs)
            torch.cuda.synchronize()
            e0.record()
            nd = max(2, args.steps // 2)
            for _ in range(nd):
                den(imgs)
            e1.record()
            torch.cuda.synchronize()
            ms_d = e0.elapsed_time(e1) / nd
            dense = {"value": args.batch / (ms_d / 1e3), "unit": UNIT, "ms_per_step": ms_d,
                     "what": "same weights, torch bf16: cuBLAS GEMMs + SDPA with materialised rel-pos bias",
                     "speedup": ms_d / ms}

    value = args.batch / (ms / 1e3)

    # ---- roofline of the dominant kernel (tcgen05 GEMM), per-launch CUDA events in the timed region
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:  # noqa: BLE001
        pass
    peak_tf = peaks.get("bf16_tflops_sustained") or 1409.4
    peak_src = "measured (sustained, MEASURED_PEAKS.json)" if peaks.get("bf16_tflops_sustained") else "fallback"
    # the tcgen05 GEMM kernel over all its launches in the timed region (QKV, proj, fc1, fc2)
    gk = {"ms": 0.0, "launches": 0, "flops": 0.0}
    for name, v in kern.items():
        if name.startswith("gemm"):
            for key in gk:
                gk[key] += v[key]
    achieved = (gk["flops"] / gk["launches"]) / (gk["ms"] / gk["launches"] * 1e-3) / 1e12 if gk["launches"] else 0.0
    traffic = None
    try:
        traffic = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text()).get("gemm_dram_bytes_per_launch")
    except Exception:  # noqa: BLE001
        pass
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": achieved / peak_tf if peak_tf else None, "traffic": traffic, "kernel": "zs_gemm2_kernel (cta_group::2)", "launches_per_step": gk["launches"] // max(args.steps, 1),
                "peak_source": peak_src}
    step_ms_total = sum(v["ms"] for v in kern.values()) / max(args.steps, 1)
    kernels = {}
    for name, v in sorted(kern.items(), key=lambda kv: -kv[1]["ms"]):
        d = {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] // max(args.steps, 1),
             "share": v["ms"] / args.steps / step_ms_total if step_ms_total else None}
        if v["flops"]:
            d["tflops"] = v["flops"] / (v["ms"] * 1e-3) / 1e12
            d["frac_bf16_peak"] = d["tflops"] / peak_tf
        if v["bytes"] and not v["flops"]:
            d["gbs"] = v["bytes"] / (v["ms"] * 1e-3) / 1e9
            d["frac_hbm_peak"] = d["gbs"] / (peaks.get("hbm_gbs") or 6547.5)
        kernels[name] = d

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        per_image, sample, cores = cpu_sample_image_seconds(args.model, args.density)
        cpu = {"value": 1.0 / per_image, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"full SAM {args.model} image encoder (patch embed, {len(cfg.layout)} blocks, neck), "
                                   f"density {args.density}, 1024x1024 synthetic images, random-init weights",
                       "model": f"sam_{args.model}", "global_batch": args.batch, "per_gpu_batch": nloc,
                       "seq_len": 4096, "parallelism": f"image-sharded dp{world}", "rel_pos": args.rel_pos,
                       "cuda_graph": bool(use_graph),
                       "l2": ("inputs larger than L2 (batch of images > 126 MB); no explicit flush"
                              if nloc * 3 * 1024 * 1024 * 4 > 126e6 else
                              f"input ({nloc * 12.6:.0f} MB) smaller than L2, not flushed: each step's own "
                              f"activation traffic ({len(cfg.layout)} blocks) is many times L2")},
            "e2e": e2e, "dense_baseline": dense, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": launches, "kernels": kernels,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
