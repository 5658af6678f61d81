"""bench.py — SAM ViT-H SparseSAM encoder throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one forward pass of this rank's shard of a 64-image batch of
synthetic 1024x1024 images through the full SAM ViT-H image encoder (patch
embed -> 32 SparseSAM blocks at density 0.4 -> neck), random-init weights of
that architecture.

Multi-GPU (BASELINE config 4, north-star (5)): N ranks, one process per GPU,
split the 64 images into contiguous shards (strong scaling; no collective on
the hot path).  ``--gpus N`` with N > 1 and no ``WORLD_SIZE`` in the
environment re-launches this script under ``torch.distributed.run`` with N
ranks (the driver's own torchrun launch is used as is); the script asserts
WORLD_SIZE == N.  After the timed region the embeddings are all-gathered over
NCCL (``parallel.gather_shards``) — the only collective — timed separately
(max over ranks) and checked: every rank's slot of the gathered batch must
equal its own shard bit for bit.  NCCL's INIT log is left on (stderr).

Reported (rank 0, one JSON line):
  value      whole-job images/s: 64 images / max-over-ranks device time per
             step (CUDA events, barrier + synchronize on both sides, K steps);
  e2e        the same through the public module with pinned-host images in
             and embeddings out (H2D + D2H inside the timed region);
  kernels    per-kernel CUDA-event breakdown.  For per-GPU batches >= 32 the
             events are recorded on the launching stream INSIDE the timed
             steps (the host runs far ahead of the GPU there, so the events
             cost no device time); for smaller batches from K separate
             traced steps after the timed region (per-launch event records
             would otherwise add host time to a launch-bound step);
  roofline   the dominant kernel family (tcgen05 GEMM) from those events;
  dense_*    the dense library encoder (cuBLAS + best SDPA backend) and this
             engine at mode="dense" (r = keep = 1) on the same GPU, with the
             FLOP-normalised ratio;
  cpu_baseline  the oracle port on the host cores (see --impl reference);
  clocks     nvidia-smi SM clocks / throttle reasons sampled during the timed region.

--impl reference times the reference algorithm's CPU implementation (the
oracle port in oracle/, pinned bit-exactly to the reference in tests/) on the
host cores: each step = one image's orderings + patch embed + neck + one
local block + one global block, all timed; the per-image time is extrapolated
to the model's block counts (labelled in the line).

--dry-run (CPU, gloo) exercises the multi-rank plumbing (re-launch, shards,
barrier/max timing, gather + check, JSON line) without CUDA; its "forward" is
a labelled CPU stand-in, not the product.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SAM ViT-H encoder images/s at density 0.4 vs dense; kernel % of BF16 peak"
UNIT = "images/s"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="vit_h")
    ap.add_argument("--density", type=float, default=0.4)
    ap.add_argument("--batch", type=int, default=64, help="global batch (images), split across ranks")
    ap.add_argument("--no-dense", action="store_true", help="skip the dense baseline legs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-gather", action="store_true", help="skip the post-run NCCL gather of the embeddings")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no side legs)")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU/gloo plumbing check of the multi-rank path with a stand-in forward (no CUDA)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="run each step's forward as one CUDA-graph replay (encoder.GraphedImageEncoder): "
                         "removes the per-kernel Python launches that bound small per-GPU batches; auto = on "
                         "when the per-GPU batch is <= 16 (the default 64 is GPU-bound either way)")
    ap.add_argument("--rel-pos", default="static", choices=["static", "sam"],
                    help="static: the reference's BiasTables (the headline config); sam: SAM's q-dependent "
                         "decomposed rel-pos (rel_pos_h / rel_pos_w tables, bias computed per query)")
    return ap.parse_args(argv)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(n: int) -> int:
    """Re-run this script under torch.distributed.run with n ranks on this node (127.0.0.1)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


# --------------------------------------------------------------------------- CPU (oracle) legs
class CpuSample:
    """One image's reference-algorithm work on the host cores (oracle port, BLAS matmul).

    Weights (one local block, one global block, the SAM frame) are drawn once; ``step()`` times
    orderings + patch embed + neck + one local block + one global block of one synthetic image and
    returns the seconds per image extrapolated to the model's 28 local + 4 global blocks (ViT-H)."""

    def __init__(self, model: str, density: float):
        import numpy as np

        from oracle import zs_oracle as O
        from paper_2605_17633_b200.config import SAM_NECK, SAM_PATCH, sam_config

        self.O, self.np = O, np
        cfg = sam_config(model, density)
        self.model, self.density, self.d = model, density, cfg.d
        self.n_loc = sum(k == "local" for k in cfg.layout)
        self.n_glob = len(cfg.layout) - self.n_loc
        rng = O.SplitMix(7)
        self.img = rng.normal((3, 1024, 1024)).astype(np.float32)
        d = cfg.d
        k_pe = 3 * SAM_PATCH * SAM_PATCH
        self.frame = dict(pe_w=rng.normal((d, k_pe), std=1 / math.sqrt(k_pe)), pe_b=np.zeros(d, np.float32),
                          pos=rng.normal((4096, d), std=0.02))
        self.neck = (rng.normal((SAM_NECK, d), std=1 / math.sqrt(d)), np.ones(SAM_NECK, np.float32),
                     np.zeros(SAM_NECK, np.float32), rng.normal((SAM_NECK, 9 * SAM_NECK), std=1 / 48.0),
                     np.ones(SAM_NECK, np.float32), np.zeros(SAM_NECK, np.float32))
        self.blocks = {}
        for kind in ("local", "global"):
            oc = O.EncCfg(d=d, heads=cfg.heads, layout=(kind,), r=(density,), keep=(density,))
            self.blocks[kind] = (oc, O.init_weights(oc))
        self.cores = os.cpu_count() or 1

    def step(self) -> tuple[float, float, str]:
        """-> (seconds per image extrapolated, wall seconds of this sample, description)."""
        O = self.O
        w0 = time.perf_counter()
        t0 = time.perf_counter()
        x = O.sam_patch_embed(self.img, **self.frame)
        orders = O.orderings(x, 14)
        t_front = time.perf_counter() - t0
        t = {}
        for kind, (oc, w) in self.blocks.items():
            t0 = time.perf_counter()
            O.encoder_forward(x, w, oc, orders=orders)
            t[kind] = time.perf_counter() - t0
        t0 = time.perf_counter()
        O.sam_neck(x, *self.neck)
        t_neck = time.perf_counter() - t0
        wall = time.perf_counter() - w0
        per_image = t_front + t_neck + self.n_loc * t["local"] + self.n_glob * t["global"]
        desc = (f"1 image SAM {self.model} d={self.density}: patch embed + orderings {t_front:.2f}s, neck "
                f"{t_neck:.2f}s, 1 local block {t['local']:.2f}s, 1 global block {t['global']:.2f}s, all timed; "
                f"per image = front + neck + {self.n_loc} x local + {self.n_glob} x global (extrapolated)")
        return per_image, wall, desc


def run_reference(args):
    world, rank, _ = dist_env()
    if world > 1 and rank != 0:
        return 0
    s = CpuSample(args.model, args.density)
    warm = max(1, args.warmup)
    per, walls, desc = [], [], ""
    for i in range(warm + args.steps):
        p, w, desc = s.step()
        if i >= warm:
            per.append(p)
            walls.append(w)
    sec_img = sum(per) / len(per)
    v = 1.0 / sec_img
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": len(per),
        "warmup": warm, "ms_per_step": 1e3 * sum(walls) / len(walls), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"full SAM {args.model} image encoder (patch embed, blocks, neck), density "
                               f"{args.density}, 1024x1024 synthetic image, random-init weights",
                   "model": f"sam_{args.model}", "global_batch": args.batch,
                   "parallelism": f"host cores (numpy BLAS, {s.cores} threads)",
                   "step": "one bounded per-image sample (see cpu_baseline.sample); ms_per_step is its wall time",
                   "extrapolated": True, "seconds_per_image": sec_img},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": s.cores, "kind": "port", "sample": desc},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region.

    In-process NVML (nvidia-ml-py) from a background thread every 5 ms, so even a timed region of
    a few milliseconds (ViT-B, one image) gets samples; falls back to `nvidia-smi -lms 100`."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, idx: int):
        self.idx = idx
        self.rows = []  # (sm_mhz, reason bitmask)
        self.max_mhz = None
        self.nvml = None
        self.proc = None
        self.path = None

    def __enter__(self):
        import threading

        try:
            import pynvml as N

            N.nvmlInit()
            h = self._nvml_handle(N)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            self.nvml, self._h = N, h
            self._stop = threading.Event()

            def run():
                while True:
                    try:
                        self.rows.append((float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)),
                                          int(N.nvmlDeviceGetCurrentClocksEventReasons(h))))
                    except Exception:  # noqa: BLE001
                        pass
                    if self._stop.wait(0.005):
                        return

            self._thr = threading.Thread(target=run, daemon=True)
            self._thr.start()
            return self
        except Exception:  # noqa: BLE001
            self.nvml = None
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.path = tempfile.mktemp(suffix=".csv")
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _nvml_handle(self, N):
        """NVML handle of CUDA device `idx` (matched by PCI location: CUDA_VISIBLE_DEVICES may
        renumber devices, NVML indices never are)."""
        try:
            import torch

            pr = torch.cuda.get_device_properties(self.idx)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return N.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:  # noqa: BLE001
            return N.nvmlDeviceGetHandleByIndex(self.idx)

    def __exit__(self, *exc):
        if self.nvml is not None:
            self._stop.set()
            self._thr.join(timeout=2)
            try:  # one last sample: the region ended just now
                self.rows.append((float(self.nvml.nvmlDeviceGetClockInfo(self._h, self.nvml.NVML_CLOCK_SM)),
                                  int(self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self._h))))
            except Exception:  # noqa: BLE001
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            self.f.close()

    def summary(self) -> dict:
        if self.nvml is not None:
            if not self.rows:
                return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "source": "nvml"}
            sm = sorted(r[0] for r in self.rows)
            reasons = sorted({n for _, m in self.rows for n, bit in self.REASONS.items() if m & bit})
            return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons,
                    "samples": len(self.rows), "source": "nvml, 5 ms"}
        try:
            rows = [r.split(", ") for r in Path(self.path).read_text().strip().splitlines() if r.strip()]
        except Exception:  # noqa: BLE001
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[1]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.strip() == "Active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][2]), "reasons": reasons, "samples": len(rows),
                "source": "nvidia-smi, 100 ms"}


# --------------------------------------------------------------------------- multi-rank helpers
class Ranks:
    """Barrier / max-over-ranks / gather for one process per device (NCCL) or CPU (gloo)."""

    def __init__(self, world: int, rank: int, dev, backend: str):
        import torch
        import torch.distributed as dist

        self.world, self.rank, self.dev, self.dist, self.torch = world, rank, dev, dist, torch
        self.cuda = dev.type == "cuda"
        if world > 1:
            kw = dict(device_id=dev) if self.cuda else {}
            dist.init_process_group(backend, **kw)
            if dist.get_world_size() != world:
                raise RuntimeError(f"process group has {dist.get_world_size()} ranks, expected {world}")

    def barrier(self):
        if self.world > 1:
            if self.cuda:
                self.dist.barrier(device_ids=[self.dev.index])
            else:
                self.dist.barrier()

    def max(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], device=self.dev, dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def all_true(self, ok: bool) -> bool:
        if self.world == 1:
            return ok
        t = self.torch.tensor([0 if ok else 1], device=self.dev, dtype=self.torch.int32)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return int(t.item()) == 0

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def timed_gather(R: Ranks, out, n_items: int, a: int, b: int, timer) -> dict:
    """All-gather the per-rank embedding shards (parallel.gather_shards, the path's only
    collective), time it (max over ranks) and check each rank's slot bit for bit."""
    from paper_2605_17633_b200.parallel import gather_shards

    gather_shards(out, n_items)  # warm the communicator
    R.barrier()
    t = timer()
    full = gather_shards(out, n_items)
    ms = R.max(t())
    ok = R.all_true(bool(full.shape[0] == n_items) and bool(R.torch.equal(full[a:b], out)))
    nbytes = full.numel() * full.element_size()
    return {"collective": "all_gather (NCCL)" if R.cuda else "all_gather (gloo)", "ms": ms,
            "bytes_gathered_per_rank": nbytes, "gbs_per_rank": nbytes / (ms * 1e-3) / 1e9 if ms else None,
            "slot_check": ok, "in_timed_region": False}


# --------------------------------------------------------------------------- dry run (CPU plumbing)
def run_dry(args):
    import torch

    from paper_2605_17633_b200.parallel import shard_bounds

    world, rank, _ = dist_env()
    if world != args.gpus:
        raise RuntimeError(f"WORLD_SIZE={world} but --gpus {args.gpus}")
    R = Ranks(world, rank, torch.device("cpu"), "gloo")
    a, b = shard_bounds(args.batch, world, rank)
    g = torch.Generator().manual_seed(100 + rank)
    imgs = torch.randn((b - a, 3, 64, 64), generator=g)

    def stand_in(x):  # NOT the product: a labelled CPU stand-in for the encoder forward
        return x.unfold(2, 16, 16).unfold(3, 16, 16).mean(dim=(-1, -2)).permute(0, 2, 3, 1).contiguous()

    def timer():
        t0 = time.perf_counter()
        return lambda: 1e3 * (time.perf_counter() - t0)

    for _ in range(args.warmup):
        out = stand_in(imgs)
    R.barrier()
    t = timer()
    for _ in range(args.steps):
        out = stand_in(imgs)
    R.barrier()
    ms = R.max(t() / args.steps)
    gather = timed_gather(R, out, args.batch, a, b, timer)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": args.batch / (ms / 1e3), "unit": UNIT, "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                          "scaling": "strong", "dry_run": True,
                          "data": "synthetic; forward = CPU stand-in (patch means), not the product",
                          "config": {"global_batch": args.batch, "per_rank_batch": b - a,
                                     "parallelism": f"image-sharded dp{world} (gloo)"},
                          "gather": gather}), flush=True)
    R.close()
    return 0


# --------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if args.impl == "reference":
            return run_reference(args)  # rank 0's work only: no need for the other ranks
        return relaunch(args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    if args.dry_run:
        return run_dry(args)

    import torch

    from paper_2605_17633_b200.config import sam_config
    from paper_2605_17633_b200.encoder import SparseSAMImageEncoder
    from paper_2605_17633_b200.parallel import shard_bounds
    from paper_2605_17633_b200.trace import NULL, Tracer
    from paper_2605_17633_b200.weights import random_frame, random_params

    world, rank, local = dist_env()
    if world != args.gpus:
        raise RuntimeError(f"WORLD_SIZE={world} but --gpus {args.gpus}: launch one rank per GPU")
    if not torch.cuda.is_available():
        raise RuntimeError("bench.py needs a CUDA device (use --dry-run for the CPU plumbing check)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    R = Ranks(world, rank, dev, "nccl")
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

    def timer(stream=None):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)

        def stop():
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1)
        return stop

    from paper_2605_17633_b200 import _lib

    with torch.no_grad():
        for _ in range(args.warmup):
            enc(imgs)
        torch.cuda.synchronize()

        use_graph = args.graph == "on" or (args.graph == "auto" and nloc <= 16)
        trace_in_region = nloc >= 32 and not use_graph
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

        tracer = Tracer()
        if trace_in_region:
            enc.core.tracer = tracer
        with ClockSampler(local) as clk:
            R.barrier()
            t = timer()
            for _ in range(args.steps):
                step(imgs)
            ms = t() / args.steps
            R.barrier()
        ms = R.max(ms)
        clocks = clk.summary()
        if not trace_in_region:
            enc.core.tracer = tracer
            for _ in range(args.steps):
                enc(imgs)
        enc.core.tracer = NULL
        kern = tracer.summary()
        out_last = enc(imgs).clone()

        # ---- the path's one collective: NCCL all_gather of the embeddings (after the timed region)
        gather = None
        if world > 1 and not args.no_gather:
            gather = timed_gather(R, out_last, args.batch, a, b, timer)
        del out_last

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
            R.barrier()
            t = timer(comp)
            with torch.cuda.stream(copy):
                dimg[0].copy_(host_in[0], non_blocking=True)
                ev_in[0].record(copy)
            for s in range(args.steps):
                bb = s & 1
                if s + 1 < args.steps:  # next step's images while this step computes
                    with torch.cuda.stream(copy):
                        if s >= 1:
                            copy.wait_event(ev_done[bb ^ 1])  # its buffer's previous forward finished
                        dimg[bb ^ 1].copy_(host_in[bb ^ 1], non_blocking=True)
                        ev_in[bb ^ 1].record(copy)
                comp.wait_event(ev_in[bb])
                if s >= 2:
                    comp.wait_event(ev_out[bb])  # dout[bb] copied out two steps ago
                if graphs:
                    graphs[bb].graph.replay()  # forward of dimg[bb] into dout[bb]
                else:
                    enc(dimg[bb], out=dout[bb])
                ev_done[bb].record(comp)
                with torch.cuda.stream(copy):
                    copy.wait_event(ev_done[bb])
                    host_out[bb].copy_(dout[bb], non_blocking=True)
                    ev_out[bb].record(copy)
            comp.wait_stream(copy)
            ms_e2e = t() / args.steps
            R.barrier()
            ms_e2e = R.max(ms_e2e)
            e2e = {"value": args.batch / (ms_e2e / 1e3), "unit": UNIT,
                   "h2d_bytes_per_step": host_in[0].numel() * 4, "d2h_bytes_per_step": host_out[0].numel() * 4,
                   "ms_per_step": ms_e2e, "copies": "side stream, double-buffered (overlap compute)"}
            del host_in, host_out, dimg, dout

        # ---- dense comparators on the same GPU (N = 1 only)
        dense = dense_same = None
        if world == 1 and not args.no_dense and not args.profile:
            dense, dense_same = dense_legs(args, cfg, params, frame, enc, imgs, timer, ms, kern)

    value = args.batch / (ms / 1e3)
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:  # noqa: BLE001
        pass
    roofline, kernels = kernel_report(kern, args.steps, peaks)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.profile:
        s = CpuSample(args.model, args.density)
        per_image, _, desc = s.step()
        cpu = {"value": 1.0 / per_image, "unit": UNIT, "cores": s.cores, "kind": "port", "sample": desc}

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
                       "kernel_timing": "events inside the timed steps" if trace_in_region
                       else "events over separate traced steps",
                       "l2": ("inputs larger than L2 (batch of images > 126 MB); no explicit flush"
                              if nloc * 3 * 1024 * 1024 * 4 > 126e6 else
                              f"input images ({nloc * 12.6:.0f} MB) fit L2 and are not flushed; every block "
                              f"streams {nloc * 4096 * cfg.d * 4 / 1e6:.0f} MB of fp32 residual rows plus "
                              f"{cfg.d * cfg.d * 24 / 1e6:.0f} MB of weights")},
            "e2e": e2e, "dense_baseline": dense, "dense_same_engine": dense_same, "roofline": roofline,
            "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": launches, "gather": gather, "kernels": kernels,
        }
        print(json.dumps(line), flush=True)
    R.close()
    return 0


def dense_legs(args, cfg, params, frame, enc, imgs, timer, ms_sparse, kern_sparse):
    """Dense library encoder (cuBLAS + the fastest SDPA backend that takes the bias) and this
    engine at mode="dense" (r = keep = 1, the reference's dense twin, encoder.py:338-339)."""
    import torch
    from torch.nn.attention import SDPBackend, sdpa_kernel

    from paper_2605_17633_b200.dense import DenseSAMEncoder
    from paper_2605_17633_b200.trace import NULL, Tracer

    nd = max(2, args.steps // 2)
    den = DenseSAMEncoder(cfg, params, frame)
    backends = {}
    for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
        try:
            with sdpa_kernel([be]):
                for _ in range(2):
                    den(imgs)
                t = timer()
                for _ in range(nd):
                    den(imgs)
                backends[name] = t() / nd
        except RuntimeError as e:  # backend rejects this mask / shape
            backends[name] = f"unavailable: {str(e).splitlines()[0][:120]}"
            torch.cuda.synchronize()
    timed = {k: v for k, v in backends.items() if isinstance(v, float)}
    best = min(timed, key=timed.get)
    ms_d = timed[best]
    B = args.batch
    sparse_tf = sum(v["flops"] for v in kern_sparse.values()) / max(args.steps, 1) / B / 1e12
    dense = {"value": B / (ms_d / 1e3), "unit": UNIT, "ms_per_step": ms_d, "sdpa_backend": best,
             "sdpa_ms_per_step": backends,
             "what": "same weights, torch bf16: cuBLAS GEMMs + SDPA with materialised rel-pos bias, SAM windowing",
             "speedup": ms_d / ms_sparse}

    for _ in range(2):
        enc(imgs, mode="dense")
    t = timer()
    for _ in range(nd):
        enc(imgs, mode="dense")
    ms_s = t() / nd
    tr = Tracer()
    enc.core.tracer = tr
    enc(imgs, mode="dense")
    enc.core.tracer = NULL
    dense_tf = sum(v["flops"] for v in tr.summary().values()) / B / 1e12
    flop_ratio = dense_tf / sparse_tf if sparse_tf else None
    same = {"value": B / (ms_s / 1e3), "unit": UNIT, "ms_per_step": ms_s,
            "what": "this engine, mode='dense' (r = keep = 1 through the same kernels)",
            "tflop_per_image_blocks": dense_tf, "sparse_tflop_per_image_blocks": sparse_tf,
            "flop_ratio": flop_ratio, "speedup": ms_s / ms_sparse,
            "speedup_per_flop": (ms_s / ms_sparse) / flop_ratio if flop_ratio else None}
    return dense, same


def kernel_report(kern: dict, steps: int, peaks: dict):
    """Roofline of the dominant kernel family + per-kernel table from the CUDA-event spans."""
    peak_tf = peaks.get("bf16_tflops_sustained") or 1409.4
    peak_src = "measured (sustained, MEASURED_PEAKS.json)" if peaks.get("bf16_tflops_sustained") else "fallback"
    hbm = peaks.get("hbm_gbs") or 6547.5
    gk = {"ms": 0.0, "launches": 0, "flops": 0.0}
    for name, v in kern.items():
        if name.startswith("gemm"):
            for key in gk:
                gk[key] += v[key]
    achieved = (gk["flops"] / gk["launches"]) / (gk["ms"] / gk["launches"] * 1e-3) / 1e12 if gk["launches"] else 0.0
    traffic, by_kernel = None, None
    try:
        prof = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text())
        traffic = prof.get("gemm_dram_bytes_per_launch")
        by_kernel = prof.get("dram_bytes_per_launch_by_kernel")
    except Exception:  # noqa: BLE001
        pass
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": achieved / peak_tf if peak_tf else None, "traffic": traffic,
                "traffic_source": "ncu --set full of one bench-config forward (tools/prof_step.py; profiles/ncu_summary.json)",
                "traffic_by_kernel": by_kernel, "kernel": "zs_gemm2_kernel (cta_group::2)",
                "launches_per_step": gk["launches"] // max(steps, 1), "peak_source": peak_src}
    total = sum(v["ms"] for v in kern.values()) / max(steps, 1)
    kernels = {}
    for name, v in sorted(kern.items(), key=lambda kv: -kv[1]["ms"]):
        d = {"ms_per_step": v["ms"] / steps, "launches_per_step": v["launches"] // max(steps, 1),
             "share": v["ms"] / steps / total if total else None}
        if v["flops"]:
            d["tflops"] = v["flops"] / (v["ms"] * 1e-3) / 1e12
            d["frac_bf16_peak"] = d["tflops"] / peak_tf
        if v["bytes"]:
            d["gbs"] = v["bytes"] / (v["ms"] * 1e-3) / 1e9
            d["frac_hbm_peak"] = d["gbs"] / hbm
        kernels[name] = d
    return roofline, kernels


if __name__ == "__main__":
    sys.exit(main())
