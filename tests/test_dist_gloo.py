"""Multi-process (world_size 2, gloo, CPU) coverage of the image-sharded batch path.

The hot path has no collective: each rank processes its contiguous shard of
images and one all_gather assembles the embeddings.  Here the per-image work
is the oracle's ordering (a per-image function), so the test checks that
sharded + gathered results equal the single-process results exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _per_image(batch: torch.Tensor) -> torch.Tensor:
    from oracle import zs_oracle as O

    out = [torch.from_numpy(O.orderings(img.numpy(), 6)["global"].astype(np.int64)) for img in batch]
    return torch.stack(out) if out else torch.zeros((0, batch.shape[1] * batch.shape[2]), dtype=torch.int64)


def _worker(rank, world, port, n_images, q):
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import zs_oracle as O
    from paper_2605_17633_b200.parallel import run_sharded

    batch = torch.from_numpy(O.SplitMix(5).normal((n_images, 12, 12, 8)))
    got = run_sharded(_per_image, batch)
    q.put((rank, got.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_images", [4, 5])
def test_sharded_batch_gathers_single_process_result(n_images):
    from oracle import zs_oracle as O

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_images, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    batch = torch.from_numpy(O.SplitMix(5).normal((n_images, 12, 12, 8)))
    ref = _per_image(batch).numpy()
    for r in range(world):
        assert np.array_equal(res[r], ref)


def _bench_line(*args, timeout=300):
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(root / "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("world,batch", [(2, 64), (3, 10)])
def test_bench_gpus_n_forms_world_and_gathers(world, batch):
    """`bench.py --gpus N` without WORLD_SIZE re-launches itself as N ranks (torch.distributed.run);
    the dry run's JSON line reports the world it formed, and the post-run all_gather puts every
    rank's shard back in its slot (checked bit for bit on every rank)."""
    line = _bench_line("--gpus", str(world), "--dry-run", "--steps", "2", "--warmup", "1", "--batch", str(batch))
    assert line["n_gpus"] == world
    assert line["dry_run"] is True
    assert line["gather"]["slot_check"] is True
    assert line["gather"]["bytes_gathered_per_rank"] == batch * 4 * 4 * 3 * 4  # [4, 4, 3] fp32 stand-in per image
    assert line["config"]["per_rank_batch"] == -(-batch // world)
