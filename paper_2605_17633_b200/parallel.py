"""Image-sharded multi-GPU batch (north-star (5)).

Images are independent through the whole encoder (orderings, attention, MLP
and every layout are per image, encoder.py:310-385), so a batch is split into
contiguous per-rank shards with NO collective on the hot path.  The only
communication is the final gather of the per-image embeddings, one
``all_gather`` over NCCL (NVLink / NVSwitch) on B200 boxes, gloo in CPU tests.
One process per GPU (torchrun); ranks with a short shard pad the gather.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split: the first n % world ranks get one extra item."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_counts(n_items: int, world: int) -> list[int]:
    return [b - a for a, b in (shard_bounds(n_items, world, r) for r in range(world))]


def gather_shards(local: torch.Tensor, n_items: int, group=None) -> torch.Tensor:
    """All-gather per-rank shards (leading dim = images) into the full batch on every rank."""
    world = dist.get_world_size(group)
    counts = shard_counts(n_items, world)
    cap = max(counts)
    if local.shape[0] != counts[dist.get_rank(group)]:
        raise ValueError(f"local shard has {local.shape[0]} items, expected {counts[dist.get_rank(group)]}")
    padded = local.new_zeros((cap,) + tuple(local.shape[1:]))
    padded[: local.shape[0]] = local
    bufs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded, group=group)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)


def run_sharded(fn, batch: torch.Tensor, group=None, gather: bool = True) -> torch.Tensor:
    """Apply ``fn`` to this rank's contiguous shard of ``batch`` and (optionally) gather the results."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    a, b = shard_bounds(batch.shape[0], world, rank)
    out = fn(batch[a:b])
    if gather and world > 1:
        return gather_shards(out, batch.shape[0], group)
    return out
