"""Multi-GPU plumbing (host logic only).

The hot path runs on one GPU. Across GPUs there are two modes, neither with a collective on
the data path:

* replicas -- every rank runs the whole workload (weak scaling; bench.py's default);
* batch sharding -- independent units (C2's 32 masks, colour channels, images) are split
  into contiguous shards, one per rank; the only exchange is gathering the per-unit scalars
  (MSE, iteration counts) at the end.

Device time of a multi-rank run is the MAX over ranks (one all-reduce of a scalar), never
wall clock. Works with any torch.distributed backend (nccl on the GPU box, gloo in the CPU
tests).
"""
from __future__ import annotations

import numpy as np


def shard(n_items: int, rank: int, world: int) -> range:
    """Contiguous, balanced shard of [0, n_items) for `rank` (sizes differ by at most one)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    lo = n_items * rank // world
    hi = n_items * (rank + 1) // world
    return range(lo, hi)


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def max_over_ranks(value: float, device=None) -> float:
    """The job's time: max of a per-rank scalar (identity when not distributed)."""
    dist = _dist()
    if dist is None:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_scalars(local: np.ndarray, n_items: int, device=None) -> np.ndarray:
    """Per-unit scalars of every rank's shard, in global unit order (all ranks get them)."""
    local = np.asarray(local, dtype=np.float64)
    dist = _dist()
    if dist is None:
        if local.size != n_items:
            raise ValueError("not distributed: the local shard must hold every unit")
        return local.copy()
    import torch
    world = dist.get_world_size()
    width = max(len(shard(n_items, r, world)) for r in range(world))
    buf = torch.full((width,), float("nan"), dtype=torch.float64, device=device)
    buf[: local.size] = torch.as_tensor(local, dtype=torch.float64)
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    parts = [outs[r][: len(shard(n_items, r, world))].cpu().numpy() for r in range(world)]
    return np.concatenate(parts)
