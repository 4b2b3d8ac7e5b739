"""Multi-GPU plumbing for batches of independent signals (C4).

The path shards naturally by signal: one process per GPU
(torchrun), each transforming its own signals; torch.distributed carries only
the start barrier and the max-over-ranks timing reduction -- nothing on the
data path.  Works with NCCL on GPUs and gloo on CPU (tests).
"""
from __future__ import annotations

import os

from .workloads import signal_seed


def rank_world():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(total: int, rank: int, world: int):
    """Contiguous [lo, hi) share of `total` signals for strong scaling."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def rank_seeds(base: int, per_rank: int, rank: int, world: int, scaling: str = "weak"):
    """Per-signal seeds of this rank.  weak: every rank transforms its own
    `per_rank` signals (global batch per_rank*world); strong: the global
    batch `per_rank` is split contiguously."""
    if scaling == "weak":
        return [signal_seed(base, rank * per_rank + i) for i in range(per_rank)]
    lo, hi = shard_range(per_rank, rank, world)
    return [signal_seed(base, i) for i in range(lo, hi)]


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (times are reported as the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
