"""Multi-GPU plumbing.

Batches of independent signals (C4) shard by signal: one process per GPU
(torchrun), each transforming its own signals; torch.distributed carries only
the start barrier and the max-over-ranks timing reduction -- nothing on the
data path.

One large signal (C5) shards by index range: rank r holds x[lo_r, hi_r)
(index_range), encodes PARTIAL bucket values of every round of every
iteration from its samples only (Plan.encode_values; bucketize is linear in
x), one all-reduce(sum) of the partial vectors (combine_partials) yields the
full vector, and the decode runs on it (Plan.decode_values) -- on every rank
or on rank 0 only.  The all-reduce adds the partials in a different order
than the single-GPU fold, a ~1e-16 relative difference.

Works with NCCL on GPUs and gloo on CPU (tests).
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


def index_range(n: int, rank: int, world: int):
    """Contiguous [lo, hi) sample range of one signal held by `rank`."""
    return shard_range(n, rank, world)


def combine_partials(y, group=None):
    """Sum the ranks' partial bucket vectors in place (one all-reduce).
    y: complex128 tensor (CUDA under NCCL, CPU under gloo)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return y
    if y.is_cuda and dist.get_backend(group) != "nccl":
        # host-side backends (gloo): reduce a host copy
        h = torch.view_as_real(y).cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        torch.view_as_real(y).copy_(h)
        return y
    dist.all_reduce(torch.view_as_real(y), op=dist.ReduceOp.SUM, group=group)
    return y


def sharded_sfft4(plan, x_local, x_lo: int, seeds, decode_on: str = "all", group=None,
                  assume_valid: bool = False):
    """One index-range-sharded transform step on this rank.

    x_local: CUDA tensor (batch, span) = x[:, x_lo:x_lo+span] of each signal.
    decode_on: "all" (every rank decodes the summed vector redundantly and
    returns the result) or "root" (rank 0 decodes; the others return None).
    Returns (f, c, count) CUDA tensors or None."""
    import torch.distributed as dist
    y = plan.encode_values(x_local, seeds, x_lo, assume_valid=assume_valid)
    combine_partials(y, group)
    rank = dist.get_rank(group) if dist.is_available() and dist.is_initialized() else 0
    if decode_on == "root" and rank != 0:
        return None
    return plan.decode_values(y, seeds)
