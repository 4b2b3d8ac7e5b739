"""Multi-GPU plumbing.

Batches of independent signals (C4) shard by signal: one process per GPU
(torchrun), each transforming its own signals; torch.distributed carries only
the start barrier and the max-over-ranks timing reduction -- nothing on the
data path.

One large signal (C5) shards its encode in one of two ways, each ending in
one all-reduce(sum) of PARTIAL bucket vectors (every round of every
iteration; bucketize is a sum over taps, linear in x) and the decode on the
full vector (Plan.decode_values) -- on every rank or on rank 0 only:
  "taps"  (x replicated, 2 GiB per GPU): rank r walks the r-th 1/world share
          of every encode task's t' segments (Plan.encode_values_part), so the
          encode work per rank shrinks as 1/world;
  "index" (no replication): rank r holds x[lo_r, hi_r) (index_range) and
          loads only those samples, but walks every tap.
The all-reduce adds the partials in a different order than the single-GPU
fold, a ~1e-16 relative difference.

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


def _agree_or_raise(exc, device, group=None):
    """Every rank learns whether any rank failed before the data collective
    (a rank that raised alone would leave the others blocked in all_reduce)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        if exc is not None:
            raise exc
        return
    backend = dist.get_backend(group)
    flag = torch.tensor([1 if exc is not None else 0], dtype=torch.int32,
                        device=device if backend == "nccl" else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    if exc is not None:
        raise exc
    if int(flag.item()):
        from . import InvalidArgument
        raise InvalidArgument("sharded_sfft4: another rank failed (see its error)")


def sharded_sfft4(plan, x, x_lo: int, seeds, decode_on: str = "all", group=None,
                  assume_valid: bool = False, mode: str = "index"):
    """One sharded transform step of one (batch of) large signal(s) on this rank.

    mode "index": x = x_local, the CUDA tensor (batch, span) of samples
      x[:, x_lo:x_lo+span] this rank holds (no replication; every rank walks
      every tap, so per-rank encode work does not shrink with the ranks).
    mode "taps": x holds whole signals (replicated); this rank walks its
      1/world share of every encode task's taps (Plan.encode_values_part),
      so the encode work per rank is 1/world; x_lo is ignored.
    Either way one all-reduce sums the partial bucket vectors.
    decode_on: "all" (every rank decodes the summed vector redundantly and
    returns the result) or "root" (rank 0 decodes; the others return None).
    A failure on any rank (e.g. a non-finite sample) raises on every rank
    before the data all-reduce.  Returns (f, c, count) CUDA tensors or None."""
    import torch.distributed as dist
    inited = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if inited else 0
    world = dist.get_world_size(group) if inited else 1
    y, exc = None, None
    try:
        if mode == "taps":
            y = plan.encode_values_part(x, seeds, rank, world, assume_valid=assume_valid)
        elif mode == "index":
            y = plan.encode_values(x, seeds, x_lo, assume_valid=assume_valid)
        else:
            raise ValueError(f"sharded_sfft4: unknown mode {mode!r}")
    except Exception as e:  # noqa: BLE001 -- re-raised after the ranks agree
        exc = e
    _agree_or_raise(exc, x.device, group)
    combine_partials(y, group)
    if decode_on == "root" and rank != 0:
        return None
    return plan.decode_values(y, seeds, folds=(mode == "taps"))
