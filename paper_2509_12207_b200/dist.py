"""Scenario sharding across GPUs.

Scenarios are independent; rank g of G simulates a contiguous range of global
scenario indices (randomness is keyed by the global index, so results do not
depend on G), then one ``all_reduce(SUM)`` of the int64 aggregate buffer
combines the per-chain counters and histograms.  Integer sums are associative,
so the reduced buffer is bit-identical for any G and any reduction order.
"""
from __future__ import annotations

from dataclasses import replace

from workloads.spec import Batch


def shard_range(rank: int, world: int, begin: int, count: int):
    """[lo, hi) of global scenario indices for `rank`: contiguous, balanced, covering [begin, begin+count)."""
    lo = begin + (rank * count) // world
    hi = begin + ((rank + 1) * count) // world
    return lo, hi


def shard_batch(b: Batch, rank: int, world: int) -> Batch:
    lo, hi = shard_range(rank, world, b.scenario_begin, b.scenario_count)
    return replace(b, scenario_begin=lo, scenario_count=hi - lo)


def allreduce_agg(agg, group=None):
    """The single collective of the path: SUM of the int64 aggregate buffer (NCCL over NVLink on GPUs)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(agg, op=dist.ReduceOp.SUM, group=group)
    return agg


def job_range(rank: int, world: int, begin: int, count: int, scaling: str = "weak"):
    """[lo, lo + n) of global scenario indices rank simulates for a config of `count` scenarios.

    weak:   every rank runs the whole configuration's size on its own global indices
            [begin + rank * count, begin + (rank + 1) * count) -- work per GPU fixed as N grows;
    strong: the configuration's `count` scenarios are partitioned (SURVEY.md §8(e):
            GPU g of G takes [floor(g S / G), floor((g + 1) S / G)))."""
    if scaling == "weak":
        return begin + rank * count, count
    if scaling == "strong":
        lo, hi = shard_range(rank, world, begin, count)
        return lo, hi - lo
    raise ValueError(f"scaling must be 'weak' or 'strong', not {scaling!r}")


def slices(lo: int, n: int, k: int):
    """Split [lo, lo + n) into k contiguous (begin, count) slices in order (sizes differ by at most 1;
    a slice may be empty when n < k)."""
    return [(lo + (i * n) // k, ((i + 1) * n) // k - (i * n) // k) for i in range(k)]


def reduce_job(launches: int, steps: int, seconds: float, device="cpu", group=None):
    """Whole-job bookkeeping across ranks: launch events and loop steps summed (int64), time as the
    max over ranks (float64).  Without a process group: the local values."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1):
        return int(launches), int(steps), float(seconds)
    n = torch.tensor([int(launches), int(steps)], dtype=torch.int64, device=device)
    t = torch.tensor([float(seconds)], dtype=torch.float64, device=device)
    dist.all_reduce(n, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(n[0].item()), int(n[1].item()), float(t[0].item())
