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
