"""Multi-GPU host logic on CPU: scenario sharding and the single
SUM allreduce of the int64 aggregate buffer, world size 2 over gloo.

Each rank computes its shard's aggregates with the CPU oracle (the CUDA path is
the same per-shard computation; tests/test_gpu_parity.py pins it to the oracle),
then calls paper_2509_12207_b200.dist.allreduce_agg.  The reduced buffer must be
bit-identical to the unsharded run: integer sums are associative and all
randomness is keyed by the global scenario index.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_12207_b200.dist import shard_batch, shard_range
from workloads import get_config
from workloads.spec import Batch


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions():
    for count in (0, 1, 7, 1000, 12345):
        for world in (1, 2, 3, 4, 8):
            got = []
            for r in range(world):
                lo, hi = shard_range(r, world, 10, count)
                assert hi >= lo
                got.extend(range(lo, hi))
            assert got == list(range(10, 10 + count))
            sizes = [shard_range(r, world, 0, count)[1] - shard_range(r, world, 0, count)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, name, count, horizon, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2509_12207_b200.dist import allreduce_agg
    cfg = get_config(name)
    b = Batch(seed=cfg.batch.seed, scenario_count=count, horizon_ns=horizon, ftight_permille=400)
    sb = shard_batch(b, rank, world)
    r = O.run(cfg.workload(), cfg.policies["urgengo"], sb)
    agg = torch.from_numpy(r.agg.copy())
    allreduce_agg(agg)
    np.save(os.path.join(out_dir, f"agg{rank}.npy"), agg.numpy())
    np.save(os.path.join(out_dir, f"rec{rank}.npy"), r.records)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_allreduce_equals_unsharded(tmp_path, world):
    count, horizon = 7, 300_000_000
    mp.spawn(_worker, args=(world, _free_port(), "paper11", count, horizon, str(tmp_path)), nprocs=world, join=True)
    from oracle import oracle as O
    cfg = get_config("paper11")
    full = O.run(cfg.workload(), cfg.policies["urgengo"],
                 Batch(seed=cfg.batch.seed, scenario_count=count, horizon_ns=horizon, ftight_permille=400))
    aggs = [np.load(tmp_path / f"agg{r}.npy") for r in range(world)]
    for a in aggs:                      # every rank holds the same reduced buffer
        assert np.array_equal(a, full.agg)
    recs = np.concatenate([np.load(tmp_path / f"rec{r}.npy") for r in range(world)])
    assert np.array_equal(recs, full.records)   # shards are the global scenarios, in order


def test_allreduce_is_noop_without_process_group():
    from paper_2509_12207_b200.dist import allreduce_agg
    a = torch.arange(5, dtype=torch.int64)
    assert torch.equal(allreduce_agg(a.clone()), a)
