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


# ---- bench.py's multi-GPU bookkeeping (paper_2509_12207_b200.dist job_range / slices / reduce_job) ----

def test_job_range_weak_and_strong():
    from paper_2509_12207_b200.dist import job_range
    for world in (1, 2, 4, 8):
        weak = [job_range(r, world, 5, 1000, "weak") for r in range(world)]
        assert weak == [(5 + r * 1000, 1000) for r in range(world)]          # per-GPU work fixed
        strong = [job_range(r, world, 5, 1000, "strong") for r in range(world)]
        assert sum(n for _, n in strong) == 1000                              # total work fixed
        assert [lo for lo, _ in strong] == [5 + (r * 1000) // world for r in range(world)]
    with pytest.raises(ValueError):
        job_range(0, 1, 0, 1, "sideways")


def test_slices_cover_the_job_once():
    from paper_2509_12207_b200.dist import slices
    for n, k in ((1_000_000, 20), (1000, 3), (7, 20), (0, 4)):
        sl = slices(123, n, k)
        assert len(sl) == k
        got = [s for b, c in sl for s in range(b, b + c)]
        assert got == list(range(123, 123 + n))
        sizes = [c for _, c in sl]
        assert max(sizes) - min(sizes) <= 1


def test_bench_sample_is_baseline_md_rule():
    import bench
    s = bench.baseline_sample(0, 1_000_000)
    assert s[:256] == list(range(256)) and s[-256:] == list(range(1_000_000 - 256, 1_000_000))
    assert all(x in s for x in range(0, 1_000_000, 9973))
    assert len(s) == len(set(range(256)) | set(range(999_744, 1_000_000)) | set(range(0, 1_000_000, 9973)))
    assert bench.baseline_sample(10, 100) == list(range(10, 110))


def _bench_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2509_12207_b200.dist import allreduce_agg, job_range, reduce_job, slices
    # bench.py's bookkeeping with the oracle standing in for the kernel: per step one slice of the
    # rank's job, the step's aggregates allreduced, accumulated; launches summed, time max-reduced
    from oracle import oracle as O
    cfg = get_config("paper11")
    w, p = cfg.workload(), cfg.policies["urgengo"]
    res = {}
    for scaling in ("weak", "strong"):
        lo, S = job_range(rank, world, 0, 6, scaling)
        total = torch.zeros(len(O.run(w, p, Batch(horizon_ns=1)).agg), dtype=torch.int64)
        local_launch = 0
        for b0, c in slices(lo, S, 2):
            r = O.run(w, p, Batch(seed=cfg.batch.seed, scenario_begin=b0, scenario_count=c, horizon_ns=200_000_000,
                                  ftight_permille=400))
            local_launch += int(r.records[:, :, 4].astype(np.int64).sum())
            step = torch.from_numpy(r.agg.copy())
            allreduce_agg(step)
            total += step
        l_sum, s_sum, t_max = reduce_job(local_launch, 1, 0.5 + rank, "cpu")
        res[scaling] = (total.numpy().tolist(), l_sum, s_sum, t_max)
    np.save(os.path.join(out_dir, f"bench{rank}.npy"), np.array([res], dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_bench_bookkeeping(tmp_path):
    """World size 2 over gloo: the reduced per-step aggregates equal the unsharded run of the whole
    job (weak: 2 x 6 scenarios, strong: the same 6 split), the launch count reduced from the ranks'
    records equals the aggregate's launch word, and the time is the max over ranks."""
    world = 2
    mp.spawn(_bench_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    from oracle import oracle as O
    cfg = get_config("paper11")
    w, p = cfg.workload(), cfg.policies["urgengo"]
    res = [np.load(tmp_path / f"bench{r}.npy", allow_pickle=True)[0] for r in range(world)]
    for scaling, count in (("weak", 12), ("strong", 6)):
        full = O.run(w, p, Batch(seed=cfg.batch.seed, scenario_count=count, horizon_ns=200_000_000,
                                 ftight_permille=400))
        for r in range(world):
            total, l_sum, s_sum, t_max = res[r][scaling]
            assert np.array_equal(np.array(total, np.int64), full.agg)
            assert l_sum == full.launches and s_sum == world and t_max == 1.5
