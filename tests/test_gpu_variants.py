"""Template variants (R33) on the CUDA path vs the oracle, bit-exact (-m gpu): kernel
records of V sets read from HBM/L2, scenarios grouped by variant in the work order."""
import random

import numpy as np
import pytest

from oracle import oracle as O
from workloads import get_config, paper11_variants
from workloads.spec import EXEC_TASK, FIFO, MS, STATIC, Batch, Kernel, Policy

from .gpu_helpers import assert_same, gpu_run
from .test_oracle_properties import random_policy, random_workload

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_12207_b200.urg import lib
    lib()


def both(w, p, b, ctx=""):
    o = O.run(w, p, b)
    r, a = gpu_run(w, p, b)
    assert_same(o, r, a, ctx)
    return o, r, a


@pytest.mark.parametrize("name", ["urgengo", "fifo", "static"])
def test_paper11_variants(name):
    cfg = get_config("paper11")
    w = paper11_variants(8)
    b = Batch(seed=cfg.batch.seed, scenario_begin=3, scenario_count=21, horizon_ns=1_000 * MS, ftight_permille=400)
    both(w, cfg.policies[name], b, name)


@pytest.mark.parametrize("seed", range(8))
def test_random_variants(seed):
    rng = random.Random(18000 + seed)
    w = random_workload(rng, C=rng.choice([1, 3, 6, 13]))
    n = w.total_kernels()
    flat = [k for ch in w.chains for t in ch.tasks for k in t.kernels]
    V = rng.choice([2, 3, 7, 40])
    w.kernel_variants = [[Kernel(rng.randint(10_000, 2 * MS), rng.randint(10_000, 2 * MS),
                                 rng.choice([50, 300, 700, 1000]), flat[i].flags) for i in range(n)]
                         for _ in range(V - 1)]
    p = random_policy(rng)
    p.kind = rng.choice([FIFO, STATIC, 2, 2, 3, 6])
    p.flags = rng.randint(0, 15) if p.kind == 2 else 0
    if rng.random() < 0.3:
        w.executors = EXEC_TASK if sum(len(ch.tasks) for ch in w.chains) <= 32 else 0
    b = Batch(seed=seed, scenario_begin=rng.randint(0, 100), scenario_count=rng.randint(1, 50),
              horizon_ns=200 * MS, ftight_permille=rng.choice([0, 400]))
    both(w, p, b, f"variants seed {seed} V={V}")


def test_throughput_and_packed_builds(monkeypatch):
    cfg = get_config("paper11")
    w = paper11_variants(16)
    monkeypatch.setenv("URG_WIDE", "1")
    b = Batch(seed=cfg.batch.seed, scenario_begin=5, scenario_count=37, horizon_ns=500 * MS, ftight_permille=400)
    for name in ("urgengo", "fifo"):
        both(w, cfg.policies[name], b, f"wide {name}")


def test_grouped_order_geometry_independent(monkeypatch):
    """The variant-grouped work order changes which warp runs which scenario, never the results."""
    cfg = get_config("paper11")
    w = paper11_variants(64)
    b = Batch(seed=cfg.batch.seed, scenario_begin=1000, scenario_count=300, horizon_ns=300 * MS, ftight_permille=400)
    ref = gpu_run(w, cfg.policies["urgengo"], b)
    for wpc in ("1", "5", "16"):
        monkeypatch.setenv("URG_WARPS_PER_CTA", wpc)
        got = gpu_run(w, cfg.policies["urgengo"], b)
        assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])
    sample = [0, 1, 63, 64, 65, 150, 299]
    for j in sample:
        o = O.run(w, cfg.policies["urgengo"], Batch(seed=b.seed, scenario_begin=b.scenario_begin + j, scenario_count=1,
                                                    horizon_ns=b.horizon_ns, ftight_permille=400))
        assert np.array_equal(o.records[0], ref[0][j]), j
