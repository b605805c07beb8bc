"""Per-task executors (R32) on the CUDA path vs the CPU oracle, bit-exact (-m gpu).

One warp lane per task thread: the pipeline recurrence cases of test_oracle_executors.py,
configs[1] under every policy, random workloads with every extended-model feature, the
throughput build, calibration, and geometry independence."""
import random

import numpy as np
import pytest

from oracle import oracle as O
from workloads import get_config
from workloads.spec import EXEC_TASK, FIFO, MS, STATIC, SYNC_ASYNC, URGENGO, US, Batch, Policy

from .gpu_helpers import assert_same, gpu_run
from .test_oracle_executors import CASES, workload
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


def paper11_te():
    cfg = get_config("paper11")
    w = cfg.workload()
    w.executors = EXEC_TASK
    return cfg, w


@pytest.mark.parametrize("case", range(len(CASES)))
def test_pipeline_cases(case):
    stages, period, offset, deadline, horizon, lam, sigma = CASES[case]
    w = workload(stages, period, offset, deadline, lam, sigma)
    for kind in (FIFO, STATIC, URGENGO):
        both(w, Policy(kind=kind, flags=0 if kind != URGENGO else 7, sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * US),
             Batch(horizon_ns=horizon), f"case {case} kind {kind}")


@pytest.mark.parametrize("name", ["urgengo", "fifo", "static"])
def test_paper11(name):
    cfg, w = paper11_te()
    b = Batch(seed=cfg.batch.seed, scenario_count=24, horizon_ns=2_000 * MS, ftight_permille=400)
    o, r, a = both(w, cfg.policies[name], b, name)
    assert o.launches > 0


@pytest.mark.parametrize("kind", [3, 4, 5, 6])
def test_paper11_classical(kind):
    cfg, w = paper11_te()
    b = Batch(seed=cfg.batch.seed, scenario_count=8, horizon_ns=2_000 * MS, ftight_permille=400)
    both(w, Policy(kind=kind, flags=0, sync_mode=cfg.policies["urgengo"].sync_mode), b, f"classical {kind}")


def _te_random_workload(rng):
    while True:
        w = random_workload(rng, C=rng.choice([1, 2, 4, 7, 11]), jitter=rng.choice([0, 3 * MS]))
        if sum(len(ch.tasks) for ch in w.chains) <= 32:
            break
    w.executors = EXEC_TASK
    return w


@pytest.mark.parametrize("seed", range(16))
def test_random_workloads(seed):
    rng = random.Random(17000 + seed)
    w = _te_random_workload(rng)
    if rng.random() < 0.5:
        from workloads.quantiles import inst_z_table, pareto_table
        w.inst_quantiles_q16 = inst_z_table()
        for ch in w.chains:
            ch.cpu_sigma_ppm, ch.gpu_sigma_ppm = rng.randint(0, 400_000), rng.randint(0, 400_000)
        if rng.random() < 0.5:
            w.kern_quantiles_q16 = pareto_table()
    p = random_policy(rng)
    p.kind = rng.choice([FIFO, STATIC, URGENGO, URGENGO, 3, 4, 5, 6])
    p.flags = rng.randint(0, 15) if p.kind == URGENGO else 0
    if p.kind == URGENGO and rng.random() < 0.3:
        p.noise_permille = rng.choice([100, 500])
    if rng.random() < 0.3:
        w.cpu_cores = rng.choice([1, 2, 4])
    if rng.random() < 0.3:
        w.contention_permille = rng.choice([200, 1000])
    if rng.random() < 0.3:
        for ch in w.chains:
            for t in ch.tasks:
                t.frees = rng.random() < 0.2
                for k in t.kernels:
                    k.flags = 1 if rng.random() < 0.2 else 0
    b = Batch(seed=seed, scenario_begin=rng.randint(0, 500), scenario_count=rng.randint(1, 24),
              horizon_ns=rng.choice([100, 300]) * MS, ftight_permille=rng.choice([0, 400]),
              fa_num=rng.choice([1, 3]), fa_den=rng.choice([1, 2]))
    both(w, p, b, f"te seed {seed}")


def test_throughput_build(monkeypatch):
    cfg, w = paper11_te()
    monkeypatch.setenv("URG_WIDE", "1")
    b = Batch(seed=cfg.batch.seed, scenario_count=16, horizon_ns=1_000 * MS, ftight_permille=400)
    for name in ("urgengo", "fifo"):
        both(w, cfg.policies[name], b, f"wide {name}")


def test_features_paper11():
    cfg, w = paper11_te()
    w.cpu_cores = 4
    w.contention_permille = 300
    w.chains[0].tasks[0].frees = True
    b = Batch(seed=cfg.batch.seed, scenario_count=6, horizon_ns=2_000 * MS, ftight_permille=400)
    p = cfg.policies["urgengo"]
    from dataclasses import replace
    both(w, replace(p, flags=p.flags | 8, noise_permille=200), b, "paper11 te + cores + alpha + free + noise")


def test_geometry_independent(monkeypatch):
    cfg, w = paper11_te()
    b = Batch(seed=cfg.batch.seed, scenario_count=40, horizon_ns=500 * MS, ftight_permille=400)
    ref = gpu_run(w, cfg.policies["urgengo"], b)
    monkeypatch.setenv("URG_WARPS_PER_CTA", "3")
    got = gpu_run(w, cfg.policies["urgengo"], b)
    assert np.array_equal(ref[0], got[0]) and np.array_equal(ref[1], got[1])


def test_calibration():
    from paper_2509_12207_b200.urg import DeviceWorkload
    cfg, w = paper11_te()
    p = cfg.policies["urgengo"]
    b = Batch(seed=cfg.batch.seed, scenario_count=3, horizon_ns=3_000 * MS, ftight_permille=400)
    with DeviceWorkload(w) as dw:
        lth, n, rows = dw.calibrate(p, b, 3_000_000_000)
    assert (lth, n) == O.calibrate(w, p, b, 3_000_000_000)
    want = O.calibration_samples(w, p, b, 3_000_000_000)
    assert n > 0 and all(np.array_equal(rows[j], want[j]) for j in range(3))


def test_rejects_predictor():
    from paper_2509_12207_b200.urg import DeviceWorkload, UrgError
    cfg, w = paper11_te()
    with DeviceWorkload(w) as dw:
        agg = torch.zeros(dw.agg_words, dtype=torch.int64, device="cuda")
        with pytest.raises(UrgError) as e:
            dw.simulate(Policy(cpu_ma_window=4), Batch(), agg, None)
        assert e.value.status == -1 and "per-task executors" in str(e.value)
