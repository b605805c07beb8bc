"""CUDA path vs the CPU oracle, element by element, through the C ABI (-m gpu).

Integer results must match bit-exactly (DESIGN.md §2 R22-R23): per-scenario
records (including rt_hash, which pins every individual response time), the
aggregate counters, both histograms, and the launch / loop-step counters.
"""
import random

import numpy as np
import pytest

from oracle import oracle as O
from workloads import get_config, paper11, toy2, w1, w2, w3
from workloads.configs import _paper11_heavy
from workloads.spec import (F_ALL, FIFO, MS, STATIC, SYNC_ASYNC, SYNC_BATCHED, SYNC_EACH, SYNC_OVERLAP, URGENGO,
                            US, Batch, Chain, Kernel, Policy, Task, Workload)

from .gpu_helpers import agg_from_records, assert_same, gpu_run
from .test_oracle_properties import random_policy, random_workload

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_12207_b200.urg import lib
    lib()   # loud failure if liburg.so is missing


def both(w, p, b, ctx=""):
    o = O.run(w, p, b)
    r, a = gpu_run(w, p, b)
    assert_same(o, r, a, ctx)
    return o, r, a


def test_philox_known_answers_device():
    from paper_2509_12207_b200.urg import philox_device
    kat = [([0, 0, 0, 0], [0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
           ([0xffffffff] * 4, [0xffffffff] * 2, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
           ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0],
            [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1])]
    out = philox_device(np.array([k[0] for k in kat]), np.array([k[1] for k in kat]))
    assert out.tolist() == [k[2] for k in kat]
    rng = np.random.default_rng(0)
    ctr = rng.integers(0, 2**32, size=(20000, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, size=(20000, 2), dtype=np.uint64).astype(np.uint32)
    dev = philox_device(ctr, key)
    for i in range(0, 20000, 997):
        assert dev[i].tolist() == O.philox(ctr[i], key[i]).tolist()


@pytest.mark.parametrize("kind,flags", [(FIFO, 0), (STATIC, 0), (URGENGO, 1), (URGENGO, 2), (URGENGO, 3), (URGENGO, 0)])
def test_w1(kind, flags):
    both(w1(), Policy(kind=kind, flags=flags, sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * MS), Batch(horizon_ns=1 * MS))


@pytest.mark.parametrize("mode", [SYNC_ASYNC, SYNC_EACH, SYNC_BATCHED, SYNC_OVERLAP])
def test_w2(mode):
    both(w2(), Policy(kind=URGENGO, flags=0, sync_mode=mode, lax_threshold_ns=-1), Batch(horizon_ns=1 * MS))


def test_w3():
    both(w3(), Policy(kind=URGENGO, flags=4, sync_mode=SYNC_ASYNC), Batch(horizon_ns=1 * MS))
    both(w3(), Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC), Batch(horizon_ns=1 * MS))


@pytest.mark.parametrize("build", ["small", "512", "packed", "ext"])
def test_w10_zero_cost_satisfied_sync(build, monkeypatch):
    """Fixture W10 (tests/golden/w10.json): a satisfied zero-cost OVERLAP sync continues in the same
    Phase B step against the step's snapshot (R21) -- in every build."""
    from workloads import w10
    from workloads.spec import F_DELAY
    _build_env(build, monkeypatch)
    p = Policy(kind=URGENGO, flags=F_DELAY, sync_mode=SYNC_OVERLAP, delta_eval_ns=500 * US, lax_threshold_ns=5 * MS)
    o, r, a = both(w10(), p, Batch(horizon_ns=1 * MS, scenario_count=_count(build)), f"w10 {build}")
    assert int(r[0, 0, 6]) == 1_600_000 and int(r[0, 1, 6]) == 2_200_000


@pytest.mark.parametrize("build", ["small", "512", "packed", "ext"])
def test_w11_binding_levels_num_pri_6(build, monkeypatch):
    """Fixture W11 (tests/golden/w11.json): NUM_PRI = 6 rank normalisation decides the dispatch order."""
    from workloads import w11
    from workloads.spec import F_BIND
    _build_env(build, monkeypatch)
    p = Policy(kind=URGENGO, flags=F_BIND, sync_mode=SYNC_ASYNC, lax_threshold_ns=1 * MS)
    o, r, a = both(w11(), p, Batch(horizon_ns=10 * MS, scenario_count=_count(build)), f"w11 {build}")
    assert [int(r[0, c, 6]) // MS for c in range(6)] == [51, 52, 53, 103, 101, 102]


def _build_env(build, monkeypatch):
    """Select a kernel build through the test hooks of urg_api.cu (fixture batches are tiny)."""
    if build == "512":
        monkeypatch.setenv("URG_SMALL", "0")
    elif build == "packed":
        monkeypatch.setenv("URG_WIDE", "1")
    elif build == "ext":
        monkeypatch.setenv("URG_EXT", "1")


def _count(build):
    return 2 if build == "packed" else 1   # both halves of a packed warp run the same fixture


@pytest.mark.parametrize("mode", [SYNC_ASYNC, SYNC_EACH, SYNC_BATCHED, SYNC_OVERLAP])
def test_toy2_all_policies(mode):
    """BASELINE.json configs[0]: every policy and UrgenGo flag combination, bit-exact."""
    cfg = get_config("toy2")
    w = toy2()
    pols = [Policy(kind=FIFO, flags=0, sync_mode=mode), Policy(kind=STATIC, flags=0, sync_mode=mode)]
    pols += [Policy(kind=URGENGO, flags=f, sync_mode=mode, lax_threshold_ns=10 * MS) for f in range(8)]
    for p in pols:
        both(w, p, cfg.batch, f"toy2 kind={p.kind} flags={p.flags} mode={mode}")


@pytest.mark.parametrize("seed", range(24))
def test_random_small_workloads(seed):
    rng = random.Random(seed)
    w = random_workload(rng, C=rng.choice([1, 2, 3, 5, 8, 13, 32]), jitter=rng.choice([0, 3 * MS]))
    w.sync_lo_ns = rng.choice([0, 10 * US])
    w.sync_hi_ns = w.sync_lo_ns + rng.choice([0, 150 * US])
    if rng.random() < 0.5:
        from workloads.quantiles import inst_z_table, pareto_table
        w.inst_quantiles_q16 = inst_z_table()
        for ch in w.chains:
            ch.cpu_sigma_ppm, ch.gpu_sigma_ppm = rng.randint(0, 500_000), rng.randint(0, 500_000)
        if rng.random() < 0.5:
            w.kern_quantiles_q16 = pareto_table()
    p = random_policy(rng)
    b = Batch(seed=seed * 7 + 1, scenario_begin=rng.randint(0, 1000), scenario_count=rng.randint(1, 40),
              horizon_ns=rng.choice([100, 300]) * MS, ftight_permille=rng.choice([0, 400, 1000]),
              fa_num=rng.choice([1, 5]), fa_den=rng.choice([1, 4]), fd_num=rng.choice([1, 3]), fd_den=rng.choice([1, 2]))
    both(w, p, b, f"seed {seed}")


@pytest.mark.parametrize("seed", range(8))
def test_random_small_workloads_512_thread_build(seed, monkeypatch):
    """URG_SMALL=0: batches of at most 8 warps per SM on the 512-thread latency build (the one
    bigger batches up to 16 warps per SM use) -- equal to the oracle like the default small build."""
    monkeypatch.setenv("URG_SMALL", "0")
    test_random_small_workloads(seed + 100)


def test_small_build_equals_512_thread_build(monkeypatch):
    """The 256-thread latency build (255-register cap) and the 512-thread one give identical
    records and aggregates on configs[1]'s workload, for every policy of the config."""
    cfg = get_config("paper11")
    w = cfg.workload()
    b = Batch(seed=cfg.batch.seed, scenario_count=300, horizon_ns=2_000 * MS, ftight_permille=400)
    for name, p in cfg.policies.items():
        r1, a1 = gpu_run(w, p, b)
        monkeypatch.setenv("URG_SMALL", "0")
        r2, a2 = gpu_run(w, p, b)
        monkeypatch.delenv("URG_SMALL")
        assert np.array_equal(r1, r2) and np.array_equal(a1, a2), name


@pytest.mark.parametrize("build", ["small", "512", "packed"])
@pytest.mark.parametrize("kind", [URGENGO, FIFO, STATIC])
def test_long_gaps_and_long_kernels(kind, build, monkeypatch):
    """Events 2^30..2^33 ns apart and kernels / CPU segments longer than 2^31 ns beside a chain
    with frequent small events: the kernel's 32-bit next-event distances go far, drift and
    are refreshed exactly, results equal to the oracle's -- in the small and
    512-thread latency builds and in the packed throughput build (64-bit head)."""
    if build == "512":
        monkeypatch.setenv("URG_SMALL", "0")
    elif build == "packed":
        monkeypatch.setenv("URG_WIDE", "1")
    S = 1_000 * MS
    a = Chain(6 * S, 5 * S, 0, [Task(1 * MS, 1 * MS, [Kernel(3 * S, 3 * S, 1000), Kernel(1 * MS, 1 * MS, 500)])])
    b = Chain(1_500 * MS, 1 * S, 2_200 * MS, [Task(2_500 * MS, 2_500 * MS, [Kernel(10 * MS, 10 * MS, 600)])])
    c = Chain(40 * MS, 30 * MS, 0, [Task(1 * MS, 1 * MS, [Kernel(200 * US, 200 * US, 300), Kernel(2 * MS, 2 * MS, 800)])])
    idle = Chain(9 * S, 1 * S, 4_400 * MS, [Task(0, 0, [Kernel(5 * MS, 5 * MS, 100)])])
    for chains in ([a, b, c, idle], [a, idle], [b, idle]):
        w = Workload(chains=chains, num_prio=6, launch_ns=21_672, launch_akb_ns=500, sync_lo_ns=10 * US,
                     sync_hi_ns=200 * US, jitter_ns=30 * MS, rt_bins=64, rt_bin_ns=100 * MS)
        p = Policy(kind=kind, flags=F_ALL if kind == URGENGO else 0, sync_mode=SYNC_OVERLAP,
                   delta_eval_ns=500 * US, lax_threshold_ns=20 * MS, sleep_ns=1 * MS, util_exempt_permille=100)
        bb = Batch(seed=0x5EED00AA, scenario_count=5, horizon_ns=20 * S)
        both(w, p, bb, f"long gaps, {len(chains)} chains, kind {kind}")


@pytest.mark.parametrize("name", ["urgengo", "fifo", "static"])
def test_paper11_small(name):
    """configs[1] workload at a size the oracle finishes in seconds: 48 scenarios x 2 s, spanning many CTAs."""
    cfg = get_config("paper11")
    b = Batch(seed=cfg.batch.seed, scenario_count=48, horizon_ns=2_000 * MS, ftight_permille=400)
    o, r, a = both(cfg.workload(), cfg.policies[name], b, name)
    assert o.launches > 0


def test_paper11_full_size_sampled():
    """configs[1] at full size in bench.py's launch configuration (1000 scenarios x 10 s, UrgenGo):
    sampled scenarios vs the oracle one by one, and the aggregate vs the GPU's own records."""
    cfg = get_config("paper11")
    w, p, b = cfg.workload(), cfg.policies["urgengo"], cfg.batch
    r, a = gpu_run(w, p, b)
    assert r.shape == (1000, 11, 8)
    recon = agg_from_records(r, w.num_chains, w.rt_bins)
    stride = 5 + w.rt_bins + 101
    for c in range(w.num_chains):
        assert np.array_equal(a[c * stride: c * stride + 5], recon[c * stride: c * stride + 5])
        assert np.array_equal(a[c * stride + 5 + w.rt_bins:(c + 1) * stride],
                              recon[c * stride + 5 + w.rt_bins:(c + 1) * stride])
        # completed instances = rt histogram mass
        comp = int(r[:, c, 0].astype(np.int64).sum() - r[:, c, 2].astype(np.int64).sum() - r[:, c, 3].astype(np.int64).sum())
        assert a[c * stride + 5: c * stride + 5 + w.rt_bins].sum() == comp
    assert a[-2] == recon[-2]
    for s in [0, 1, 2, 333, 500, 998, 999]:
        bs = Batch(seed=b.seed, scenario_begin=s, scenario_count=1, horizon_ns=b.horizon_ns,
                   ftight_permille=b.ftight_permille)
        o = O.run(w, p, bs)
        assert np.array_equal(o.records[0], r[s]), f"scenario {s}"


def test_heavy_tail_and_sweep_points():
    """configs[3] (Pareto kernel factors) and two configs[2] sweep points, exact."""
    lth = get_config("paper11").policies["urgengo"].lax_threshold_ns
    wj = _paper11_heavy()
    for p in [Policy(kind=URGENGO, flags=F_ALL, sync_mode=SYNC_OVERLAP, lax_threshold_ns=lth),
              Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC)]:
        both(wj, p, Batch(seed=0x5EED0004, scenario_count=16, horizon_ns=3_000 * MS, ftight_permille=400), "jitter")
    cfg3 = get_config("usweep")
    for bb in (cfg3.sweep[0], cfg3.sweep[-1]):
        b = Batch(seed=bb.seed, scenario_begin=12345, scenario_count=16, horizon_ns=2_000 * MS,
                  ftight_permille=400, fa_num=bb.fa_num, fa_den=bb.fa_den)
        for name in ("urgengo", "static"):
            both(cfg3.workload(), cfg3.policies[name], b, f"usweep {bb.fa_num}/{bb.fa_den} {name}")


def test_edge_cases():
    cfg = get_config("paper11")
    w, p = cfg.workload(), cfg.policies["urgengo"]
    # empty batch: no-op
    r, a = gpu_run(w, p, Batch(scenario_count=0, horizon_ns=MS))
    assert not a.any()
    # horizon 0: nothing admitted
    both(w, p, Batch(seed=3, scenario_count=4, horizon_ns=0), "H=0")
    # one bin, explicit tight set, single chain
    w1c = toy2()
    w1c.rt_bins = 1
    both(w1c, p, Batch(seed=5, scenario_count=3, horizon_ns=700 * MS, tight_explicit=1, tight_mask=0b10), "rt_bins=1")
    solo = Workload(chains=[paper11().chains[10]], jitter_ns=0, inst_quantiles_q16=None)
    both(solo, p, Batch(seed=9, scenario_count=2, horizon_ns=20_000 * MS), "C=1 llama")


def test_sharding_invariance_single_gpu():
    """Sub-range calls add up to the full-range call (SURVEY.md §4 fake-shard test)."""
    import torch

    from paper_2509_12207_b200.dist import shard_batch
    from paper_2509_12207_b200.urg import DeviceWorkload
    cfg = get_config("paper11")
    w, p = cfg.workload(), cfg.policies["urgengo"]
    b = Batch(seed=cfg.batch.seed, scenario_count=300, horizon_ns=1_000 * MS, ftight_permille=400)
    with DeviceWorkload(w) as dw:
        full = torch.zeros(dw.agg_words, dtype=torch.int64, device="cuda")
        dw.simulate(p, b, full)
        parts = torch.zeros_like(full)
        for g in range(3):
            dw.simulate(p, shard_batch(b, g, 3), parts)
        torch.cuda.synchronize()
        assert torch.equal(full, parts)


def test_host_variant_matches_device():
    from paper_2509_12207_b200.urg import DeviceWorkload
    cfg = get_config("paper11")
    w, p = cfg.workload(), cfg.policies["urgengo"]
    b = Batch(seed=cfg.batch.seed, scenario_count=64, horizon_ns=1_000 * MS, ftight_permille=400)
    r, a = gpu_run(w, p, b)
    agg = np.zeros_like(a)
    rec = np.zeros_like(r)
    with DeviceWorkload(w) as dw:
        dw.simulate_host(p, b, agg, rec)
        per, overall = dw.miss_ratios(agg)
    assert np.array_equal(agg, a) and np.array_equal(rec, r)
    tot = rec[:, :, 0].astype(np.int64).sum(0)
    miss = rec[:, :, 1].astype(np.int64).sum(0)
    assert overall == O.overall_miss_ratio(miss, tot)


@pytest.fixture
def wide_build(monkeypatch):
    """Force the throughput instantiations (1024-thread CTAs, <= 64 registers) that
    urg_simulate_batch picks for batches larger than 16 warps per SM."""
    monkeypatch.setenv("URG_WIDE", "1")
    yield


@pytest.mark.parametrize("name", ["urgengo", "fifo", "static"])
def test_wide_build_paper11(wide_build, name):
    cfg = get_config("paper11")
    b = Batch(seed=cfg.batch.seed, scenario_begin=777, scenario_count=40, horizon_ns=2_000 * MS, ftight_permille=400)
    both(cfg.workload(), cfg.policies[name], b, f"wide {name}")


def test_wide_build_heavy_tail_and_toy(wide_build):
    lth = get_config("paper11").policies["urgengo"].lax_threshold_ns
    both(_paper11_heavy(), Policy(kind=URGENGO, flags=F_ALL, sync_mode=SYNC_OVERLAP, lax_threshold_ns=lth),
         Batch(seed=0x5EED0004, scenario_count=16, horizon_ns=3_000 * MS, ftight_permille=400), "wide jitter")
    for mode in (SYNC_ASYNC, SYNC_EACH, SYNC_BATCHED, SYNC_OVERLAP):
        for f in (0, 3, 7):
            both(toy2(), Policy(kind=URGENGO, flags=f, sync_mode=mode, lax_threshold_ns=10 * MS),
                 get_config("toy2").batch, f"wide toy2 {f} {mode}")


def test_throughput_batch_sampled():
    """A batch large enough to select the throughput build by itself (> 16 warps per SM):
    configs[4]'s workload, 4000 scenarios x 200 ms, sampled scenarios vs the oracle."""
    cfg = get_config("scaleout")
    w, p = cfg.workload(), cfg.policies["urgengo"]
    b = Batch(seed=cfg.batch.seed, scenario_count=4000, horizon_ns=200 * MS, ftight_permille=400)
    r, a = gpu_run(w, p, b)
    recon = agg_from_records(r, w.num_chains, w.rt_bins)
    assert a[-2] == recon[-2]
    for s in [0, 1, 2047, 3998, 3999]:
        o = O.run(w, p, Batch(seed=b.seed, scenario_begin=s, scenario_count=1, horizon_ns=b.horizon_ns,
                              ftight_permille=400))
        assert np.array_equal(o.records[0], r[s]), f"scenario {s}"


@pytest.mark.parametrize("flags", [8, 9, 10, 15])
def test_w4_collisions(flags):
    from workloads import w4
    both(w4(), Policy(kind=URGENGO, flags=flags, sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * MS), Batch(horizon_ns=1 * MS),
         f"w4 flags={flags}")


@pytest.mark.parametrize("seed", range(8))
def test_collisions_random(seed):
    rng = random.Random(5000 + seed)
    w = random_workload(rng, C=rng.choice([2, 4, 7, 16]))
    p = random_policy(rng)
    p.kind = URGENGO
    p.flags = rng.randint(0, 7) | 8
    p.lax_threshold_ns = rng.choice([2 * MS, 8 * MS, 30 * MS])
    both(w, p, Batch(seed=seed, scenario_count=rng.randint(1, 24), horizon_ns=300 * MS), f"coll seed {seed}")


def test_collisions_paper11(wide_build):
    from workloads.spec import collision_hist
    cfg = get_config("paper11")
    w = cfg.workload()
    for flags in (8 | 7, 8 | 5):     # UrgenGo with and without delayed launching (P:790 comparison)
        p = Policy(kind=URGENGO, flags=flags, sync_mode=SYNC_OVERLAP,
                   lax_threshold_ns=cfg.policies["urgengo"].lax_threshold_ns)
        o, r, a = both(w, p, Batch(seed=cfg.batch.seed, scenario_count=12, horizon_ns=2_000 * MS, ftight_permille=400),
                       f"paper11 collisions flags={flags}")
        assert collision_hist(a, w.num_chains, w.rt_bins).sum() > 0


def test_sweep_points_match_oracle():
    """paper_2509_12207_b200.sweep runs each study point through the C ABI; two points of
    three studies checked against the oracle's aggregates (Eq. 3 and collisions included)."""
    from dataclasses import replace as rp
    from paper_2509_12207_b200 import sweep as SW
    cfg = get_config("paper11")
    w, base = cfg.workload(), cfg.policies["urgengo"]
    b = Batch(seed=cfg.batch.seed, scenario_count=6, horizon_ns=1_000 * MS, ftight_permille=400)
    pts = [SW.sync_modes(base, b)[0], SW.num_prio(base, b)[1], SW.collisions(base, b)[0]]
    res = SW.run(w, pts)
    for pt, r in zip(pts, res):
        ww = rp(w, num_prio=pt.num_prio) if pt.num_prio else w
        o = O.run(ww, pt.policy, pt.batch)
        assert r.launches == o.launches and r.steps == o.steps
        tot = o.records[:, :, 0].astype(np.int64).sum(0)
        miss = o.records[:, :, 1].astype(np.int64).sum(0)
        assert r.overall_miss == O.overall_miss_ratio(miss, tot), pt.label


def _gpu_calibrate(w, p, b, window_ns=30_000_000_000):
    from paper_2509_12207_b200.urg import DeviceWorkload
    with DeviceWorkload(w) as dw:
        return dw.calibrate(p, b, window_ns)


def test_calibration_fixtures():
    """urg_calibrate on the hand-worked W1 / W3 sampling pins."""
    p = Policy(kind=URGENGO, flags=7, sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * MS)
    lth, n, rows = _gpu_calibrate(w1(), p, Batch(horizon_ns=20 * MS))
    assert (lth, n) == (4 * MS, 9) and rows[0].tolist() == [4 * MS] * 9
    lth, n, rows = _gpu_calibrate(w1(), p, Batch(horizon_ns=20 * MS), window_ns=5 * MS)
    assert n == 4
    assert _gpu_calibrate(w3(), p, Batch(horizon_ns=20 * MS))[:2] == (-1, 0)


def test_calibration_paper11_matches_stored_threshold():
    """configs[1] scenario 0, 30 s window (10 s horizon): the GPU reproduces the oracle's
    samples one by one and the stored L_th (workloads/calibrated.json)."""
    import json
    import os
    cfg = get_config("paper11")
    w, p = cfg.workload(), cfg.policies["urgengo"]
    b = Batch(seed=cfg.batch.seed, scenario_count=1, horizon_ns=cfg.batch.horizon_ns, ftight_permille=400)
    lth, n, rows = _gpu_calibrate(w, p, b)
    stored = json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "workloads", "calibrated.json")))
    assert (lth, n) == (stored["paper11"], stored["_samples"]["paper11"])
    assert np.array_equal(rows[0], O.calibration_samples(w, p, b)[0])


@pytest.mark.parametrize("seed", range(6))
def test_calibration_pooled_random(seed):
    rng = random.Random(7000 + seed)
    w = random_workload(rng, C=rng.choice([2, 5, 11, 32]))
    p = random_policy(rng)
    p.kind = URGENGO
    b = Batch(seed=seed, scenario_begin=rng.randint(0, 100), scenario_count=rng.randint(1, 30),
              horizon_ns=rng.choice([200, 500]) * MS, ftight_permille=rng.choice([0, 400]))
    win = rng.choice([50 * MS, 30_000 * MS])
    lth, n, rows = _gpu_calibrate(w, p, b, win)
    orows = O.calibration_samples(w, p, b, win)
    assert [r.tolist() for r in rows] == [r.tolist() for r in orows]
    assert (lth, n) == O.calibrate(w, p, b, win)


@pytest.mark.parametrize("eps,W", [(300, 0), (0, 8), (500, 3), (1000, 1)])
def test_noise_and_predictor_paper11(eps, W):
    """R25 estimation noise and R26 CPU moving average on configs[1], both builds."""
    cfg = get_config("paper11")
    p = Policy(**{**cfg.policies["urgengo"].__dict__, "noise_permille": eps, "cpu_ma_window": W})
    b = Batch(seed=cfg.batch.seed, scenario_begin=40, scenario_count=10, horizon_ns=2_000 * MS, ftight_permille=400)
    both(cfg.workload(), p, b, f"paper11 eps={eps} W={W}")


def test_noise_and_predictor_wide(wide_build):
    cfg = get_config("paper11")
    p = Policy(**{**cfg.policies["urgengo"].__dict__, "noise_permille": 300, "cpu_ma_window": 8})
    both(cfg.workload(), p, Batch(seed=cfg.batch.seed, scenario_count=9, horizon_ns=2_000 * MS, ftight_permille=400),
         "wide noise+ma")


@pytest.mark.parametrize("seed", range(8))
def test_noise_and_predictor_random(seed):
    rng = random.Random(9000 + seed)
    w = random_workload(rng, C=rng.choice([1, 3, 6, 13]))
    if rng.random() < 0.5:
        from workloads.quantiles import inst_z_table
        w.inst_quantiles_q16 = inst_z_table()
        for ch in w.chains:
            ch.cpu_sigma_ppm = rng.randint(0, 400_000)
    p = random_policy(rng)
    p.kind = URGENGO
    p.noise_permille = rng.choice([0, 1, 250, 1000])
    p.cpu_ma_window = rng.choice([0, 1, 2, 8, 64])
    both(w, p, Batch(seed=seed, scenario_count=rng.randint(1, 20), horizon_ns=300 * MS), f"noise/ma seed {seed}")


@pytest.mark.parametrize("kind", [3, 4, 5, 6])
def test_classical_policies(kind):
    """R27 classical policies: W1 (NUM_PRI 3), random workloads, configs[1] in both builds."""
    w = w1()
    w.num_prio = 3
    both(w, Policy(kind=kind, flags=0, sync_mode=SYNC_ASYNC), Batch(horizon_ns=1 * MS), f"w1 kind {kind}")
    rng = random.Random(11000 + kind)
    for _ in range(4):
        wr = random_workload(rng, C=rng.choice([2, 5, 9, 32]))
        pr = random_policy(rng)
        pr.kind = kind
        pr.cpu_ma_window = rng.choice([0, 4])
        both(wr, pr, Batch(seed=kind, scenario_count=rng.randint(1, 12), horizon_ns=300 * MS), f"rand kind {kind}")
    cfg = get_config("paper11")
    b = Batch(seed=cfg.batch.seed, scenario_count=8, horizon_ns=2_000 * MS, ftight_permille=400)
    both(cfg.workload(), Policy(kind=kind, flags=0, sync_mode=SYNC_OVERLAP), b, f"paper11 kind {kind}")


def test_classical_policies_wide(wide_build):
    cfg = get_config("paper11")
    b = Batch(seed=cfg.batch.seed, scenario_begin=100, scenario_count=8, horizon_ns=2_000 * MS, ftight_permille=400)
    for kind in (3, 4, 5, 6):
        both(cfg.workload(), Policy(kind=kind, flags=0, sync_mode=SYNC_ASYNC), b, f"wide kind {kind}")


def _with_frees(w, n):
    """The first n tasks (chain-major) end with cudaFree (the PAPER.md:909 experiment knob)."""
    k = 0
    for ch in w.chains:
        for t in ch.tasks:
            t.frees = k < n
            k += 1
    return w


def test_cudafree_fixtures():
    from workloads import w6
    for two in (False, True):
        for kind in (FIFO, STATIC, URGENGO, 3, 5):
            both(w6(two), Policy(kind=kind, flags=7 if kind == URGENGO else 0, sync_mode=SYNC_ASYNC,
                                 lax_threshold_ns=-1), Batch(horizon_ns=1 * MS), f"w6 {two} {kind}")


@pytest.mark.parametrize("seed", range(8))
def test_cudafree_random(seed):
    rng = random.Random(12000 + seed)
    w = random_workload(rng, C=rng.choice([2, 4, 11, 32]))
    for ch in w.chains:
        for t in ch.tasks:
            t.frees = rng.random() < 0.3
    w.free_ns = rng.choice([1, 50 * US, 188 * US, 2 * MS])
    p = random_policy(rng)
    p.kind = rng.choice([FIFO, STATIC, URGENGO, 3, 4, 5, 6])
    both(w, p, Batch(seed=seed, scenario_count=rng.randint(1, 16), horizon_ns=300 * MS), f"free seed {seed}")


@pytest.mark.parametrize("n", [1, 4])
def test_cudafree_paper11(n, wide_build):
    cfg = get_config("paper11")
    w = _with_frees(cfg.workload(), n)
    b = Batch(seed=cfg.batch.seed, scenario_count=8, horizon_ns=2_000 * MS, ftight_permille=400)
    for name in ("urgengo", "fifo", "static"):
        both(w, cfg.policies[name], b, f"paper11 frees={n} {name}")


@pytest.fixture
def ext_build(monkeypatch):
    """Force the extended-model instantiations (R25/R26/R28 resolved at run time)."""
    monkeypatch.setenv("URG_EXT", "1")
    yield


def test_extended_build_equals_core(ext_build):
    """With noise, predictor and cudaFree off, the extended build reproduces the oracle exactly
    like the core build (W1, toy2, paper11, a classical policy)."""
    both(w1(), Policy(kind=URGENGO, flags=3, sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * MS), Batch(horizon_ns=1 * MS), "ext w1")
    for mode in (SYNC_ASYNC, SYNC_OVERLAP):
        both(toy2(), Policy(kind=URGENGO, flags=7, sync_mode=mode, lax_threshold_ns=10 * MS), get_config("toy2").batch,
             "ext toy2")
    cfg = get_config("paper11")
    b = Batch(seed=cfg.batch.seed, scenario_count=8, horizon_ns=2_000 * MS, ftight_permille=400)
    for name in ("urgengo", "fifo", "static"):
        both(cfg.workload(), cfg.policies[name], b, f"ext paper11 {name}")
    both(cfg.workload(), Policy(kind=5, flags=0, sync_mode=SYNC_OVERLAP), b, "ext paper11 hrrn")


@pytest.mark.parametrize("seed", range(10))
def test_packed_two_scenarios_per_warp(seed, wide_build):
    """PK build (two scenarios per warp, throughput core build, C <= 16): random workloads and
    policies, odd scenario counts (the last warp's upper half has no scenario)."""
    rng = random.Random(13000 + seed)
    w = random_workload(rng, C=rng.choice([1, 2, 5, 11, 16]), jitter=rng.choice([0, 2 * MS]))
    if rng.random() < 0.5:
        from workloads.quantiles import inst_z_table, pareto_table
        w.inst_quantiles_q16 = inst_z_table()
        for ch in w.chains:
            ch.cpu_sigma_ppm, ch.gpu_sigma_ppm = rng.randint(0, 500_000), rng.randint(0, 500_000)
        if rng.random() < 0.5:
            w.kern_quantiles_q16 = pareto_table()
    p = random_policy(rng)
    p.kind = rng.choice([FIFO, STATIC, URGENGO, URGENGO, 3, 4, 5, 6])
    p.flags = rng.randint(0, 15) if p.kind == URGENGO else 0
    b = Batch(seed=seed, scenario_begin=rng.randint(0, 50), scenario_count=rng.choice([1, 3, 7, 33, 64]),
              horizon_ns=rng.choice([150, 400]) * MS, ftight_permille=rng.choice([0, 400]))
    both(w, p, b, f"pk seed {seed}")


def test_packed_equals_unpacked_large_batch(monkeypatch):
    """configs[4]'s workload, 5001 scenarios (throughput build): the packed and the one-scenario-
    per-warp kernels give identical records and aggregates."""
    cfg = get_config("scaleout")
    w, p = cfg.workload(), cfg.policies["urgengo"]
    b = Batch(seed=cfg.batch.seed, scenario_count=5001, horizon_ns=150 * MS, ftight_permille=400)
    r1, a1 = gpu_run(w, p, b)
    monkeypatch.setenv("URG_PACK", "0")
    r2, a2 = gpu_run(w, p, b)
    assert np.array_equal(r1, r2) and np.array_equal(a1, a2)
    o = O.run(w, p, Batch(seed=b.seed, scenario_begin=5000, scenario_count=1, horizon_ns=b.horizon_ns,
                          ftight_permille=400))
    assert np.array_equal(o.records[0], r1[5000])


def test_cpu_cores_fixtures():
    from workloads import w7
    for cores in (0, 1, 2):
        for kind in (FIFO, STATIC, URGENGO, 4):
            both(w7(cores), Policy(kind=kind, flags=0, sync_mode=SYNC_ASYNC, lax_threshold_ns=-1),
                 Batch(horizon_ns=2 * MS), f"w7 cores={cores} kind={kind}")


@pytest.mark.parametrize("seed", range(10))
def test_cpu_cores_random(seed):
    rng = random.Random(14000 + seed)
    w = random_workload(rng, C=rng.choice([2, 4, 7, 13, 32]))
    w.cpu_cores = rng.choice([1, 2, 3, 8])
    p = random_policy(rng)
    p.kind = rng.choice([FIFO, STATIC, URGENGO, URGENGO, 3, 5])
    p.flags = rng.randint(0, 15) if p.kind == URGENGO else 0
    if rng.random() < 0.3:
        p.cpu_ma_window = 4
    both(w, p, Batch(seed=seed, scenario_count=rng.randint(1, 16), horizon_ns=300 * MS), f"cores seed {seed}")


@pytest.mark.parametrize("cores", [1, 2, 8])
def test_cpu_cores_paper11(cores):
    cfg = get_config("paper11")
    w = cfg.workload()
    w.cpu_cores = cores
    b = Batch(seed=cfg.batch.seed, scenario_count=6, horizon_ns=2_000 * MS, ftight_permille=400)
    for name in ("urgengo", "fifo", "static"):
        both(w, cfg.policies[name], b, f"paper11 cores={cores} {name}")


def test_contention_fixtures_and_random():
    """R30 contention slow-down: W8 hand-worked cases, random workloads, configs[1]."""
    from workloads import w8
    for alpha in (0, 600, 2000):
        for kind in (FIFO, URGENGO):
            both(w8(alpha), Policy(kind=kind, flags=0, sync_mode=SYNC_ASYNC, lax_threshold_ns=-1),
                 Batch(horizon_ns=1 * MS), f"w8 alpha={alpha}")
    rng = random.Random(15000)
    for i in range(6):
        w = random_workload(rng, C=rng.choice([2, 5, 11, 32]))
        w.contention_permille = rng.choice([100, 600, 3000])
        p = random_policy(rng)
        both(w, p, Batch(seed=i, scenario_count=rng.randint(1, 12), horizon_ns=300 * MS), f"contention {i}")
    cfg = get_config("paper11")
    w = cfg.workload()
    w.contention_permille = 500
    both(w, cfg.policies["urgengo"], Batch(seed=cfg.batch.seed, scenario_count=6, horizon_ns=2_000 * MS,
                                           ftight_permille=400), "paper11 contention")


@pytest.mark.parametrize("wpc", ["1", "3", "16"])
def test_results_independent_of_geometry(wpc, monkeypatch):
    """Dynamic scenario fetch: the warps-per-CTA geometry changes which warp simulates which
    scenario, never the results (records keyed by global scenario index)."""
    cfg = get_config("paper11")
    w, p = cfg.workload(), cfg.policies["urgengo"]
    b = Batch(seed=cfg.batch.seed, scenario_count=50, horizon_ns=1_000 * MS, ftight_permille=400)
    ref_r, ref_a = gpu_run(w, p, b)
    monkeypatch.setenv("URG_WARPS_PER_CTA", wpc)
    r, a = gpu_run(w, p, b)
    assert np.array_equal(r, ref_r) and np.array_equal(a, ref_a)


def test_largest_template_that_fits():
    """A template near the shared-memory budget (9000 kernel records, ~150 KB) in both builds."""
    rng = random.Random(77)
    tasks = [Task(rng.randint(0, 2 * MS), rng.randint(0, 2 * MS),
                  [Kernel(rng.randint(1000, 300_000), rng.randint(1000, 300_000), rng.choice([100, 500, 1000]))
                   for _ in range(900)]) for _ in range(10)]
    w = Workload(chains=[Chain(400 * MS, 300 * MS, 0, tasks[:5]), Chain(500 * MS, 350 * MS, 0, tasks[5:])],
                 num_prio=6, jitter_ns=0, rt_bins=2048)
    p = Policy(kind=URGENGO, flags=7, sync_mode=SYNC_OVERLAP, lax_threshold_ns=5 * MS)
    both(w, p, Batch(seed=3, scenario_count=5, horizon_ns=900 * MS), "big template")
    import os as _os
    _os.environ["URG_WIDE"] = "1"
    try:
        both(w, p, Batch(seed=3, scenario_count=5, horizon_ns=900 * MS), "big template wide")
    finally:
        del _os.environ["URG_WIDE"]


def _with_copies(w, h2d_ns=300 * US, d2h_ns=100 * US):
    """Every task starts with an H2D memcpy and ends with a D2H memcpy (R31), in every template variant."""
    from paper_2509_12207_b200.sweep import with_copies
    return with_copies(w, h2d_ns, d2h_ns)


def test_copy_engine():
    """R31 memcpy on the copy engine: W9, random workloads, configs[1] with H2D/D2H copies,
    also together with cudaFree and shared CPU cores."""
    from workloads import w9
    for copies in (True, False):
        for kind in (FIFO, STATIC, URGENGO, 5):
            both(w9(copies), Policy(kind=kind, flags=0, sync_mode=SYNC_ASYNC, lax_threshold_ns=-1),
                 Batch(horizon_ns=1 * MS), f"w9 {copies} {kind}")
    rng = random.Random(16000)
    for i in range(6):
        w = random_workload(rng, C=rng.choice([2, 5, 11, 32]))
        for ch in w.chains:
            for t in ch.tasks:
                for k in t.kernels:
                    k.flags = 1 if rng.random() < 0.3 else 0
        p = random_policy(rng)
        both(w, p, Batch(seed=i, scenario_count=rng.randint(1, 12), horizon_ns=300 * MS), f"copies {i}")
    cfg = get_config("paper11")
    w = _with_copies(cfg.workload())
    b = Batch(seed=cfg.batch.seed, scenario_count=6, horizon_ns=2_000 * MS, ftight_permille=400)
    for name in ("urgengo", "fifo"):
        both(w, cfg.policies[name], b, f"paper11 copies {name}")
    w.cpu_cores = 2
    w.chains[0].tasks[0].frees = True
    both(w, cfg.policies["urgengo"], b, "paper11 copies + cores + free")


def test_binding_rejects_bad_buffers():
    """urg.py refuses buffers the kernel would overrun or misread: wrong dtype, size,
    layout or device of agg / records, before any launch."""
    import torch

    from paper_2509_12207_b200.urg import DeviceWorkload
    w, p = w1(), Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC)
    b = Batch(horizon_ns=1 * MS, scenario_count=4)
    with DeviceWorkload(w) as dw:
        good = torch.zeros(dw.agg_words, dtype=torch.int64, device="cuda")
        rec = torch.zeros((4, 2, 8), dtype=torch.int32, device="cuda")
        for bad in (good.to(torch.int32), good[:-1], good.cpu(), torch.zeros(2 * dw.agg_words, dtype=torch.int64,
                                                                             device="cuda")[::2]):
            with pytest.raises(ValueError):
                dw.simulate(p, b, bad, rec)
        for bad in (rec[:3], rec.to(torch.int64), rec.cpu(), rec.transpose(0, 1)):
            with pytest.raises(ValueError):
                dw.simulate(p, b, good, bad)
        dw.simulate(p, b, good, rec)
        dw.check()
        with pytest.raises(ValueError):
            dw.simulate_host(p, b, np.zeros(dw.agg_words, np.int32))
        with pytest.raises(ValueError):
            dw.simulate_host(p, b, np.zeros(dw.agg_words, np.int64), np.zeros((3, 2, 8), np.uint32))
