"""The debug build of the CUDA path (liburg_debug.so, -DURG_DEBUG) -- SURVEY.md §5 / DESIGN.md §5:

* a one-scenario event trace recorded on the device in the oracle's trace schema
  ("time_ns, seq, kind, chain, instance, detail"), diffed event by event against the
  CPU oracle's trace of the same scenario;
* the invariants of SPEC.md:171-174 checked on the device in every step (a kernel never starts
  before it is ready; capacity <= 1000 permille; a kernel retires exactly at its end; every kernel
  of a finished instance launched and completed once; record counts consistent; no event in the
  past; urgent tasks at level 0), reported through urg_check.

Lanes run Phase B in parallel, so the device trace interleaves lanes within a step; both traces
are compared in the canonical form: per event time, per lane, that lane's events in program order
(Phase A retire, Phase B, Phase C dispatch).  The oracle also writes rows for the extended model
(CPU cores, cudaFree, executors) that the device trace does not; the workloads here use none.
"""
import random
from collections import defaultdict
from dataclasses import replace

import numpy as np
import pytest

from oracle import oracle as O
from workloads import get_config, toy2, w1, w2, w10, w11
from workloads.spec import (F_BIND, F_DELAY, FIFO, MS, STATIC, SYNC_ASYNC, SYNC_BATCHED, SYNC_EACH, SYNC_OVERLAP,
                            URGENGO, US, Batch, Policy)

from .gpu_helpers import gpu_run
from .test_oracle_properties import random_policy, random_workload

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

K = O.TRACE_CODES
DEVICE_KINDS = {K[k] for k in ("STEP", "INST_START", "TASK_START", "EVAL", "DELAY", "BIND", "ENQUEUE", "DISPATCH",
                               "RETIRE", "SYNC_CALL", "SYNC_RET", "FREE_CLOSE", "INST_DONE", "EARLY_EXIT",
                               "COLLISION")}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2509_12207_b200.urg import lib_debug
    lib_debug()   # loud failure if liburg_debug.so is missing


def canonical(rows):
    """{(t, lane): [(kind, instance, a, b), ...] in row order} for the device kinds."""
    g = defaultdict(list)
    for t, kind, c, i, a, b in np.asarray(rows, np.int64).tolist():
        if kind in DEVICE_KINDS:
            g[(t, c)].append((kind, i, a, b))
    return g


def diff_traces(o_rows, g_rows, ctx):
    o, g = canonical(o_rows), canonical(g_rows)
    keys = sorted(set(o) | set(g))
    for k in keys:
        if o.get(k) != g.get(k):
            names = {v: n for n, v in K.items()}
            fmt = lambda evs: [(names[e[0]],) + e[1:] for e in (evs or [])]   # noqa: E731
            raise AssertionError(f"{ctx}: trace differs at (t, lane) = {k}:\n oracle {fmt(o.get(k))}\n device "
                                 f"{fmt(g.get(k))}")
    assert sum(len(v) for v in o.values()) == sum(len(v) for v in g.values())
    return sum(len(v) for v in o.values())


def _env(build, monkeypatch):
    if build == "512":
        monkeypatch.setenv("URG_SMALL", "0")
    elif build == "packed":
        monkeypatch.setenv("URG_WIDE", "1")
    elif build == "wide":
        monkeypatch.setenv("URG_WIDE", "1")
        monkeypatch.setenv("URG_PACK", "0")
    elif build == "ext":
        monkeypatch.setenv("URG_EXT", "1")


def device_trace(w, p, b, scenario):
    from paper_2509_12207_b200.urg import DeviceWorkload
    with DeviceWorkload(w, debug=True) as dw:
        rows, agg = dw.trace(p, b, scenario)
    return rows, agg


def check_scenario(w, p, b, scenario, ctx):
    o = O.run(w, p, replace(b, scenario_begin=scenario, scenario_count=1), trace_cap=4_000_000)
    assert len(o.trace) < 4_000_000
    rows, _ = device_trace(w, p, b, scenario)
    n = diff_traces(o.trace, rows, ctx)
    assert n > 0
    return n


BUILDS = ["small", "512", "packed", "wide", "ext"]


@pytest.mark.parametrize("build", BUILDS)
def test_trace_fixtures(build, monkeypatch):
    _env(build, monkeypatch)
    cnt = 2 if build in ("packed", "wide") else 1
    for kind, flags in ((FIFO, 0), (STATIC, 0), (URGENGO, 1), (URGENGO, 2), (URGENGO, 3)):
        p = Policy(kind=kind, flags=flags, sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * MS)
        check_scenario(w1(), p, Batch(horizon_ns=1 * MS, scenario_count=cnt), 0, f"w1 {kind}/{flags} {build}")
    for mode in (SYNC_ASYNC, SYNC_EACH, SYNC_BATCHED, SYNC_OVERLAP):
        p = Policy(kind=URGENGO, flags=0, sync_mode=mode, lax_threshold_ns=-1)
        check_scenario(w2(), p, Batch(horizon_ns=1 * MS, scenario_count=cnt), 0, f"w2 {mode} {build}")
    p = Policy(kind=URGENGO, flags=F_DELAY, sync_mode=SYNC_OVERLAP, delta_eval_ns=500 * US, lax_threshold_ns=5 * MS)
    check_scenario(w10(), p, Batch(horizon_ns=1 * MS, scenario_count=cnt), 0, f"w10 {build}")
    p = Policy(kind=URGENGO, flags=F_BIND, sync_mode=SYNC_ASYNC, lax_threshold_ns=1 * MS)
    check_scenario(w11(), p, Batch(horizon_ns=10 * MS, scenario_count=cnt), 0, f"w11 {build}")


@pytest.mark.parametrize("mode", [SYNC_ASYNC, SYNC_EACH, SYNC_BATCHED, SYNC_OVERLAP])
def test_trace_toy2_every_policy(mode):
    cfg = get_config("toy2")
    pols = [Policy(kind=FIFO, flags=0, sync_mode=mode), Policy(kind=STATIC, flags=0, sync_mode=mode)]
    pols += [Policy(kind=URGENGO, flags=f, sync_mode=mode, lax_threshold_ns=10 * MS) for f in range(16)]
    for p in pols:
        check_scenario(toy2(), p, cfg.batch, 0, f"toy2 {p.kind}/{p.flags}/{mode}")


@pytest.mark.parametrize("seed", range(12))
def test_trace_random_workloads(seed, monkeypatch):
    rng = random.Random(9000 + seed)
    build = BUILDS[seed % len(BUILDS)]
    _env(build, monkeypatch)
    w = random_workload(rng, C=rng.choice([2, 3, 5, 8, 11]), jitter=rng.choice([0, 3 * MS]))
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
    p.flags |= rng.choice([0, 8])        # the collision metric rows too
    b = Batch(seed=seed, scenario_begin=rng.randint(0, 100), scenario_count=6, horizon_ns=200 * MS,
              ftight_permille=rng.choice([0, 400]))
    check_scenario(w, p, b, b.scenario_begin + rng.randint(0, 5), f"random {seed} {build}")


@pytest.mark.parametrize("name,pol", [("paper11", "urgengo"), ("paper11", "fifo"), ("jitter", "urgengo")])
def test_trace_paper_workloads(name, pol, monkeypatch):
    """One scenario of the paper-shaped workloads (64 template variants, heavy tails), 400 ms
    horizon, in the throughput build with two scenarios per warp and in the latency build."""
    cfg = get_config(name)
    w, p = cfg.workload(), cfg.policies[pol]
    b = replace(cfg.batch, scenario_begin=9973, scenario_count=40, horizon_ns=400 * MS)
    n1 = check_scenario(w, p, b, 9973 + 17, f"{name} {pol} latency")
    monkeypatch.setenv("URG_WIDE", "1")
    n2 = check_scenario(w, p, b, 9973 + 17, f"{name} {pol} packed")
    assert n1 == n2 > 1000


@pytest.mark.parametrize("build", BUILDS)
def test_device_invariants_hold(build, monkeypatch):
    """The debug build checks the SPEC.md:171-174 invariants at every step; no trip on random
    workloads and on paper11 / jitter batches, and its records equal the product build's."""
    from paper_2509_12207_b200.urg import DeviceWorkload
    _env(build, monkeypatch)
    rng = random.Random(31 + BUILDS.index(build))
    cases = []
    for _ in range(6):
        w = random_workload(rng, C=rng.choice([2, 5, 11]), jitter=rng.choice([0, 3 * MS]))
        cases.append((w, random_policy(rng), Batch(seed=rng.randint(0, 99), scenario_count=64, horizon_ns=300 * MS)))
    for name in ("paper11", "jitter"):
        cfg = get_config(name)
        cases.append((cfg.workload(), cfg.policies["urgengo"], replace(cfg.batch, scenario_count=300,
                                                                       horizon_ns=1_000 * MS)))
    for w, p, b in cases:
        r0, a0 = gpu_run(w, p, b)
        with DeviceWorkload(w, debug=True) as dw:
            agg = torch.zeros(dw.agg_words, dtype=torch.int64, device="cuda")
            rec = torch.zeros((b.scenario_count, w.num_chains, 8), dtype=torch.int32, device="cuda")
            dw.simulate(p, b, agg, rec)
            dw.check()
            dw.check()          # the error word is clear after a report (and stays clear)
        assert np.array_equal(rec.cpu().numpy().view(np.uint32), r0) and np.array_equal(agg.cpu().numpy(), a0)
