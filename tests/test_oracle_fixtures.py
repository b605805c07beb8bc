"""The oracle against hand-worked timelines (tests/golden/w*.json) and single-chain
closed forms.  The expected values were derived by hand from the paper's
mechanisms (DESIGN.md Model M0), not by running any simulator."""
import json
import os
import random

import numpy as np
import pytest

from oracle import oracle as O
from workloads import w1, w2, w3
from workloads.spec import (US, FIFO, MS, REC_EARLY, REC_LAUNCH, REC_MISS, REC_SUMRT_HI, REC_SUMRT_LO,
                            REC_TOTAL, SYNC_ASYNC, SYNC_BATCHED, SYNC_EACH, SYNC_OVERLAP, URGENGO,
                            F_EARLY_EXIT, Batch, Chain, Kernel, Policy, Task, Workload)

from .conftest import GOLDEN


def _gold(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _sum_rt(rec):
    return int(rec[REC_SUMRT_LO]) | (int(rec[REC_SUMRT_HI]) << 32)


@pytest.mark.parametrize("case", _gold("w1.json")["cases"], ids=lambda c: c["policy"])
def test_w1_two_chain_timelines(case):
    p = Policy(kind=case["kind"], flags=case["flags"], sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * MS)
    r = O.run(w1(), p, Batch(horizon_ns=1 * MS))
    rec = r.records[0]
    for c in range(2):
        assert rec[c, REC_TOTAL] == 1
        assert _sum_rt(rec[c]) == int(round(case["rt_ms"][c] * MS))
        assert rec[c, REC_MISS] == case["miss"][c]
    eq3 = O.overall_miss_ratio(rec[:, REC_MISS], rec[:, REC_TOTAL])
    assert eq3 == case["eq3"]
    assert r.launches == case["launches"]


def test_w1_laxities_in_trace():
    """The EVAL trace entries carry Eq. 2 laxities 2 ms / 4 ms (chain A at t = 1 ms) and 92 ms (B at 1.5 ms)."""
    g = _gold("w1.json")["laxities_ms"]
    p = Policy(kind=URGENGO, flags=3, sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * MS)
    r = O.run(w1(), p, Batch(horizon_ns=1 * MS), trace_cap=1000)
    ev = [(int(t), int(c), int(a)) for t, k, c, i, a, b in r.trace if k == O.TRACE_CODES["EVAL"]]
    assert (1 * MS, 0, int(g["A_attempt_k0_t1"] * MS)) in ev
    assert (1 * MS, 0, int(g["A_attempt_k1_t1"] * MS)) in ev
    assert (1_500_000, 1, int(g["B_attempt_k0_t1.5"] * MS)) in ev


@pytest.mark.parametrize("mode", ["ASYNC", "OVERLAP", "BATCHED", "EACH"])
def test_w2_sync_modes(mode):
    g = _gold("w2.json")
    p = Policy(kind=URGENGO, flags=0, sync_mode=g["sync_mode"][mode], lax_threshold_ns=-1)
    r = O.run(w2(), p, Batch(horizon_ns=1 * MS))
    assert _sum_rt(r.records[0, 0]) == int(round(g["rt_ms"][mode] * MS))
    assert r.launches == 8


def test_w3_early_exit():
    g = _gold("w3.json")
    r = O.run(w3(), Policy(kind=URGENGO, flags=F_EARLY_EXIT, sync_mode=SYNC_ASYNC), Batch(horizon_ns=1 * MS),
              trace_cap=200)
    e = g["urgengo_early_exit"]
    rec = r.records[0, 0]
    assert (rec[REC_TOTAL], rec[REC_MISS], rec[REC_EARLY], rec[REC_LAUNCH]) == (e["total"], e["miss"], e["early"],
                                                                               e["launches"])
    evals = [int(a) for t, k, c, i, a, b in r.trace if k == O.TRACE_CODES["TASK_START"] or k == O.TRACE_CODES["EVAL"]]
    assert int(e["L_task0_ms"] * MS) in evals and int(e["L_task1_ms"] * MS) in evals
    f = g["fifo"]
    r = O.run(w3(), Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC), Batch(horizon_ns=1 * MS))
    rec = r.records[0, 0]
    assert (rec[REC_TOTAL], rec[REC_MISS], rec[REC_EARLY], rec[REC_LAUNCH]) == (f["total"], f["miss"], f["early"],
                                                                               f["launches"])
    assert _sum_rt(rec) == int(round(f["rt_ms"] * MS))


# ---------------------------------------------------------------------------
# Single-chain closed form (max-plus recurrence), independent of the event loop
# ---------------------------------------------------------------------------

def closed_form_rt(tasks, lam, sigma, mode, delta):
    """Response time of one instance of one chain running alone (no contention).

    Per task: CPU segment, then launches of lam each; kernel k becomes available at
    e_k (end of its launch call); it starts at max(e_k, f_{k-1}) and ends f_k = start + d_k.
    A synchronisation called at c waiting for kernels < j returns at max(c, f_{j-1}) + sigma.
    (R16-R17.)"""
    t = 0
    f_prev = 0          # completion of the previous kernel on the stream
    for cpu, kernels in tasks:
        t += cpu
        first_close = True
        acc = 0
        f = []          # completion times of this task's kernels
        batch_start = 0
        for k, (d, est) in enumerate(kernels):
            t += lam                            # launch call
            start = max(t, f_prev)
            f_prev = start + d
            f.append(f_prev)
            last = k == len(kernels) - 1
            if mode == SYNC_EACH or (mode == SYNC_ASYNC and last):
                t = max(t, f[k]) + sigma
                continue
            if mode == SYNC_BATCHED:
                acc += est
                if acc >= delta or last:
                    acc = 0
                    t = max(t, f[k]) + sigma
                continue
            if mode == SYNC_OVERLAP:
                acc += est
                if last:
                    t = max(t, f[k]) + sigma
                elif acc >= delta:
                    acc = 0
                    if batch_start > 0:
                        t = max(t, f[batch_start - 1]) + sigma
                    batch_start = k + 1
    return t


@pytest.mark.parametrize("mode", [SYNC_ASYNC, SYNC_EACH, SYNC_BATCHED, SYNC_OVERLAP])
def test_single_chain_closed_form(mode):
    rng = random.Random(100 + mode)
    for trial in range(60):
        ntask = rng.randint(1, 3)
        tasks, spec = [], []
        for _ in range(ntask):
            cpu = rng.choice([0, rng.randint(1, 3 * MS)])
            ks = []
            for _ in range(rng.randint(1, 12)):
                d = rng.randint(1, 400_000)
                est = rng.choice([d, rng.randint(1, 400_000)])
                ks.append((d, est))
            tasks.append((cpu, ks))
            spec.append(Task(cpu, cpu, [Kernel(d, e, rng.choice([50, 400, 1000])) for d, e in ks]))
        lam = rng.choice([0, 1000, 21_672, 200_000])
        sigma = rng.choice([0, 10_000, 50_000])
        delta = rng.choice([1, 300_000, 500_000, 10**9])
        w = Workload(chains=[Chain(10_000 * MS, 5_000 * MS, 0, spec)], launch_ns=lam, launch_akb_ns=0,
                     sync_lo_ns=sigma, sync_hi_ns=sigma, jitter_ns=0)
        expect = closed_form_rt(tasks, lam, sigma, mode, delta)
        # policy independence of a lone chain with lambda_akb = 0
        for kind, flags in [(FIFO, 0), (1, 0), (URGENGO, 1), (URGENGO, 3)]:
            p = Policy(kind=kind, flags=flags, sync_mode=mode, delta_eval_ns=delta, lax_threshold_ns=MS)
            r = O.run(w, p, Batch(horizon_ns=1))
            assert _sum_rt(r.records[0, 0]) == expect, (trial, kind, flags)


@pytest.mark.parametrize("case", _gold("w4.json")["cases"], ids=lambda c: c["policy"])
def test_w4_kernel_collisions(case):
    """Collision histogram and response times of the hand-worked W4 (R24)."""
    from workloads import w4
    from workloads.spec import collision_hist
    w = w4()
    p = Policy(kind=case["kind"], flags=case["flags"], sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * MS)
    r = O.run(w, p, Batch(horizon_ns=1 * MS))
    h = collision_hist(r.agg, w.num_chains, w.rt_bins)
    want = np.zeros_like(h)
    for k, v in case["hist"].items():
        want[int(k)] = v
    assert h.tolist() == want.tolist()
    for c in range(3):
        assert _sum_rt(r.records[0][c]) == int(round(case["rt_ms"][c] * MS))
        assert r.records[0][c, REC_MISS] == case["miss"][c]


def test_collisions_need_concurrency():
    """A single chain never collides (SPEC.md:580 'no concurrent execution -> all-zero histogram'),
    and the metric does not change the schedule (records identical with and without it)."""
    from workloads import w3
    from workloads.spec import F_COLLISIONS, collision_hist
    w = w3()
    for lth in (-1, 10 * MS):
        a = O.run(w, Policy(kind=URGENGO, flags=7 | F_COLLISIONS, sync_mode=SYNC_ASYNC, lax_threshold_ns=lth),
                  Batch(horizon_ns=1 * MS))
        b = O.run(w, Policy(kind=URGENGO, flags=7, sync_mode=SYNC_ASYNC, lax_threshold_ns=lth), Batch(horizon_ns=1 * MS))
        assert not collision_hist(a.agg, 1, w.rt_bins).any()
        assert np.array_equal(a.records, b.records)


def test_calibration_samples_w1():
    """TH_urgent sampling (Q5) on W1 with H = 20 ms, threshold disabled.
    Hand-derived: no AKB entry at 0 ms; A holds entries with last laxity 4 ms (its k1 attempt at
    t = 1 ms) from 1 ms until its final sync returns at 10 ms, and is always more urgent than B
    (92 ms) -> one 4 ms sample at each of 1..9 ms; nothing after.  A 5 ms window keeps 1..4 ms."""
    p = Policy(kind=URGENGO, flags=7, sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * MS)
    s = O.calibration_samples(w1(), p, Batch(horizon_ns=20 * MS))
    assert s[0].tolist() == [4 * MS] * 9
    assert O.calibration_samples(w1(), p, Batch(horizon_ns=20 * MS), window_ns=5 * MS)[0].tolist() == [4 * MS] * 4
    assert O.calibrate(w1(), p, Batch(horizon_ns=20 * MS)) == (4 * MS, 9)


def test_calibration_skips_negative_laxity_w3():
    """W3 with the threshold disabled: the only AKB entry (k0, t = 1..2.8 ms) has laxity
    4.5 - 2 - 2 - 1 = -0.5 ms < 0, so every sample is skipped (SPEC.md:328 'negatives
    excluded') and the calibration has no threshold (-1)."""
    p = Policy(kind=URGENGO, flags=7, sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * MS)
    assert O.calibration_samples(w3(), p, Batch(horizon_ns=20 * MS))[0].tolist() == []
    assert O.calibrate(w3(), p, Batch(horizon_ns=20 * MS)) == (-1, 0)


def test_calibration_pools_scenarios():
    """A batch's threshold is the nearest-rank percentile of all its scenarios' samples."""
    from workloads import get_config
    cfg = get_config("paper11")
    b = Batch(seed=cfg.batch.seed, scenario_begin=3, scenario_count=3, horizon_ns=2_000 * MS, ftight_permille=400)
    p = cfg.policies["urgengo"]
    per = O.calibration_samples(cfg.workload(), p, b)
    assert all(len(x) > 0 for x in per)
    lth, n = O.calibrate(cfg.workload(), p, b)
    assert n == sum(len(x) for x in per)
    assert lth == O.nearest_rank_lth(np.concatenate(per))


def _evals(r, chain):
    return [(int(t), int(a)) for t, k, c, i, a, b in r.trace if k == O.TRACE_CODES["EVAL"] and c == chain]


@pytest.mark.parametrize("eps", [1, 300, 500])
def test_noise_w1_laxities(eps):
    """R25: during task tau of instance i the remaining estimated work R of
    Eq. 2 is scaled by (1000 + n)/1000, n = (w mod (2 eps + 1)) - eps, w the Philox word
    (tag 6, chain, instance, tau) -- drawn here with the KAT-pinned Philox primitive.  W1's
    chain A at t = 1 ms: R = 4 + 1 = 5 ms (k0 attempt) and 2 + 1 = 3 ms (k1 attempt)."""
    b = Batch(seed=77, horizon_ns=1 * MS)
    p = Policy(kind=URGENGO, flags=0, sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * MS, noise_permille=eps)
    r = O.run(w1(), p, b, trace_cap=1000)
    w = int(O.philox([0, (6 << 24) | (0 << 16), 0, 0], [b.seed & 0xFFFFFFFF, b.seed >> 32])[0])
    n = w % (2 * eps + 1) - eps
    want = [(0, 8 * MS - (5 * MS * (1000 + n)) // 1000),            # task start, R = 4 + 1 ms
            (1 * MS, 8 * MS - (5 * MS * (1000 + n)) // 1000 - 1 * MS),
            (1 * MS, 8 * MS - (3 * MS * (1000 + n)) // 1000 - 1 * MS)]
    assert _evals(r, 0)[:3] == want


def test_noise_zero_is_exact_eq2():
    from workloads import get_config
    cfg = get_config("paper11")
    b = Batch(seed=cfg.batch.seed, scenario_count=2, horizon_ns=1_000 * MS, ftight_permille=400)
    p = cfg.policies["urgengo"]
    a = O.run(cfg.workload(), p, b)
    q = Policy(**{**p.__dict__, "noise_permille": 0})
    assert np.array_equal(O.run(cfg.workload(), q, b).records, a.records)


def test_cpu_predictor_moving_average():
    """R26: one chain, CPU segment actually 1 ms but profiled at 5 ms.  Instance 0
    uses the profiled 5 ms (no measurement yet): L(task start) = 50 - 2 - 5 = 43 ms.  Instance 1
    (t_arr = 100 ms) uses the mean of the one measurement, 1 ms: L = 150 - 2 - 1 - 100 = 47 ms.
    Without the predictor both instances use 5 ms (43 ms)."""
    ch = Chain(100 * MS, 50 * MS, 0, [Task(1 * MS, 5 * MS, [Kernel(2 * MS, 2 * MS, 1000)])])
    w = Workload(chains=[ch], num_prio=6, launch_ns=0, launch_akb_ns=0, sync_lo_ns=0, sync_hi_ns=0, jitter_ns=0)
    b = Batch(horizon_ns=150 * MS)
    on = O.run(w, Policy(kind=URGENGO, flags=0, sync_mode=SYNC_ASYNC, cpu_ma_window=8), b, trace_cap=1000)
    off = O.run(w, Policy(kind=URGENGO, flags=0, sync_mode=SYNC_ASYNC), b, trace_cap=1000)
    assert (0, 43 * MS) in _evals(on, 0) and (100 * MS, 47 * MS) in _evals(on, 0)
    assert (100 * MS, 43 * MS) in _evals(off, 0)


@pytest.mark.parametrize("W", [1, 3, 8])
def test_cpu_predictor_replayed_from_trace(W):
    """R26 recomputed independently from the trace: measured CPU durations are the gaps between
    a task start and the chain's next evaluation (its launch attempt, lambda aside); the estimate
    of instance i is the floor mean of the last min(W, h) measurements of earlier instances."""
    from workloads.quantiles import inst_z_table
    ch = Chain(20 * MS, 40 * MS, 0, [Task(3 * MS, 3 * MS, [Kernel(1 * MS, 1 * MS, 500)])], cpu_sigma_ppm=300_000)
    w = Workload(chains=[ch], num_prio=6, launch_ns=0, launch_akb_ns=0, sync_lo_ns=0, sync_hi_ns=0, jitter_ns=0,
                 inst_quantiles_q16=inst_z_table())
    r = O.run(w, Policy(kind=URGENGO, flags=0, sync_mode=SYNC_ASYNC, cpu_ma_window=W),
              Batch(seed=5, horizon_ns=400 * MS), trace_cap=10000)
    ev = _evals(r, 0)
    starts = [int(t) for t, k, c, i, a, b in r.trace if k == O.TRACE_CODES["TASK_START"]]
    hist = []
    for i, ts in enumerate(starts):
        pred = 3 * MS if not hist else sum(hist[-W:]) // len(hist[-W:])
        t_arr = i * 20 * MS
        assert (ts, t_arr + 40 * MS - 1 * MS - pred - ts) in ev, i
        nxt = min(t for t, a in ev if t > ts)          # the launch attempt ends the CPU segment
        hist.append(nxt - ts)


@pytest.mark.parametrize("kind", [3, 4, 5, 6])
def test_w1_classical_policies(kind):
    """W1 with NUM_PRI = 3 under EDF / SJF / HRRN / LCUF (R27).  Hand-derived: A binds
    alone at 1 ms (level 1); at 1.5 ms B ranks 2nd of {A, B} under every policy -- A's deadline
    8 < 100 ms (EDF), its remaining work 0 < 6.5 ms (SJF), infinite response ratio (HRRN) and
    utilisation 4/1000 < 5/1000 (LCUF) -- so B takes level 2; at 3 ms A1 (level 1) beats B0
    (level 2): A1 3-5 ms, B0 5-10 ms, the STATIC timeline."""
    w = w1()
    w.num_prio = 3
    r = O.run(w, Policy(kind=kind, flags=0, sync_mode=SYNC_ASYNC), Batch(horizon_ns=1 * MS))
    assert [_sum_rt(r.records[0][c]) for c in range(2)] == [5 * MS, 10 * MS]
    assert r.launches == 3


@pytest.mark.parametrize("case", _gold("w6.json")["cases"], ids=lambda c: c["name"])
def test_w6_cudafree_barrier(case):
    """R28 device barrier: hand-worked response times under every policy kind (the barrier
    does not depend on priorities here)."""
    from workloads import w6
    w = w6(case["two_chains"])
    for kind in (FIFO, URGENGO):
        r = O.run(w, Policy(kind=kind, flags=0, sync_mode=SYNC_ASYNC, lax_threshold_ns=-1), Batch(horizon_ns=1 * MS))
        assert [_sum_rt(r.records[0][c]) for c in range(w.num_chains)] == [int(round(x * MS)) for x in case["rt_ms"]]


def test_cudafree_serialises_requests():
    """Two chains each ending with cudaFree at the same time: requests are served one after
    the other in chain order, each costing free_ns once the device is idle (R28)."""
    t = Task(1 * MS, 1 * MS, [Kernel(1 * MS, 1 * MS, 400)], frees=True)
    w = Workload(chains=[Chain(1000 * MS, 100 * MS, 0, [t]), Chain(1000 * MS, 100 * MS, 0, [t])], num_prio=2,
                 launch_ns=0, launch_akb_ns=0, sync_lo_ns=0, sync_hi_ns=0, jitter_ns=0, free_ns=300 * US)
    r = O.run(w, Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC), Batch(horizon_ns=1 * MS))
    # both kernels run 1-2 ms (u 400 + 400); both frees requested at 2 ms: chain 0 served 2-2.3, chain 1 2.3-2.6
    assert [_sum_rt(r.records[0][c]) for c in range(2)] == [2_300_000, 2_600_000]


@pytest.mark.parametrize("case", _gold("w7.json")["cases"], ids=lambda c: c["name"])
def test_w7_cpu_cores(case):
    """R29: chains' threads sharing CPU cores with policy priorities (hand-derived)."""
    from workloads import w7
    w = w7(case["cores"])
    r = O.run(w, Policy(kind=case["kind"], flags=0, sync_mode=SYNC_ASYNC, lax_threshold_ns=-1), Batch(horizon_ns=2 * MS))
    assert [_sum_rt(r.records[0][c]) for c in range(2)] == [int(round(x * MS)) for x in case["rt_ms"]]


@pytest.mark.parametrize("case", _gold("w8.json")["cases"], ids=lambda c: str(c["alpha_permille"]))
def test_w8_contention(case):
    from workloads import w8
    w = w8(case["alpha_permille"])
    for kind in (FIFO, URGENGO):
        r = O.run(w, Policy(kind=kind, flags=0, sync_mode=SYNC_ASYNC, lax_threshold_ns=-1), Batch(horizon_ns=1 * MS))
        assert [_sum_rt(r.records[0][c]) for c in range(2)] == [int(round(x * MS)) for x in case["rt_ms"]]


@pytest.mark.parametrize("case", _gold("w9.json")["cases"], ids=lambda c: str(c["copies"]))
def test_w9_copy_engine(case):
    from workloads import w9
    w = w9(case["copies"])
    for kind in (FIFO, URGENGO):
        r = O.run(w, Policy(kind=kind, flags=0, sync_mode=SYNC_ASYNC, lax_threshold_ns=-1), Batch(horizon_ns=1 * MS))
        assert [_sum_rt(r.records[0][c]) for c in range(2)] == [int(round(x * MS)) for x in case["rt_ms"]]


def test_toy2_fifo_first_dispatches():
    """configs[0] (toy2) under FIFO: the first eight dispatches match the hand derivation."""
    from workloads import get_config, toy2
    g = _gold("toy2_fifo_first_dispatches.json")
    cfg = get_config("toy2")
    r = O.run(toy2(), cfg.policies["fifo"], cfg.batch, trace_cap=100_000)
    got = [[int(c), int(i), int(a), int(t), int(b)] for t, k, c, i, a, b in r.trace
           if k == O.TRACE_CODES["DISPATCH"]][:8]
    want = [[c, i, k, int(round(s * MS)), int(round(e * MS))] for c, i, k, s, e in g["dispatches"]]
    assert got == want


# ---------------------------------------------------------------------------
# W10: a zero-cost, already-satisfied OVERLAP sync (R21 same-t continuation)
# ---------------------------------------------------------------------------

def _w10_policy():
    from workloads.spec import F_DELAY
    return Policy(kind=URGENGO, flags=F_DELAY, sync_mode=SYNC_OVERLAP, delta_eval_ns=500 * US,
                  lax_threshold_ns=5 * MS, sleep_ns=1 * MS, util_exempt_permille=100)


def test_w10_zero_cost_satisfied_sync():
    """PAPER.md:504-509 with sigma = 0: A's second batch close at 1.2 ms waits for a batch that is
    already complete; the sync returns at the same t and A's next launch attempt reads the Phase B
    snapshot taken before B's kernel reached the AKB -> no delay, rt_A = 1.6 ms (the per-round
    reading of SURVEY.md:529-532 would give 3.5 ms)."""
    from workloads import w10
    g = _gold("w10.json")
    r = O.run(w10(), _w10_policy(), Batch(horizon_ns=1 * MS), trace_cap=1000)
    rec = r.records[0]
    for c in range(2):
        assert rec[c, REC_TOTAL] == 1
        assert _sum_rt(rec[c]) == int(round(g["rt_ms"][c] * MS))
        assert rec[c, REC_MISS] == g["miss"][c]
    assert r.launches == g["launches"]
    K = O.TRACE_CODES
    assert sum(1 for row in r.trace if row[1] == K["DELAY"]) == g["delays"]
    s = g["satisfied_sync"]
    t12 = int(round(s["t_ms"] * MS))
    calls = [(int(t), int(a), int(b)) for t, k, c, i, a, b in r.trace if k == K["SYNC_CALL"] and c == s["chain"]]
    assert (t12, s["target"], s["cost"]) in calls
    rets = [int(t) for t, k, c, i, a, b in r.trace if k == K["SYNC_RET"] and c == s["chain"]]
    assert t12 in rets, "the satisfied zero-cost sync returns at the call time"
    # the next launch attempt of A is evaluated at that same t (one loop step: exactly one STEP at 1.2 ms)
    assert sum(1 for row in r.trace if row[1] == K["STEP"] and row[0] == t12) == 1
    enq = [(int(t), int(a)) for t, k, c, i, a, b in r.trace if k == K["ENQUEUE"] and c == 0]
    assert enq == [(1_100_000, 0), (1_200_000, 1), (1_300_000, 2)]


# ---------------------------------------------------------------------------
# W11: UrgenGo's rank normalisation at NUM_PRI = 6 inside a simulation (R15)
# ---------------------------------------------------------------------------

def test_w11_binding_levels_num_pri_6():
    from workloads import w11
    from workloads.spec import F_BIND
    g = _gold("w11.json")
    p = Policy(kind=URGENGO, flags=F_BIND, sync_mode=SYNC_ASYNC, lax_threshold_ns=1 * MS)
    r = O.run(w11(), p, Batch(horizon_ns=10 * MS), trace_cap=1000)
    K = O.TRACE_CODES
    ev = {int(c): int(a) for t, k, c, i, a, b in r.trace if k == K["EVAL"] and int(t) == (int(c) + 1) * MS}
    assert [ev[c] for c in range(6)] == [x * MS for x in g["laxity_at_binding_ms"]]
    binds = sorted((int(c), int(a)) for t, k, c, i, a, b in r.trace if k == K["BIND"])
    assert [lv for _, lv in binds] == g["levels"]
    rec = r.records[0]
    assert [_sum_rt(rec[c]) for c in range(6)] == [x * MS for x in g["rt_ms"]]
    assert rec[:, REC_MISS].tolist() == g["miss"]
    assert O.overall_miss_ratio(rec[:, REC_MISS], rec[:, REC_TOTAL]) == g["eq3"]
    assert r.launches == g["launches"]
    # without binding every task sits at NUM_PRI - 1 and the waiting heads go in ready order
    rf = O.run(w11(), Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC), Batch(horizon_ns=10 * MS))
    assert [_sum_rt(rf.records[0, c]) for c in range(6)] == [x * MS for x in g["fifo_rt_ms"]]
