"""Invariants, special-case reductions and brute-force enumeration for the oracle.

* Invariants (R16-R21) are checked on
  the oracle's event trace of random multi-chain workloads.
* Reductions: cases where two configurations must coincide exactly (SURVEY.md
  §8(c) "Reductions" (a)-(e)).
* Brute force (T1): every feasible GPU dispatch sequence of tiny two/three-chain
  inputs is enumerated; the oracle's schedule must be in the set, must be the
  member a greedy (level, ready, chain) decision tree selects, and its miss
  count must lie within the set's range.
"""
import itertools
import random

import numpy as np
import pytest

from oracle import oracle as O
from workloads.spec import (F_BIND, F_DELAY, F_EARLY_EXIT, FIFO, MS, STATIC, SYNC_ASYNC, SYNC_BATCHED,
                            SYNC_EACH, SYNC_OVERLAP, URGENGO, US, Batch, Chain, Kernel, Policy, Task,
                            Workload)

K = O.TRACE_CODES


def random_workload(rng, C=None, jitter=0, tables=False):
    C = C or rng.randint(2, 6)
    chains = []
    for c in range(C):
        P = rng.choice([20, 30, 50, 70]) * MS
        D = rng.choice([10, 20, 40, 60]) * MS
        tasks = []
        for _ in range(rng.randint(1, 3)):
            ks = [Kernel(rng.randint(10 * US, 2 * MS), rng.randint(10 * US, 2 * MS), rng.choice([50, 200, 400, 700, 1000]))
                  for _ in range(rng.randint(1, 8))]
            cpu = rng.choice([0, rng.randint(100 * US, 3 * MS)])
            tasks.append(Task(cpu, rng.choice([cpu, rng.randint(0, 3 * MS)]), ks))
        chains.append(Chain(P, D, rng.randint(0, 5 * MS), tasks))
    return Workload(chains=chains, num_prio=rng.choice([1, 2, 3, 6]), launch_ns=rng.choice([0, 5 * US, 21_672]),
                    launch_akb_ns=rng.choice([0, 500]), sync_lo_ns=10 * US, sync_hi_ns=rng.choice([10 * US, 200 * US]),
                    jitter_ns=jitter, rt_bins=64, rt_bin_ns=1 * MS)


def random_policy(rng):
    return Policy(kind=rng.choice([FIFO, STATIC, URGENGO]), flags=rng.randint(0, 7),
                  sync_mode=rng.choice([SYNC_ASYNC, SYNC_EACH, SYNC_BATCHED, SYNC_OVERLAP]),
                  delta_eval_ns=rng.choice([100 * US, 500 * US, 2 * MS]), lax_threshold_ns=rng.choice([-1, 2 * MS, 8 * MS]),
                  sleep_ns=rng.choice([1 * MS, 300 * US]), util_exempt_permille=100)


def check_trace_invariants(w, p, b, r):
    """Per-event invariants over one scenario's trace."""
    utils = [[k.util_permille for t in ch.tasks for k in t.kernels] for ch in w.chains]
    Ns = [len(u) for u in utils]
    tr = r.trace
    last_t = -1
    enq, disp, ret = {}, {}, {}
    used = 0
    steps = 0
    for t, kind, c, i, a, bb in tr:
        t, kind, c, i, a, bb = map(int, (t, kind, c, i, a, bb))
        if kind == K["STEP"]:
            assert t > last_t, "simulation clock must increase strictly between steps"
            last_t = t
            steps += 1
            continue
        assert t == last_t
        key = (c, i, a)
        if kind == K["ENQUEUE"]:
            assert key not in enq, "each kernel launched at most once"
            enq[key] = (t, bb)
            assert 0 <= bb < max(w.num_prio, 1)
        elif kind == K["DISPATCH"]:
            assert key in enq and enq[key][0] <= t, "no kernel starts before its launch"
            if a > 0 and (c, i, a - 1) in enq:
                assert (c, i, a - 1) in ret and ret[(c, i, a - 1)] <= t, "stream predecessor finished"
            assert key not in disp
            disp[key] = (t, bb)
            used += utils[c][a]
            assert used <= 1000, "capacity"
        elif kind == K["RETIRE"]:
            assert key in disp and disp[key][1] == t, "non-preemptive: ends exactly start + d"
            ret[key] = t
            used -= utils[c][a]
        elif kind == K["BIND"]:
            if p.kind == FIFO:
                assert a == w.num_prio - 1
        elif kind == K["INST_DONE"]:
            for k in range(Ns[c]):
                assert (c, i, k) in ret, "completed instance: every kernel completed"
    # per-stream FIFO completion order
    for (c, i, k), t in ret.items():
        if k > 0:
            assert ret[(c, i, k - 1)] <= t
    assert steps == r.steps
    assert len(enq) == r.launches


@pytest.mark.parametrize("seed", range(40))
def test_random_invariants(seed):
    rng = random.Random(seed)
    w = random_workload(rng)
    p = random_policy(rng)
    b = Batch(seed=seed, horizon_ns=rng.choice([50, 150, 300]) * MS)
    r = O.run(w, p, b, trace_cap=2_000_000)
    assert len(r.trace) < 2_000_000
    check_trace_invariants(w, p, b, r)
    rec = r.records[0].astype(np.int64)
    assert (rec[:, 1] <= rec[:, 0]).all() and (rec[:, 2] + rec[:, 3] <= rec[:, 1]).all()
    # admitted arrivals (jitter 0): #{i >= 0 : O + i P < H}
    for c, ch in enumerate(w.chains):
        n = 0 if ch.offset_ns >= b.horizon_ns else -(-(b.horizon_ns - ch.offset_ns) // ch.period_ns)
        assert rec[c, 0] == n
    # determinism
    r2 = O.run(w, p, b, trace_cap=2_000_000)
    assert np.array_equal(r.records, r2.records) and np.array_equal(r.trace, r2.trace)


def test_delay_and_binding_rules_in_trace():
    """Delay only for non-exempt kernels while another chain holds a truly urgent
    active kernel and the launcher itself is not urgent; a
    truly urgent task is bound to level 0."""
    rng = random.Random(77)
    checked_delay = checked_bind = 0
    for trial in range(30):
        w = random_workload(rng, C=rng.randint(2, 5))
        p = Policy(kind=URGENGO, flags=F_BIND | F_DELAY, sync_mode=rng.choice([SYNC_ASYNC, SYNC_OVERLAP]),
                   lax_threshold_ns=rng.choice([5 * MS, 15 * MS]))
        r = O.run(w, p, Batch(seed=trial, horizon_ns=200 * MS), trace_cap=2_000_000)
        utils = [[k.util_permille for t in ch.tasks for k in t.kernels] for ch in w.chains]
        akb = [0] * w.num_chains      # active kernels per chain, from ENQUEUE / SYNC_RET
        launched = [0] * w.num_chains
        L = [0] * w.num_chains
        snapL, snapA = list(L), list(akb)
        last_eval = {}
        for t, kind, c, i, a, bb in r.trace:
            t, kind, c, i, a, bb = map(int, (t, kind, c, i, a, bb))
            if kind == K["STEP"]:
                snapL, snapA = list(L), list(akb)
            elif kind == K["EVAL"]:
                L[c] = a
                last_eval[c] = a
            elif kind == K["ENQUEUE"]:
                akb[c] += 1
                launched[c] = a + 1
            elif kind == K["INST_START"]:
                launched[c] = 0
            elif kind == K["EARLY_EXIT"]:
                akb[c] = 0
            elif kind == K["SYNC_RET"]:
                akb[c] = launched[c] - a          # covered kernels leave the AKB
            elif kind == K["DELAY"]:
                own = last_eval[c]
                assert utils[c][a] >= 100 and not (0 <= own <= p.lax_threshold_ns)
                assert any(snapA[o] > 0 and 0 <= snapL[o] <= p.lax_threshold_ns for o in range(w.num_chains) if o != c)
                checked_delay += 1
            elif kind == K["BIND"]:
                own = last_eval[c]
                if 0 <= own <= p.lax_threshold_ns:
                    assert a == 0
                    checked_bind += 1
                else:
                    assert a >= 1 or w.num_prio == 1
    assert checked_delay > 0 and checked_bind > 0


def _ul_rank_key(L, chain):
    """Sort key: most urgent first by UL = 1/L (L = 0 saturates to +inf),
    ties by the smaller chain id.  Exact rationals -- no laxity key trick."""
    from fractions import Fraction
    ul = Fraction(10**30) if L == 0 else Fraction(1, L)
    return (-ul, chain)


def _normalised_level(r, n_r, num_prio):
    """R15 written from PAPER.md:466 "normalize these rankings to the range (1, NUM_PRI-1)" and
    SPEC.md:402-404 (n_r = 4: rank 1 -> 1, rank 4 -> 5; n_r = 1 -> the middle level)."""
    if num_prio <= 2:
        return num_prio - 1
    if n_r == 1:
        return 1 + (num_prio - 2) // 2
    return 1 + ((r - 1) * (num_prio - 2)) // (n_r - 1)


@pytest.mark.parametrize("seed", range(12))
def test_binding_level_exact_in_trace(seed):
    """Every UrgenGo binding (R15) replayed from the trace with NUM_PRI in {3, 4, 6, 8}: an urgent
    task takes level 0; any other ranks among itself and the chains AKB-active in the Phase B
    snapshot by the exact 1/L order, and takes the normalised level recomputed here."""
    rng = random.Random(4242 + seed)
    checked = {0: 0, 1: 0}
    for trial in range(6):
        w = random_workload(rng, C=rng.randint(3, 7))
        w.num_prio = rng.choice([3, 4, 6, 8])
        p = Policy(kind=URGENGO, flags=F_BIND | rng.choice([0, F_DELAY]), sync_mode=rng.choice([SYNC_ASYNC, SYNC_OVERLAP]),
                   lax_threshold_ns=rng.choice([1 * MS, 5 * MS, 15 * MS]))
        r = O.run(w, p, Batch(seed=trial, horizon_ns=200 * MS), trace_cap=2_000_000)
        akb = [0] * w.num_chains
        launched = [0] * w.num_chains
        L = [0] * w.num_chains
        snapL, snapA = list(L), list(akb)
        for t, kind, c, i, a, bb in r.trace:
            t, kind, c, i, a, bb = map(int, (t, kind, c, i, a, bb))
            if kind == K["STEP"]:
                snapL, snapA = list(L), list(akb)
            elif kind == K["EVAL"]:
                L[c] = a
            elif kind == K["ENQUEUE"]:
                akb[c] += 1
                launched[c] = a + 1
            elif kind == K["INST_START"]:
                launched[c] = 0
            elif kind == K["EARLY_EXIT"]:
                akb[c] = 0
            elif kind == K["SYNC_RET"]:
                akb[c] = launched[c] - a
            elif kind == K["BIND"]:
                own = L[c]                       # the EVAL of this launch attempt
                if 0 <= own <= p.lax_threshold_ns:
                    assert a == 0
                    checked[0] += 1
                    continue
                members = [(own, c)] + [(snapL[o], o) for o in range(w.num_chains) if o != c and snapA[o] > 0]
                order = sorted(members, key=lambda m: _ul_rank_key(*m))
                rnk = 1 + [m[1] for m in order].index(c)
                assert a == _normalised_level(rnk, len(members), w.num_prio), (t, c, rnk, len(members))
                checked[1] += 1
    assert checked[1] > 20


def _records(w, p, b):
    return O.run(w, p, b).records


@pytest.mark.parametrize("seed", range(15))
def test_reductions(seed):
    rng = random.Random(1000 + seed)
    w = random_workload(rng)
    w.launch_akb_ns = 0
    b = Batch(seed=seed, horizon_ns=200 * MS)
    # (a) UrgenGo with binding, delay and early exit off, ASYNC, lambda_akb = 0 == FIFO, trace-equal
    fifo = Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC)
    off = Policy(kind=URGENGO, flags=0, sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * MS)
    ra, rb = O.run(w, fifo, b, trace_cap=10**6), O.run(w, off, b, trace_cap=10**6)
    drop = {K["EVAL"]}
    ta = np.array([r for r in ra.trace if r[1] not in drop])
    tb = np.array([r for r in rb.trace if r[1] not in drop])
    assert np.array_equal(ta, tb) and np.array_equal(ra.records, rb.records)
    # (b) BATCHED / OVERLAP with Delta_eval >= every task's estimated total == ASYNC
    for mode in (SYNC_BATCHED, SYNC_OVERLAP):
        big = Policy(kind=URGENGO, flags=F_BIND, sync_mode=mode, delta_eval_ns=10**12, lax_threshold_ns=5 * MS)
        asy = Policy(kind=URGENGO, flags=F_BIND, sync_mode=SYNC_ASYNC, lax_threshold_ns=5 * MS)
        assert np.array_equal(_records(w, big, b), _records(w, asy, b))
    # (c) NUM_PRI = 1: binding is a no-op
    w1p = random_workload(random.Random(1000 + seed))
    w1p.num_prio = 1
    for mode in (SYNC_ASYNC, SYNC_OVERLAP):
        on = Policy(kind=URGENGO, flags=F_BIND | F_DELAY, sync_mode=mode, lax_threshold_ns=5 * MS)
        nob = Policy(kind=URGENGO, flags=F_DELAY, sync_mode=mode, lax_threshold_ns=5 * MS)
        assert np.array_equal(_records(w1p, on, b), _records(w1p, nob, b))
    # (e) L_th < 0 (never urgent): delay is a no-op
    for mode in (SYNC_ASYNC, SYNC_OVERLAP):
        d = Policy(kind=URGENGO, flags=F_BIND | F_DELAY, sync_mode=mode, lax_threshold_ns=-1)
        nd = Policy(kind=URGENGO, flags=F_BIND, sync_mode=mode, lax_threshold_ns=-1)
        assert np.array_equal(_records(w, d, b), _records(w, nd, b))


@pytest.mark.parametrize("seed", range(8))
def test_single_server_when_all_util_full(seed):
    """(d) u = 1000 for every kernel: the GPU is a single non-preemptive server."""
    rng = random.Random(500 + seed)
    w = random_workload(rng)
    for ch in w.chains:
        for t in ch.tasks:
            for k in t.kernels:
                k.util_permille = 1000
    r = O.run(w, random_policy(rng), Batch(seed=seed, horizon_ns=150 * MS), trace_cap=10**6)
    running = 0
    for t, kind, c, i, a, bb in r.trace:
        if kind == K["DISPATCH"]:
            running += 1
            assert running == 1
        elif kind == K["RETIRE"]:
            running -= 1


# ---------------------------------------------------------------------------
# T1: brute-force enumeration of dispatch sequences on tiny inputs
# ---------------------------------------------------------------------------

def enumerate_schedules(enq_t, durs, utils):
    """All feasible non-preemptive dispatch sequences.  Chain c's kernels are all
    on its stream from enq_t[c] (lambda = 0, ASYNC); at every event time any
    subset of waiting heads that fits the remaining capacity may start."""
    C = len(durs)
    out = []

    def rec(t, nxt, run_end, prev_end, sched):
        # retire
        run_end = list(run_end)
        for c in range(C):
            if run_end[c] is not None and run_end[c] == t:
                prev_end[c] = t
                run_end[c] = None
                nxt[c] += 1
        if all(nxt[c] == len(durs[c]) for c in range(C)):
            out.append((tuple(sorted(sched)), tuple(prev_end)))
            return
        used = sum(utils[c][nxt[c]] for c in range(C) if run_end[c] is not None)
        waiting = [c for c in range(C) if run_end[c] is None and nxt[c] < len(durs[c]) and enq_t[c] <= t]
        for r_ in range(len(waiting) + 1):
            for S in itertools.combinations(waiting, r_):
                if used + sum(utils[c][nxt[c]] for c in S) > 1000:
                    continue
                re = list(run_end)
                for c in S:
                    re[c] = t + durs[c][nxt[c]]
                future = [e for e in re if e is not None] + [e for e in enq_t if e > t]
                if not future:
                    continue        # idles forever with work left: not a schedule
                # a subset that leaves a startable head idle while nothing will ever change is pruned above;
                # otherwise advance to the next event
                rec(min(future), list(nxt), re, list(prev_end), sched + [(t, c, nxt[c]) for c in S])

    rec(min(enq_t), [0] * C, [None] * C, [0] * C, [])
    return out


def greedy_walk(enq_t, durs, utils, levels):
    """The member of the schedule tree picked by (level, ready, chain) greedy admission (R20)."""
    C = len(durs)
    t = min(enq_t)
    nxt, run_end, prev_end = [0] * C, [None] * C, [0] * C
    ready = [None] * C
    sched = []
    while True:
        for c in range(C):
            if run_end[c] is not None and run_end[c] == t:
                prev_end[c] = t; run_end[c] = None; nxt[c] += 1
                ready[c] = t if nxt[c] < len(durs[c]) else None
            if ready[c] is None and nxt[c] == 0 and enq_t[c] <= t:
                ready[c] = enq_t[c]
        if all(nxt[c] == len(durs[c]) for c in range(C)):
            return tuple(sorted(sched)), tuple(prev_end)
        used = sum(utils[c][nxt[c]] for c in range(C) if run_end[c] is not None)
        waiting = sorted((levels[c], ready[c], c) for c in range(C)
                         if run_end[c] is None and nxt[c] < len(durs[c]) and enq_t[c] <= t)
        for _, _, c in waiting:
            if used + utils[c][nxt[c]] <= 1000:
                used += utils[c][nxt[c]]
                run_end[c] = t + durs[c][nxt[c]]
                sched.append((t, c, nxt[c]))
        t = min([e for e in run_end if e is not None] + [e for e in enq_t if e > t])


@pytest.mark.parametrize("seed", range(60))
def test_bruteforce_tiny(seed):
    rng = random.Random(seed)
    C = rng.choice([2, 2, 3])
    durs = [[rng.choice([1, 2, 3]) * MS for _ in range(rng.randint(1, 3))] for _ in range(C)]
    utils = [[rng.choice([400, 700, 1000]) for _ in d] for d in durs]
    cpu = [rng.choice([0, 1, 2]) * MS for _ in range(C)]
    Ds = [rng.choice([3, 5, 8]) * MS for _ in range(C)]
    chains = [Chain(1000 * MS, Ds[c], 0, [Task(cpu[c], cpu[c], [Kernel(d, d, u) for d, u in zip(durs[c], utils[c])])])
              for c in range(C)]
    w = Workload(chains=chains, num_prio=rng.choice([2, 3]), launch_ns=0, launch_akb_ns=0, sync_lo_ns=0,
                 sync_hi_ns=0, jitter_ns=0)
    space = enumerate_schedules(cpu, durs, utils)
    assert space
    for p in [Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC),
              Policy(kind=STATIC, flags=0, sync_mode=SYNC_ASYNC),
              Policy(kind=URGENGO, flags=F_BIND, sync_mode=SYNC_ASYNC, lax_threshold_ns=rng.choice([-1, 2 * MS]))]:
        r = O.run(w, p, Batch(horizon_ns=500 * MS), trace_cap=10_000)
        sched = tuple(sorted((int(t), int(c), int(a)) for t, k, c, i, a, b in r.trace if k == K["DISPATCH"]))
        levels = {}
        for t, k, c, i, a, b in r.trace:
            if k == K["BIND"]:
                levels[int(c)] = int(a)
        fin = [None] * C
        for t, k, c, i, a, b in r.trace:
            if k == K["INST_DONE"]:
                fin[int(c)] = int(t)
        members = {s for s, _ in space}
        assert sched in members                                        # (1) feasible
        g_sched, g_fin = greedy_walk(cpu, durs, utils, [levels[c] for c in range(C)])
        assert sched == g_sched and tuple(fin) == g_fin                # (2)/(3) decision-tree member
        misses = int(r.records[0, :, 1].sum())
        all_miss = [sum(1 for c in range(C) if f[c] > Ds[c]) for _, f in space]
        assert min(all_miss) <= misses <= max(all_miss)                # (4)
        if p.kind == FIFO:
            assert all(v == w.num_prio - 1 for v in levels.values())


def _replay_collisions(w, lth, trace):
    """Independent recount of DESIGN.md R24 from the event trace: snapshot of (stream busy,
    level, last laxity) at the start of each Phase B, checked at every enqueue of an urgent
    chain.  Returns the histogram by number of colliding tasks."""
    C = w.num_chains
    busy, level, lax = [0] * C, [0] * C, [0] * C
    snap = None
    hist = np.zeros(33, np.int64)

    def key(L):
        return (1 << 63) if L == 0 else ((1 << 62) - L if L > 0 else -(1 << 62) - L)

    for t, kind, c, i, a, bb in trace:
        kind, c, a, bb = int(kind), int(c), int(a), int(bb)
        if kind == K["STEP"]:
            snap = None
            continue
        if kind == K["RETIRE"]:
            busy[c] -= 1
            continue
        if snap is None:
            snap = (list(busy), list(level), list(lax))
        if kind == K["EVAL"]:
            lax[c] = a
        elif kind == K["BIND"]:
            level[c] = a
        elif kind == K["ENQUEUE"]:
            busy[c] += 1
            if 0 <= lax[c] <= lth:
                sb, sl, sL = snap
                k = sum(1 for o in range(C) if o != c and sb[o] > 0 and sl[o] <= level[c] and key(sL[o]) < key(lax[c]))
                if k:
                    hist[min(k + 1, 32)] += 1
    return hist


@pytest.mark.parametrize("seed", range(12))
def test_collision_histogram_replayed_from_trace(seed):
    from workloads.spec import F_COLLISIONS, collision_hist
    rng = random.Random(1000 + seed)
    w = random_workload(rng, C=rng.randint(2, 6))
    p = random_policy(rng)
    p.kind = URGENGO
    p.lax_threshold_ns = rng.choice([2 * MS, 8 * MS, 30 * MS])
    p.flags = rng.randint(0, 7) | F_COLLISIONS
    b = Batch(seed=seed, scenario_count=1, horizon_ns=400 * MS)
    r = O.run(w, p, b, trace_cap=400_000)
    assert len(r.trace) < 400_000
    got = collision_hist(r.agg, w.num_chains, w.rt_bins)
    want = _replay_collisions(w, p.lax_threshold_ns, r.trace)
    assert got.tolist() == want.tolist()
    plain = O.run(w, Policy(kind=p.kind, flags=p.flags & 7, sync_mode=p.sync_mode, delta_eval_ns=p.delta_eval_ns,
                            lax_threshold_ns=p.lax_threshold_ns, sleep_ns=p.sleep_ns), b)
    assert np.array_equal(plain.records, r.records)   # a metric: the schedule is unchanged


def _norm_level(r, n_r, num_prio):
    if num_prio <= 2:
        return num_prio - 1
    if n_r <= 1:
        return 1 + (num_prio - 2) // 2
    return 1 + ((r - 1) * (num_prio - 2)) // (n_r - 1)


def _replay_classical_binds(w, kind, trace):
    """Recompute every BIND level of a classical policy (R27) from the trace: the rank
    of the binding chain among itself and the chains with active kernels at the round snapshot,
    keyed by the chains' arrival, remaining estimated work and utilisation."""
    from tests.test_oracle_pins import _brute_rank
    C = w.num_chains
    est = [[k.estimate_ns for t in ch.tasks for k in t.kernels] for ch in w.chains]
    cpu = [[t.cpu_estimate_ns for t in ch.tasks] for ch in w.chains]
    ends = [np.cumsum([len(t.kernels) for t in ch.tasks]).tolist() for ch in w.chains]
    G = [sum(e) for e in est]
    launched, cpu_idx, akb, tarr = [0] * C, [0] * C, [0] * C, [0] * C
    snap, checked = None, 0

    def R(c):
        return sum(est[c][launched[c]:]) + sum(cpu[c][cpu_idx[c]:])

    for t, kind_, c, i, a, bb in trace:
        k, c, a, bb, t = int(kind_), int(c), int(a), int(bb), int(t)
        if k == K["STEP"]:
            snap = None
            continue
        if k == K["RETIRE"]:
            continue
        if snap is None:
            snap = [(akb[o] > 0, tarr[o], R(o)) for o in range(C)]
        if k == K["INST_START"]:
            launched[c], cpu_idx[c], akb[c], tarr[c] = 0, 0, 0, a
        elif k == K["ENQUEUE"]:
            launched[c] = a + 1
            akb[c] += 1
            if launched[c] in ends[c]:
                cpu_idx[c] = ends[c].index(launched[c]) + 1
        elif k == K["SYNC_RET"]:
            akb[c] = launched[c] - a
        elif k == K["BIND"]:
            members = [o for o in range(C) if o == c or snap[o][0]]
            ta = [tarr[o] if o == c else snap[o][1] for o in members]
            RR = [R(c) if o == c else snap[o][2] for o in members]
            D = [w._Dp[o] for o in members]
            Pp = [w._Pp[o] for o in members]
            GG = [G[o] for o in members]
            # ties break by chain id: members are in chain order, so list index order = id order
            r = _brute_rank(kind, ta, D, RR, GG, Pp, members.index(c), t)
            assert a == _norm_level(r, len(members), w.num_prio), (t, c, a, r, len(members))
            checked += 1
    return checked


@pytest.mark.parametrize("kind", [3, 4, 5, 6])
@pytest.mark.parametrize("seed", range(4))
def test_classical_binding_replayed_from_trace(kind, seed):
    rng = random.Random(300 + 10 * kind + seed)
    w = random_workload(rng, C=rng.randint(2, 6))
    w.num_prio = rng.choice([3, 4, 6])
    w.jitter_ns = 0
    p = random_policy(rng)
    p.kind = kind
    b = Batch(seed=seed, scenario_count=1, horizon_ns=300 * MS)
    r = O.run(w, p, b, trace_cap=500_000)
    assert len(r.trace) < 500_000
    w._Dp = [ch.deadline_ns for ch in w.chains]       # f_d = 1, no tight set
    w._Pp = [ch.period_ns for ch in w.chains]         # f_a = 1
    assert _replay_classical_binds(w, kind, r.trace) > 0


@pytest.mark.parametrize("kind", [3, 4, 5, 6])
def test_classical_single_chain_is_fifo(kind):
    """With one chain nothing contends, so every policy gives FIFO's records."""
    rng = random.Random(kind)
    w = random_workload(rng, C=1)
    b = Batch(seed=1, scenario_count=3, horizon_ns=300 * MS)
    base = Policy(kind=FIFO, flags=0, sync_mode=SYNC_OVERLAP)
    a = O.run(w, base, b)
    c = O.run(w, Policy(kind=kind, flags=0, sync_mode=SYNC_OVERLAP), b)
    assert np.array_equal(a.records, c.records)


@pytest.mark.parametrize("seed", range(10))
def test_cudafree_barrier_invariants(seed):
    """R28 on random workloads with cudaFree tasks: while a request is pending or served no
    kernel starts; a request is served only when no kernel runs; a served request returns
    exactly free_ns later; requests are served in (request time, chain) order."""
    rng = random.Random(4000 + seed)
    w = random_workload(rng, C=rng.randint(2, 6))
    for ch in w.chains:
        for t in ch.tasks:
            t.frees = rng.random() < 0.4
    w.free_ns = rng.choice([50 * US, 188 * US, 2 * MS])
    p = random_policy(rng)
    r = O.run(w, p, Batch(seed=seed, scenario_count=1, horizon_ns=300 * MS), trace_cap=400_000)
    pending, serving, running = {}, None, set()
    served = []
    for t, k, c, i, a, bb in r.trace:
        t, k, c, i, a = int(t), int(k), int(c), int(i), int(a)
        name = O.TRACE_KINDS[k]
        if name == "FREE_CALL":
            pending[c] = t
        elif name == "FREE_START":
            assert not running, "a cudaFree is served only on an idle device"
            assert serving is None
            head = min(pending, key=lambda x: (pending[x], x))
            assert c == head, "requests are served in (time, chain) order"
            assert a == t + w.free_ns
            serving = (c, a)
            del pending[c]
            served.append(c)
        elif name == "FREE_RET":
            assert serving is not None and serving == (c, t)
            serving = None
        elif name == "DISPATCH":
            assert not pending and serving is None, "no kernel starts during a barrier"
            running.add((c, i, a))
        elif name == "RETIRE":
            running.discard((c, i, a))
    assert r.records[0][:, 0].sum() > 0


@pytest.mark.parametrize("seed", range(10))
def test_cpu_cores_invariants(seed):
    """R29 on random workloads: never more than K jobs hold a core, a preempted job keeps exactly
    its unfinished work, FIFO (equal priorities) never preempts, and K >= C cores reproduce the
    one-core-per-thread model exactly."""
    rng = random.Random(6000 + seed)
    w = random_workload(rng, C=rng.randint(2, 6))
    p = random_policy(rng)
    b = Batch(seed=seed, scenario_count=1, horizon_ns=300 * MS)
    base = O.run(w, p, b)
    w.cpu_cores = w.num_chains
    assert np.array_equal(O.run(w, p, b).records, base.records)
    K = rng.choice([1, 2])
    w.cpu_cores = K
    r = O.run(w, p, b, trace_cap=400_000)
    running, last_t = {}, None
    for t, k, c, i, a, bb in r.trace:
        t, k, c, a = int(t), int(k), int(c), int(a)
        if t != last_t:                                  # the core count holds between instants
            assert len(running) <= K
            last_t = t
        for x in [x for x, (st, rem) in running.items() if st + rem <= t]:
            del running[x]                               # completed jobs release their core
        name = O.TRACE_KINDS[k]
        if name == "CPU_RUN":
            assert c not in running
            running[c] = (t, a)
        elif name == "CPU_STOP":
            assert p.kind != FIFO, "equal priorities never preempt"
            st, rem = running.pop(c)
            assert a == rem - (t - st) and a > 0
    assert len(running) <= K
    assert r.records[:, :, 0].sum() > 0


@pytest.mark.parametrize("seed", range(8))
def test_contention_durations_replayed(seed):
    """R30: every kernel's run time is its contention-free duration d plus
    floor(d * alpha * U_run / 10^6), U_run the utilisation already running at its start
    (d taken from the alpha = 0 run of the same scenario: durations are keyed by chain,
    instance and kernel, not by the schedule)."""
    rng = random.Random(8000 + seed)
    w = random_workload(rng, C=rng.randint(2, 6))
    p = random_policy(rng)
    b = Batch(seed=seed, scenario_count=1, horizon_ns=300 * MS)
    base = O.run(w, p, b, trace_cap=400_000)
    d0 = {(int(c), int(i), int(a)): int(bb) - int(t) for t, k, c, i, a, bb in base.trace if k == K["DISPATCH"]}
    w.contention_permille = rng.choice([100, 600, 3000])
    r = O.run(w, p, b, trace_cap=400_000)
    util = {c: [k.util_permille for tk in ch.tasks for k in tk.kernels] for c, ch in enumerate(w.chains)}
    running, checked = {}, 0
    for t, k, c, i, a, bb in r.trace:
        t, k, c, i, a, bb = int(t), int(k), int(c), int(i), int(a), int(bb)
        if k == K["RETIRE"]:
            running.pop((c, i, a))
        elif k == K["DISPATCH"]:
            u_run = sum(running.values())
            if (c, i, a) in d0:
                d = d0[(c, i, a)]
                assert bb - t == d + d * w.contention_permille * u_run // 1_000_000
                checked += 1
            running[(c, i, a)] = util[c][a]
    assert checked > 0


@pytest.mark.parametrize("seed", range(8))
def test_copy_engine_invariants(seed):
    """R31 on random workloads with memcpy operations: at most one memcpy runs at any time,
    memcpys do not count against the compute capacity, and a memcpy starts only when the
    engine is free, in (ready time, chain) order among the waiting memcpy heads."""
    rng = random.Random(9000 + seed)
    w = random_workload(rng, C=rng.randint(2, 6))
    for ch in w.chains:
        for t in ch.tasks:
            for k in t.kernels:
                k.flags = 1 if rng.random() < 0.3 else 0
    p = random_policy(rng)
    r = O.run(w, p, Batch(seed=seed, scenario_count=1, horizon_ns=300 * MS), trace_cap=400_000)
    kinds = {c: [k.flags & 1 for t in ch.tasks for k in t.kernels] for c, ch in enumerate(w.chains)}
    util = {c: [k.util_permille for t in ch.tasks for k in t.kernels] for c, ch in enumerate(w.chains)}
    copy_run, used, n_copy = None, 0, 0
    for t, k, c, i, a, bb in r.trace:
        t, k, c, i, a = int(t), int(k), int(c), int(i), int(a)
        name = O.TRACE_KINDS[k]
        if name == "DISPATCH":
            if kinds[c][a]:
                assert copy_run is None, "one memcpy at a time"
                copy_run = (c, i, a)
                n_copy += 1
            else:
                used += util[c][a]
                assert used <= 1000
        elif name == "RETIRE":
            if kinds[c][a]:
                assert copy_run == (c, i, a)
                copy_run = None
            else:
                used -= util[c][a]
    assert n_copy > 0


def test_oracle_is_not_limited_to_a_warp():
    """The oracle's chain limit is its own (64, its scratch arrays), not the GPU path's 32 lanes: a
    40-chain workload simulates under three policies with every trace invariant and every arrival
    admitted; 65 chains are rejected."""
    rng = random.Random(5)
    w = random_workload(rng, C=40)
    for p in (Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC),
              Policy(kind=URGENGO, flags=F_BIND | F_DELAY, sync_mode=SYNC_OVERLAP, lax_threshold_ns=5 * MS),
              Policy(kind=STATIC, flags=0, sync_mode=SYNC_EACH)):
        b = Batch(seed=11, horizon_ns=100 * MS, ftight_permille=400)
        r = O.run(w, p, b, trace_cap=2_000_000)
        check_trace_invariants(w, p, b, r)
        assert r.records.shape[1] == 40
        for c, ch in enumerate(w.chains):
            n = 0 if ch.offset_ns >= b.horizon_ns else -(-(b.horizon_ns - ch.offset_ns) // ch.period_ns)
            assert r.records[0, c, 0] == n
    w.chains = w.chains + w.chains[:25]
    with pytest.raises(ValueError):
        O.run(w, Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC), Batch(horizon_ns=10 * MS))
