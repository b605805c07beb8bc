"""Pins of the oracle's per-task executors (R32; "each task is executed
by a dedicated thread").

The pin is a closed-form recurrence written here from the rule, not from the oracle: with one
chain, FIFO launching, asynchronous launches, constant times and kernels small enough never to
wait for GPU capacity, every stage j is a server with a constant service time

    S_j = end of its last kernel + sigma,   kernel m enqueued at c_j + (m+1) * lambda,
                                            started at max(enqueue, end of kernel m-1),

stage 0 starts instance i at max(arrival_i, end of instance i-1), and stage j > 0, when it
frees at f, takes the newest message published strictly before f (a subscription of depth 1:
a newer message replaces an untaken one; a message published exactly at f is delivered at
the end of the round in which the stage frees, so an older one is taken first), else waits
for the next message.  The last stage records its instances in order; skipped instances are
misses with the early-exit marker in the hash.
"""
import numpy as np
import pytest

from oracle import oracle as O
from workloads.spec import (EXEC_CHAIN, EXEC_TASK, FIFO, REC_EARLY, REC_HASH, REC_LAUNCH, REC_MISS, REC_SUMRT_HI,
                            REC_SUMRT_LO, REC_TOTAL, REC_UNFIN, SYNC_ASYNC, Batch, Chain, Kernel, Policy, Task,
                            Workload)

FNV = 16777619


def fold(h, x):
    return ((h ^ (x & 0xFFFFFFFF)) * FNV) & 0xFFFFFFFF


def service_time(cpu, kern, lam, sigma):
    t_enq, end = cpu, 0
    for d in kern:
        t_enq += lam
        end = max(t_enq, end) + d
    return max(t_enq, end) + sigma, [cpu + (m + 1) * lam for m in range(len(kern))]


def pipeline(stages, period, offset, deadline, horizon, lam, sigma):
    """Expected record of the single chain (closed-form recurrence, see module docstring)."""
    H_stop = horizon + deadline
    S, enq = zip(*[service_time(c, k, lam, sigma) for c, k in stages])
    launches = 0
    # stage 0: admitted arrivals, serial server
    pub, f = [], 0
    i = 0
    while offset + i * period < horizon:
        st = max(offset + i * period, f)
        if st > H_stop:
            break
        launches += sum(1 for e in enq[0] if st + e <= H_stop)
        f = st + S[0]
        if f <= H_stop:
            pub.append((f, i))
        i += 1
    taken = []   # (instance, start, end) of the last stage processed so far
    for j in range(1, len(stages)):
        out, f, last, k = [], 0, -1, 0
        taken = []
        while True:
            avail = [(p, i) for p, i in pub if i > last and p < f]
            if avail:
                p, i = max(avail, key=lambda x: x[1])
                st = f
            else:
                nxt = [(p, i) for p, i in pub if i > last]
                if not nxt:
                    break
                p, i = nxt[0]
                st = p
            if st > H_stop:
                break
            launches += sum(1 for e in enq[j] if st + e <= H_stop)
            end = st + S[j]
            taken.append((i, st, end))
            last, f = i, end
            if end <= H_stop:
                out.append((end, i))
            else:
                break
        pub = out
    if len(stages) == 1:
        taken = [(i, None, p) for p, i in pub]
    # last stage: records in instance order
    h, miss, sum_rt, expect = 2166136261, 0, 0, 0
    for i, st, end in taken:
        for _ in range(expect, i):
            h = fold(fold(h, 0xFFFFFFFF), 0xFFFFFFFF)
            miss += 1
        expect = i
        if end <= H_stop:
            rt = end - (offset + i * period)
            miss += rt > deadline
            sum_rt += rt
            h = fold(fold(h, rt), rt >> 32)
            expect = i + 1
    admitted = 0
    while offset + admitted * period < horizon:
        admitted += 1
    unfin = admitted - expect
    return dict(total=admitted, miss=miss + unfin, early=0, unfin=unfin, launches=launches, hash=h, sum_rt=sum_rt)


def workload(stages, period, offset, deadline, lam, sigma, executors=EXEC_TASK):
    tasks = [Task(c, c, [Kernel(d, d, 300) for d in k]) for c, k in stages]
    return Workload(chains=[Chain(period, deadline, offset, tasks)], num_prio=1, launch_ns=lam, launch_akb_ns=0,
                    sync_lo_ns=sigma, sync_hi_ns=sigma, jitter_ns=0, rt_bins=64, rt_bin_ns=1_000_000,
                    executors=executors)


CASES = [
    # (stages [(cpu, [kernel durations])], period, offset, deadline, horizon, lambda, sigma)
    ([(1_000, [3_000, 2_000]), (2_000, [4_000])], 20_000, 500, 60_000, 400_000, 700, 300),       # pure pipeline
    ([(1_000, [3_000]), (2_000, [15_000, 9_000])], 10_000, 0, 80_000, 500_000, 1_000, 500),      # slow 2nd stage: drops
    ([(500, [2_000]), (500, [30_000]), (1_000, [5_000])], 7_000, 123, 90_000, 700_000, 250, 0),  # 3 stages, drops
    ([(1_000, [1_000]), (1_000, [1_000])], 4_000, 0, 20_000, 100_000, 1_000, 0),                 # ties: S0 = S1 = P
    ([(1_000, [9_000]), (1_000, [9_000])], 5_000, 0, 40_000, 200_000, 500, 500),                 # both stages slow
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_pipeline_recurrence(case):
    stages, period, offset, deadline, horizon, lam, sigma = CASES[case]
    want = pipeline(stages, period, offset, deadline, horizon, lam, sigma)
    w = workload(stages, period, offset, deadline, lam, sigma)
    r = O.run(w, Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC), Batch(horizon_ns=horizon))
    rec = r.records[0, 0]
    got = dict(total=int(rec[REC_TOTAL]), miss=int(rec[REC_MISS]), early=int(rec[REC_EARLY]),
               unfin=int(rec[REC_UNFIN]), launches=int(rec[REC_LAUNCH]), hash=int(rec[REC_HASH]),
               sum_rt=int(rec[REC_SUMRT_LO]) | (int(rec[REC_SUMRT_HI]) << 32))
    assert got == want


def test_cases_exercise_drops_and_pipelining():
    """The recurrence cases are not degenerate: some skip instances, some overlap stages."""
    drops = []
    for stages, period, offset, deadline, horizon, lam, sigma in CASES:
        want = pipeline(stages, period, offset, deadline, horizon, lam, sigma)
        drops.append(want["miss"] - want["unfin"])
        S = [service_time(c, k, lam, sigma)[0] for c, k in stages]
        assert sum(S) > period or want["total"] > 1
    assert max(drops) > 0 and min(drops) == 0


def test_single_task_chains_equal_chain_threads():
    """With one task per chain, a per-task executor is the chain's thread (R32 reduces to R6)."""
    from workloads import paper11
    from workloads.spec import URGENGO
    w = paper11()
    for ch in w.chains:
        ch.tasks = ch.tasks[:1]
    b = Batch(seed=3, scenario_count=4, horizon_ns=300_000_000)
    for p in (Policy(), Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC)):
        a = O.run(w, p, b)
        w.executors = EXEC_TASK
        t = O.run(w, p, b)
        w.executors = EXEC_CHAIN
        assert np.array_equal(a.records, t.records)
        assert np.array_equal(a.agg, t.agg)
    assert Policy().kind == URGENGO


def test_paper11_task_executors_invariants():
    """paper11 under per-task executors: record identities, launches never exceed the chain-mode
    bound of kernels per admitted instance, and every stage thread ran."""
    from workloads import paper11
    w = paper11()
    w.executors = EXEC_TASK
    b = Batch(seed=5, scenario_count=3, horizon_ns=1_000_000_000)
    r = O.run(w, Policy(), b, trace_cap=2_000_000)
    rec = r.records.astype(np.int64)
    assert (rec[..., REC_MISS] <= rec[..., REC_TOTAL]).all()
    assert (rec[..., REC_UNFIN] <= rec[..., REC_MISS]).all()
    kern = np.array([sum(len(t.kernels) for t in ch.tasks) for ch in w.chains])
    assert (rec[..., REC_LAUNCH] <= rec[..., REC_TOTAL] * kern[None, :]).all()
    tr = O.run(w, Policy(), Batch(seed=5, scenario_count=1, horizon_ns=1_000_000_000), trace_cap=2_000_000).trace
    pub, take = O.TRACE_CODES["PUBLISH"], O.TRACE_CODES["TAKE"]
    assert (tr[:, 1] == pub).sum() > 0 and (tr[:, 1] == take).sum() > 0
    # a take never precedes the publication of the same instance by the previous stage
    first_pub = {}
    for t, k, c, i, _, _ in tr:
        if k == pub:
            first_pub.setdefault((c + 1, i), t)
    for t, k, c, i, _, _ in tr:
        if k == take:
            assert (c, i) in first_pub and first_pub[(c, i)] <= t


def test_rejects_predictor_and_too_many_threads():
    from workloads import paper11
    w = paper11()
    w.executors = EXEC_TASK
    with pytest.raises(ValueError):
        O.run(w, Policy(cpu_ma_window=4), Batch())
    w.chains = w.chains * 3              # 33 chains, 66 tasks > the oracle's 64 threads
    with pytest.raises(ValueError):
        O.run(w, Policy(), Batch())
