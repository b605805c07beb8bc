"""Pins of template variants (R33; SURVEY.md §8(d) cfg 2 "64 templates, scenario s uses
template s mod 64") in the oracle: the definition written out -- scenario s of a V-variant workload
is scenario s of the one-template workload whose kernels are set s mod V."""
import copy

import numpy as np

from oracle import oracle as O
from workloads import paper11_variants, toy2
from workloads.spec import FIFO, SYNC_ASYNC, Batch, Policy


def _as_single(w, v):
    """The one-template workload whose kernels are variant v of w."""
    w1 = copy.deepcopy(w)
    if v:
        recs = iter(w.kernel_variants[v - 1])
        for ch in w1.chains:
            for t in ch.tasks:
                t.kernels = [copy.copy(next(recs)) for _ in t.kernels]
    w1.kernel_variants = None
    return w1


def test_scenario_uses_variant_s_mod_v():
    w = paper11_variants(5)
    p = Policy()
    b = Batch(seed=11, scenario_begin=7, scenario_count=6, horizon_ns=400_000_000, ftight_permille=400)
    got = O.run(w, p, b).records
    for j in range(b.scenario_count):
        s = b.scenario_begin + j
        one = O.run(_as_single(w, s % 5), p, Batch(seed=11, scenario_begin=s, scenario_count=1,
                                                   horizon_ns=b.horizon_ns, ftight_permille=400)).records[0]
        assert np.array_equal(got[j], one), s


def test_identical_variants_equal_one_template():
    w = toy2()
    n = w.total_kernels()
    flat = [k for ch in w.chains for t in ch.tasks for k in t.kernels]
    assert len(flat) == n
    wv = copy.deepcopy(w)
    wv.kernel_variants = [copy.deepcopy(flat) for _ in range(3)]
    b = Batch(seed=2, scenario_count=8, horizon_ns=1_000_000_000)
    for p in (Policy(lax_threshold_ns=10_000_000), Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC)):
        a, v = O.run(w, p, b), O.run(wv, p, b)
        assert np.array_equal(a.records, v.records) and np.array_equal(a.agg, v.agg)


def test_variants_differ_and_keep_structure():
    """The 64 paper11 templates share chains, task totals and kernel counts, not kernel durations."""
    w = paper11_variants(64)
    n = w.total_kernels()
    base = [k for ch in w.chains for t in ch.tasks for k in t.kernels]
    assert w.num_variants == 64 and all(len(v) == n for v in w.kernel_variants)
    sums0 = []
    i = 0
    for ch in w.chains:
        for t in ch.tasks:
            sums0.append(sum(k.nominal_ns for k in base[i:i + len(t.kernels)]))
            i += len(t.kernels)
    for v in w.kernel_variants[:8]:
        i, sums = 0, []
        for ch in w.chains:
            for t in ch.tasks:
                sums.append(sum(k.nominal_ns for k in v[i:i + len(t.kernels)]))
                i += len(t.kernels)
        assert sums == sums0                                   # per-task totals of Table 2 / Table 4
        assert [k.nominal_ns for k in v] != [k.nominal_ns for k in base]
