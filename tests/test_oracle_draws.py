"""Pins of the oracle's scenario initialisation and random draws (R3-R5), read back
from its event trace:

* R3 factors (§6.2): P' = P / f_a, D' = D * f_d, the tight
  subset halved, ceil(f_tight * C) chains -- SPEC.md's examples (120 ms at f_d = 1.5 -> 180 ms;
  10 chains at f_tight = 0.4 -> exactly 4 at 60 ms) and hand-computed floors.
* R3 arrivals (§5 "periodically with a 15 ms jitter"):
  [0, 150, 300] ms without jitter; with J = 15 ms every offset in [0, 15] ms.
* R4 per-instance and per-kernel factors (Table 2 "+-" read as one sigma,
  SPEC.md:108): hand-computed durations for constant quantile tables (truncation toward zero,
  the 0.1 floor, the clamps to [1, 2^32 - 1]), and the table index = top 12 bits of the word.
* R5 sync cost ("10-200 us"): sigma_lo + w mod (sigma_hi - sigma_lo + 1), in range,
  and the return time max(t_call, t_sat) + sigma.

Where a draw's word is needed it is recomputed with tests/philox_ref.py, a Python Philox written
separately from the oracle's C copy and checked here against the Random123 KAT vectors.  The
trace rows are (t, kind, chain, instance, a, b): INST_START a = t_arr; EVAL a = laxity;
DISPATCH a = kernel, b = end time; SYNC_CALL a = target, b = cost.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from workloads.spec import (FIFO, MS, SYNC_ASYNC, SYNC_EACH, URGENGO, US, Batch, Chain, Kernel, Policy, Task,
                            Workload)

from . import philox_ref as PR
from .conftest import GOLDEN

K = O.TRACE_CODES
EVAL_ONLY = Policy(kind=URGENGO, flags=0, sync_mode=SYNC_ASYNC, lax_threshold_ns=-1)   # evaluates, never acts


def test_test_side_philox_known_answers():
    n = 0
    for line in open(os.path.join(GOLDEN, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        assert PR.philox4x32_10(v[:4], v[4:6]) == v[6:]
        n += 1
    assert n == 3


def _rows(r, kind):
    return [tuple(int(x) for x in row) for row in r.trace if row[1] == K[kind]]


def _probe_chains(C, period=150 * MS, deadline=120 * MS):
    """C chains whose Eq. 2 laxity at their first task start is D' - 1 us: one CPU segment with
    estimate 0, one kernel estimated 1 us."""
    return [Chain(period, deadline, 0, [Task(10 * US, 0, [Kernel(1 * US, 1 * US, 10)])]) for _ in range(C)]


def _dprime_at_start(w, b):
    """D' of every chain of scenario b.scenario_begin, read from the EVAL of instance 0's task start."""
    r = O.run(w, EVAL_ONLY, b, trace_cap=100_000)
    d = {}
    for t, _, c, i, a, _b in _rows(r, "EVAL"):
        if i == 0 and c not in d:
            assert t == 0
            d[c] = a + 1 * US
    return [d[c] for c in range(w.num_chains)]


def _wl(chains, **kw):
    base = dict(num_prio=2, launch_ns=0, launch_akb_ns=0, sync_lo_ns=0, sync_hi_ns=0, jitter_ns=0)
    base.update(kw)
    return Workload(chains=chains, **base)


# ---------------------------------------------------------------------------------------------
# R3: deadline and arrival factors, the tight subset
# ---------------------------------------------------------------------------------------------

def test_factor_identity():
    """f_a = f_d = 1, f_tight = 0: the configuration is unchanged."""
    w = _wl(_probe_chains(3))
    assert _dprime_at_start(w, Batch(horizon_ns=1 * MS)) == [120 * MS] * 3


def test_fd_scales_deadlines():
    """base deadline 120 ms, f_d = 1.5 -> 180 ms; f_d = 0.7 -> 84 ms (PAPER.md:600 range)."""
    w = _wl(_probe_chains(4))
    assert _dprime_at_start(w, Batch(horizon_ns=1 * MS, fd_num=3, fd_den=2)) == [180 * MS] * 4
    assert _dprime_at_start(w, Batch(horizon_ns=1 * MS, fd_num=7, fd_den=10)) == [84 * MS] * 4


def test_fd_floor_then_tight_halving():
    """D' = floor(D * fd_num / fd_den), then halved with floor for a tight chain: 120 ms x 3/2 tight
    -> 90 ms; 120 000 001 ns tight -> 60 000 000 ns; 100 ns x 2/3 -> 66 ns."""
    w = _wl(_probe_chains(2))
    b = Batch(horizon_ns=1 * MS, fd_num=3, fd_den=2, tight_explicit=1, tight_mask=0b01)
    assert _dprime_at_start(w, b) == [90 * MS, 180 * MS]
    w2 = _wl([Chain(150 * MS, 120_000_001, 0, [Task(10 * US, 0, [Kernel(1 * US, 1 * US, 10)])])])
    assert _dprime_at_start(w2, Batch(horizon_ns=1 * MS, tight_explicit=1, tight_mask=1)) == [60_000_000]
    w3 = _wl([Chain(150 * MS, 100, 0, [Task(0, 0, [Kernel(1, 0, 10)])])])
    r = O.run(w3, EVAL_ONLY, Batch(horizon_ns=1 * MS, fd_num=2, fd_den=3), trace_cap=1000)
    assert _rows(r, "EVAL")[0][4] == 66


@pytest.mark.parametrize("s", range(30))
def test_tight_subset_ten_chains(s):
    """10 chains, f_tight = 0.4, D = 120 ms -> exactly ceil(0.4 * 10) = 4 chains at 60 ms
    and 6 at 120 ms, in every scenario; the 4 are the chains with the smallest (TIGHT word, id)
    (R3, the per-scenario seeded selection of SPEC.md's design-decision ledger)."""
    w = _wl(_probe_chains(10))
    seed = 0x5EED0002
    d = _dprime_at_start(w, Batch(seed=seed, scenario_begin=s, horizon_ns=1 * MS, ftight_permille=400))
    assert sorted(d) == [60 * MS] * 4 + [120 * MS] * 6
    words = [(PR.word(seed, s, PR.TAG_TIGHT, c, 0, 0), c) for c in range(10)]
    want = {c for _, c in sorted(words)[:4]}
    assert {c for c in range(10) if d[c] == 60 * MS} == want


def test_tight_count_rounds_up():
    """ceil, not floor: 11 chains (paper11's C0-C10) at 0.4 -> 5 tight (4.4 rounds up); 0.1 -> 2;
    1.0 -> all; 0 -> none; 1 permille of 11 chains -> 1."""
    w = _wl(_probe_chains(11))
    for pm, n in ((400, 5), (100, 2), (1000, 11), (0, 0), (1, 1)):
        for s in (0, 7):
            d = _dprime_at_start(w, Batch(seed=3, scenario_begin=s, horizon_ns=1 * MS, ftight_permille=pm))
            assert d.count(60 * MS) == n and d.count(120 * MS) == 11 - n, (pm, s)


def test_tight_selection_varies_by_scenario():
    w = _wl(_probe_chains(10))
    sets = {tuple(_dprime_at_start(w, Batch(seed=9, scenario_begin=s, horizon_ns=1 * MS, ftight_permille=400)))
            for s in range(12)}
    assert len(sets) > 4


def _arrivals(w, b, chain=0):
    r = O.run(w, EVAL_ONLY, b, trace_cap=200_000)
    return [a for t, _, c, i, a, _b in _rows(r, "INST_START") if c == chain], r


def test_arrivals_zero_jitter():
    """period 150 ms, jitter 0, 0.45 s -> arrivals [0, 150, 300] ms (H is exclusive)."""
    w = _wl(_probe_chains(1))
    arr, r = _arrivals(w, Batch(horizon_ns=450 * MS))
    assert arr == [0, 150 * MS, 300 * MS]
    assert r.records[0, 0, 0] == 3
    arr, r = _arrivals(w, Batch(horizon_ns=450 * MS + 1))
    assert arr == [0, 150 * MS, 300 * MS, 450 * MS]


def test_fa_scales_periods():
    """P' = floor(P * fa_den / fa_num): 150 ms at f_a = 2 -> 75 ms; 100 ms at f_a = 3 -> 33 333 333 ns;
    usweep's u = 0.5 point (f_a = 5000/12082): 150 ms -> 362 460 000 ns."""
    arr, _ = _arrivals(_wl(_probe_chains(1)), Batch(horizon_ns=300 * MS, fa_num=2, fa_den=1))
    assert arr == [0, 75 * MS, 150 * MS, 225 * MS]
    arr, _ = _arrivals(_wl(_probe_chains(1, period=100 * MS)), Batch(horizon_ns=100 * MS, fa_num=3, fa_den=1))
    assert arr == [0, 33_333_333, 66_666_666, 99_999_999]
    arr, _ = _arrivals(_wl(_probe_chains(1)), Batch(horizon_ns=1000 * MS, fa_num=5000, fa_den=12082))
    assert arr == [0, 362_460_000, 724_920_000]


def test_arrival_offset_keeps_period():
    """A chain offset O shifts every arrival: O + i P'."""
    ch = [Chain(150 * MS, 120 * MS, 7 * MS, [Task(10 * US, 0, [Kernel(1 * US, 1 * US, 10)])])]
    arr, _ = _arrivals(_wl(ch), Batch(horizon_ns=400 * MS))
    assert arr == [7 * MS, 157 * MS, 307 * MS]


def test_arrivals_with_jitter():
    """period 150 ms, jitter 15 ms -> every offset in [0, 15] ms, inter-arrival in
    [135, 165] ms; each offset is the ARR word of (chain, instance) mod (J + 1)."""
    J = 15 * MS
    seed = 0x5EED0004
    w = _wl(_probe_chains(3), jitter_ns=J)
    offs = []
    for s in (0, 1, 999_999):
        b = Batch(seed=seed, scenario_begin=s, horizon_ns=15_000 * MS)
        r = O.run(w, EVAL_ONLY, b, trace_cap=400_000)
        rows = _rows(r, "INST_START")
        for c in range(3):
            arr = [a for t, _, cc, i, a, _b in rows if cc == c]
            assert len(arr) == 100
            for i, a in enumerate(arr):
                o = a - i * 150 * MS
                assert 0 <= o <= J
                assert o == PR.word(seed, s, PR.TAG_ARR, c, i, 0) % (J + 1)
                offs.append(o)
            gaps = np.diff(arr)
            assert gaps.min() >= 135 * MS and gaps.max() <= 165 * MS
    assert min(offs) < 1 * MS and max(offs) > 14 * MS      # the whole window is used


# ---------------------------------------------------------------------------------------------
# R4: per-instance and per-kernel factors, the duration arithmetic
# ---------------------------------------------------------------------------------------------

def _durations(z_q16, g_q16, gpu_sigma, cpu_sigma, noms=(2_000_000, 1), cpu=10 * MS, horizon=1 * MS):
    """One chain, one instance: the CPU segment's duration (= k0's dispatch time, lambda = 0) and
    every kernel's run time, with constant quantile tables z (per instance) and G (per kernel)."""
    ch = Chain(1000 * MS, 100_000 * MS, 0, [Task(cpu, cpu, [Kernel(n, n, 1000) for n in noms])],
               cpu_sigma_ppm=cpu_sigma, gpu_sigma_ppm=gpu_sigma)
    w = _wl([ch], inst_quantiles_q16=np.full(4096, z_q16, np.int32),
            kern_quantiles_q16=None if g_q16 is None else np.full(4096, g_q16, np.uint32))
    r = O.run(w, Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC), Batch(horizon_ns=horizon), trace_cap=1000)
    disp = _rows(r, "DISPATCH")
    e = disp[0][0]
    return e, [b - t for t, _, c, i, a, b in disp]


def test_r4_one_sigma_up():
    """z = +1.0 (65536), sigma_g = 10 %: F = 65536 + trunc(6553.6) = 72089;
    k0: (2 000 000 * 72089) >> 16 = 2 199 981, x G = 2.0 -> 4 399 962 ns; k1: 1 ns -> 1 -> 2 ns.
    CPU: sigma_c = 25 % -> F_c = 81920 (1.25): 10 ms -> 12 500 000 ns."""
    e, d = _durations(65536, 131072, 100_000, 250_000)
    assert e == 12_500_000
    assert d == [4_399_962, 2]


def test_r4_factor_floor_and_min_duration():
    """z = -3.0, sigma_g = 50 %: F = 65536 - 98304 < 0 -> floored at 6554 (0.1);
    k0: (2 000 000 * 6554) >> 16 = 200 012 ns; k1: (1 * 6554) >> 16 = 0 -> clamped to 1 ns.
    sigma_c = 0: the CPU segment keeps its nominal 10 ms."""
    e, d = _durations(-196608, 65536, 500_000, 0)
    assert e == 10 * MS
    assert d == [200_012, 1]


def test_r4_truncation_toward_zero():
    """z = -1.0, sigma_g = 10 %: z * sigma / 10^6 = -6553.6 truncates to -6553 (floor would give
    -6554): F = 58983, k0 = (2 000 000 * 58983) >> 16 = 1 800 018 ns (not 1 799 987).
    sigma_c = 100 %: F_c = 0 -> floor 6554: 10 ms -> 1 000 061 ns.  No per-kernel table: G = 1."""
    e, d = _durations(-65536, None, 100_000, 1_000_000)
    assert e == 1_000_061
    assert d == [1_800_018, 1]


def test_r4_duration_upper_clamp():
    """A 4 s kernel at F = 72089 and G = 2.0: 8 799 926 756 ns exceeds u32 -> 2^32 - 1."""
    e, d = _durations(65536, 131072, 100_000, 0, noms=(4_000_000_000,), cpu=0, horizon=1 * MS)
    assert d == [0xFFFFFFFF]


def test_r4_table_index_is_top_12_bits():
    """Non-constant tables: z[j] = (j - 2048) * 32 (sigma_g = 100 %), G[j] = 65536 + 16 j.  Every
    kernel's duration is ((nom * F) >> 16) * G >> 16 with F = max(6554, 65536 + z[w_INST >> 20]) (word 0 of
    (chain, instance)) and G = G[w_KERN >> 20] (word k of (chain, instance))."""
    seed = 0x5EED0004
    z = (np.arange(4096, dtype=np.int64) - 2048) * 32
    G = 65536 + 16 * np.arange(4096, dtype=np.int64)
    noms = [300_000, 1_234_567, 77_777, 5_000_000, 42]
    ch = Chain(40 * MS, 1000 * MS, 0, [Task(1 * MS, 1 * MS, [Kernel(n, n, 1000) for n in noms])],
               cpu_sigma_ppm=0, gpu_sigma_ppm=1_000_000)
    w = _wl([ch], inst_quantiles_q16=z.astype(np.int32), kern_quantiles_q16=G.astype(np.uint32))
    n_checked = 0
    for s in (0, 5, 123_456):
        r = O.run(w, Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC),
                  Batch(seed=seed, scenario_begin=s, horizon_ns=400 * MS), trace_cap=10_000)
        for t, _, c, i, k, end in _rows(r, "DISPATCH"):
            F = max(6554, 65536 + int(z[PR.word(seed, s, PR.TAG_INST, c, i, 0) >> 20]))   # 0.1 floor
            g = int(G[PR.word(seed, s, PR.TAG_KERN, c, i, k) >> 20])
            want = max(1, min(0xFFFFFFFF, (((noms[k] * F) >> 16) * g) >> 16))
            assert end - t == want, (s, i, k)
            n_checked += 1
    assert n_checked == 3 * 10 * 5


def test_r4_cpu_factor_uses_word_one():
    """The CPU factor of an instance is drawn from word 1 of (chain, instance) (word 0 is the GPU's):
    z[j] = (j - 2048) * 32, sigma_c = 100 %, CPU 1 ms -> e = (10^6 * F_c) >> 16."""
    seed = 77
    z = (np.arange(4096, dtype=np.int64) - 2048) * 32
    ch = Chain(40 * MS, 1000 * MS, 0, [Task(1 * MS, 1 * MS, [Kernel(10 * US, 10 * US, 1000)])],
               cpu_sigma_ppm=1_000_000, gpu_sigma_ppm=0)
    w = _wl([ch], inst_quantiles_q16=z.astype(np.int32))
    r = O.run(w, Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC), Batch(seed=seed, horizon_ns=400 * MS),
              trace_cap=10_000)
    starts = {i: t for t, _, c, i, a, b in _rows(r, "INST_START")}
    for t, _, c, i, k, end in _rows(r, "DISPATCH"):
        Fc = max(6554, 65536 + int(z[PR.word(seed, 0, PR.TAG_INST, 0, i, 1) >> 20]))
        assert t - starts[i] == (1 * MS * Fc) >> 16


# ---------------------------------------------------------------------------------------------
# R5: sync-call cost
# ---------------------------------------------------------------------------------------------

def test_r5_sync_cost_draws_and_return_time():
    """every issued sync costs sigma in [10, 200] us, sigma = 10 us + w mod 190 001 with
    w the SYNC word of (chain, instance, ordinal of the sync within the instance); it returns at
    max(t_call, t_satisfied) + sigma (SYNC_EACH: one sync per kernel, ordinals 0..5 over two tasks)."""
    seed = 0x5EED0002
    tasks = [Task(1 * MS, 1 * MS, [Kernel(300 * US, 300 * US, 1000) for _ in range(3)]) for _ in range(2)]
    w = _wl([Chain(20 * MS, 1000 * MS, 0, tasks), Chain(30 * MS, 1000 * MS, 1 * MS, tasks)],
            sync_lo_ns=10 * US, sync_hi_ns=200 * US, launch_ns=21_672)
    costs = []
    for s in (0, 4242):
        r = O.run(w, Policy(kind=FIFO, flags=0, sync_mode=SYNC_EACH), Batch(seed=seed, scenario_begin=s,
                                                                            horizon_ns=300 * MS), trace_cap=100_000)
        calls = _rows(r, "SYNC_CALL")
        rets = _rows(r, "SYNC_RET")
        retired = {(c, i, k): t for t, _, c, i, k, _b in _rows(r, "RETIRE")}
        ordinal = {}
        for (tc, _, c, i, target, cost), (tr_, _2, c2, i2, target2, _3) in zip(
                sorted(calls, key=lambda x: (x[2], x[0])), sorted(rets, key=lambda x: (x[2], x[0]))):
            m = ordinal.get((c, i), 0)
            ordinal[(c, i)] = m + 1
            assert cost == 10 * US + PR.word(seed, s, PR.TAG_SYNC, c, i, m) % (190 * US + 1)
            assert (c2, i2, target2) == (c, i, target)
            assert tr_ == max(tc, retired[(c, i, target - 1)]) + cost
            costs.append(cost)
    assert min(costs) >= 10 * US and max(costs) <= 200 * US
    assert len(costs) >= 300 and 80 * US < np.mean(costs) < 130 * US


def test_r5_constant_cost_when_range_is_empty():
    tasks = [Task(1 * MS, 1 * MS, [Kernel(300 * US, 300 * US, 1000)])]
    w = _wl([Chain(20 * MS, 1000 * MS, 0, tasks)], sync_lo_ns=37 * US, sync_hi_ns=37 * US)
    r = O.run(w, Policy(kind=FIFO, flags=0, sync_mode=SYNC_EACH), Batch(horizon_ns=100 * MS), trace_cap=10_000)
    assert {b for *_, b in _rows(r, "SYNC_CALL")} == {37 * US}
