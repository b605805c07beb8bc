"""BASELINE.json configurations at their full sizes, in the launch configuration bench.py times,
checked on sampled outputs the oracle computes one by one (BASELINE.md's sampling rule), plus
properties that hold at any size (aggregates = sums of the per-scenario records, R23).

* configs[3] ("jitter", the bench headline): two whole 50 000-scenario bench slices at the 60 s
  horizon -- the first and the last of the 1M -- in the packed throughput build; scenarios 0,
  9973, ..., 999 999 against the oracle;
* configs[4] ("scaleout"): a 100 000-scenario slice from the middle of the 100M, the first 256,
  the last 256 and every 9973rd scenario against the oracle;
* configs[2] ("usweep"): the u = 0.5 and u = 1.2 points at 100 000 scenarios under UrgenGo,
  FIFO and STATIC, sampled.
"""
import multiprocessing as mp
from concurrent.futures import ProcessPoolExecutor
from dataclasses import replace

import numpy as np
import pytest

from workloads import get_config

from .gpu_helpers import agg_from_records, gpu_run
from .oracle_pool import oracle_one

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def sampled_parity(name, pol, b, rec, sample):
    """Oracle records of `sample` (global indices inside b) equal the GPU's, one scenario per job."""
    # spawned workers: the parent holds a CUDA context; the children run only the C oracle
    with ProcessPoolExecutor(max_workers=min(16, len(sample)), mp_context=mp.get_context("spawn")) as ex:
        res = list(ex.map(oracle_one, [(name, pol, b, s) for s in sample]))
    bad = [s for s, r in res if not np.array_equal(r, rec[s - b.scenario_begin])]
    assert not bad, f"{name}/{pol}: scenarios {bad[:8]} differ from the oracle"
    return len(res)


def baseline_sample(begin, count, stride=9973, head=256):
    idx = set(range(begin, begin + min(head, count))) | set(range(begin + max(0, count - head), begin + count))
    idx |= set(range(begin, begin + count, stride))
    return sorted(idx)


def check_consistency(w, rec, agg):
    """Counters, miss-ratio bins and the launch total of the aggregate are the records' sums (R23)."""
    want = agg_from_records(rec, w.num_chains, w.rt_bins)
    stride = 5 + w.rt_bins + 101
    for c in range(w.num_chains):
        base = c * stride
        assert np.array_equal(agg[base: base + 5], want[base: base + 5])
        assert np.array_equal(agg[base + 5 + w.rt_bins: base + stride], want[base + 5 + w.rt_bins: base + stride])
    assert agg[-2] == want[-2]
    # every completed instance lands in exactly one rt bin
    for c in range(w.num_chains):
        base = c * stride
        completed = int(rec[:, c, 0].astype(np.int64).sum() - rec[:, c, 2].astype(np.int64).sum()
                        - rec[:, c, 3].astype(np.int64).sum())
        assert int(agg[base + 5: base + 5 + w.rt_bins].sum()) == completed


@pytest.mark.parametrize("slice_begin", [0, 950_000])
def test_configs3_full_horizon_bench_slices(slice_begin):
    cfg = get_config("jitter")
    w, p = cfg.workload(), cfg.policies["urgengo"]
    b = replace(cfg.batch, scenario_begin=slice_begin, scenario_count=50_000)
    assert b.horizon_ns == 60_000_000_000
    rec, agg = gpu_run(w, p, b)
    check_consistency(w, rec, agg)
    sample = [s for s in range(0, 1_000_000, 9973) if slice_begin <= s < slice_begin + 50_000]
    sample += [slice_begin, slice_begin + 49_999]
    if slice_begin == 950_000:
        sample.append(999_999)
    n = sampled_parity("jitter", "urgengo", b, rec, sorted(set(sample)))
    assert n >= 7


def test_configs4_slice_sampled():
    cfg = get_config("scaleout")
    w, p = cfg.workload(), cfg.policies["urgengo"]
    b = replace(cfg.batch, scenario_begin=50_000_000, scenario_count=100_000)
    rec, agg = gpu_run(w, p, b)
    check_consistency(w, rec, agg)
    assert sampled_parity("scaleout", "urgengo", b, rec, baseline_sample(b.scenario_begin, b.scenario_count)) == 522


@pytest.mark.parametrize("point", [0, 7])
@pytest.mark.parametrize("pol", ["urgengo", "fifo", "static"])
def test_configs2_sweep_points(point, pol):
    """u = 0.5 (point 0) and u = 1.2 (point 7, overload) at 100 000 scenarios."""
    cfg = get_config("usweep")
    w, p = cfg.workload(), cfg.policies[pol]
    b = cfg.sweep[point]
    assert b.scenario_count == 100_000
    rec, agg = gpu_run(w, p, b)
    check_consistency(w, rec, agg)
    sample = baseline_sample(b.scenario_begin, b.scenario_count, stride=9973, head=4)
    assert sampled_parity("usweep", pol, b, rec, sample) == 18
