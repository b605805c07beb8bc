"""The seeded input generators (workloads/): determinism and the paper's totals."""
import numpy as np

from workloads import paper11, toy2
from workloads.quantiles import inst_z_table, pareto_table
from workloads.spec import MS
from workloads.templates import TABLE2, TABLE4, synth_kernel_times


def test_paper11_deterministic():
    a, b = paper11().flat(), paper11().flat()
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_paper11_matches_tables():
    """Chain totals = Table 2 E^gpu_C / E^cpu_C; kernel counts are
    sums of Table 4 N_k per SURVEY.md Q17; sum N = 4240."""
    w = paper11()
    assert w.total_kernels() == 4240
    for c, ch in enumerate(w.chains):
        P, D, ecpu, _, egpu, _, names = TABLE2[c]
        assert ch.period_ns == P * MS and ch.deadline_ns == D * MS
        assert sum(k.nominal_ns for t in ch.tasks for k in t.kernels) == int(round(egpu * MS))
        assert sum(t.cpu_nominal_ns for t in ch.tasks) == int(round(ecpu * MS))
        assert [len(t.kernels) for t in ch.tasks] == [TABLE4[n][0] for n in names]
        assert all(k.nominal_ns >= 1 and 0 <= k.util_permille <= 1000 for t in ch.tasks for k in t.kernels)


def test_paper11_utilisation():
    """u = sum_c E^gpu_C / P_C = 1.2082 at f_a = 1 (Table 2; SURVEY.md §8(d) cfg 3 rounds it to 1.207)."""
    u = sum(egpu / P for P, _, _, _, egpu, _, _ in TABLE2)
    assert abs(u - 1.2082) < 1e-4


def test_kernel_synthesis_exact_and_skewed():
    rng = np.random.default_rng(0)
    d = synth_kernel_times(323, int(19.8 * MS), rng)
    assert len(d) == 323 and sum(d) == int(19.8 * MS) and min(d) >= 1
    assert np.median(d) < np.mean(d)              # right-skewed: most kernels short
    assert synth_kernel_times(1, 10 * MS, rng) == [10 * MS]


def test_quantile_tables():
    z = inst_z_table()
    assert z.dtype == np.int32 and len(z) == 4096
    assert np.all(np.diff(z) >= 0) and abs(int(z.sum())) <= 4096 and z.min() >= -3 * 65536 and z.max() <= 3 * 65536
    p = pareto_table()
    assert p.dtype == np.uint32 and abs(p.mean() / 65536 - 1) < 1e-4 and p.max() <= 64 * 65536 * 2


def test_toy2_shape():
    w = toy2()
    assert w.num_chains == 2 and w.total_kernels() == 30 and w.num_prio == 2
