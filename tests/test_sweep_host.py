"""Host-side construction of the design-option studies (no GPU): each study varies
exactly the knob the paper's experiment varies."""
from workloads import get_config
from workloads.spec import (F_BIND, F_COLLISIONS, F_DELAY, F_EARLY_EXIT, SYNC_ASYNC, SYNC_BATCHED, SYNC_EACH,
                            SYNC_OVERLAP)


def test_studies_vary_one_knob():
    from paper_2509_12207_b200 import sweep as SW
    cfg = get_config("paper11")
    base, b = cfg.policies["urgengo"], cfg.batch
    assert [p.policy.sync_mode for p in SW.sync_modes(base, b)] == [SYNC_EACH, SYNC_ASYNC, SYNC_BATCHED, SYNC_OVERLAP]
    de = SW.delta_eval(base, b)
    assert [p.policy.delta_eval_ns for p in de] == [100_000, 250_000, 500_000, 1_000_000, 2_000_000, 4_000_000]
    assert all(p.policy.flags == base.flags for p in de)
    assert [p.num_prio for p in SW.num_prio(base, b)] == [1, 2, 3, 4, 5, 6]
    ab = SW.ablation(base, b)
    assert [p.policy.flags & (F_BIND | F_DELAY) for p in ab] == [0, F_BIND, F_DELAY, F_BIND | F_DELAY]
    assert all(p.policy.flags & F_EARLY_EXIT == base.flags & F_EARLY_EXIT for p in ab)
    co = SW.collisions(base, b)
    assert all(p.policy.flags & F_COLLISIONS for p in co)
    assert [bool(p.policy.flags & F_DELAY) for p in co] == [False, True]
    us = SW.utilisation(base, get_config("usweep").sweep)
    assert len(us) == 8 * 3


def test_policy_study_kinds():
    from paper_2509_12207_b200 import sweep as SW
    cfg = get_config("paper11")
    kinds = [p.policy.kind for p in SW.policies(cfg.policies["urgengo"], cfg.batch)]
    assert kinds == [2, 0, 1, 3, 4, 5, 6]


def test_workload_transforms():
    """sweep's workload transforms change exactly what their study varies."""
    from paper_2509_12207_b200 import sweep as SW
    w = get_config("paper11").workload()
    f2 = SW.with_frees(w, 2)
    flags = [t.frees for ch in f2.chains for t in ch.tasks]
    assert flags[:2] == [True, True] and not any(flags[2:])
    assert not any(t.frees for ch in w.chains for t in ch.tasks)          # the original is untouched
    cp = SW.with_copies(w)
    for ch0, ch1 in zip(w.chains, cp.chains):
        for t0, t1 in zip(ch0.tasks, ch1.tasks):
            assert len(t1.kernels) == len(t0.kernels) + 2
            assert t1.kernels[0].flags == 1 and t1.kernels[-1].flags == 1
            assert [k.nominal_ns for k in t1.kernels[1:-1]] == [k.nominal_ns for k in t0.kernels]
    pts = SW.cpu_cores(get_config("paper11").policies["urgengo"], get_config("paper11").batch)
    assert sorted({p.cores for p in pts}) == [0, 1, 2, 4, 8]
    assert sorted({p.alpha for p in SW.contention(get_config("paper11").policies["urgengo"],
                                                   get_config("paper11").batch)}) == [0, 250, 500, 1000, 2000]


def test_executors_study():
    from paper_2509_12207_b200 import sweep as SW
    from workloads.spec import EXEC_CHAIN, EXEC_TASK
    cfg = get_config("paper11")
    pts = SW.executors(cfg.policies["urgengo"], cfg.batch)
    assert [p.executors for p in pts] == [EXEC_CHAIN] * 3 + [EXEC_TASK] * 3
    assert [p.policy.kind for p in pts[:3]] == [p.policy.kind for p in pts[3:]] == [2, 1, 0]


def test_copies_keep_template_variants_aligned():
    from paper_2509_12207_b200 import sweep as SW
    from workloads import paper11_variants
    w = SW.with_copies(paper11_variants(3))
    n = w.total_kernels()
    assert all(len(v) == n for v in w.kernel_variants)
    flags0 = [k.flags for ch in w.chains for t in ch.tasks for k in t.kernels]
    assert all([k.flags for k in v] == flags0 for v in w.kernel_variants)
