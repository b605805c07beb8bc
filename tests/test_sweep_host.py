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
