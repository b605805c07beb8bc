"""Design-option studies of UrgenGo on the batched GPU simulator.

Each study is a list of policy / workload / batch variants of one base configuration,
run through the same C-ABI call (``urg_simulate_batch``) on the current CUDA device:

* ``sync_modes``   -- launch synchronisation: synchronous, asynchronous, batched, and
                      UrgenGo's overlapped batches (Fig. fig:9_launch);
* ``delta_eval``   -- urgency-evaluation interval Delta_eval (fig:10_resolution);
* ``num_prio``     -- number of binding streams 1..6 (fig:5_stream_num);
* ``ablation``     -- binding only / delay only / both (fig:4_ablation);
* ``collisions``   -- kernel collisions of urgent kernels with and without delayed
                      launching, by number of colliding tasks (fig:8_collision);
* ``policies``     -- UrgenGo against the vanilla (FIFO), PAAM-like static, EDF, SJF, HRRN
                      and lowest-chain-utilisation-first policies (fig:6_policy);
* ``cudafree``     -- 0..4 tasks ending with cudaFree, a device-wide barrier (PAPER.md:907-911,
                      fig:15_vector_free; R28);
* ``cpu_cores``    -- the chains' threads on 1..8 shared CPU cores with the policy's SCHED_FIFO
                      priorities (R29);
* ``contention``   -- kernel slow-down from co-running kernels (R30);
* ``memcpy``       -- H2D/D2H memcpys around every task on the copy engine (Table 3; R31);
* ``executors``    -- one thread per chain against one executor thread per task, tasks of
                      successive instances pipelined (R32);
* ``utilisation``  -- UrgenGo vs FIFO vs static priorities over an arrival-rate sweep
                      (BASELINE.json configs[2]; PAPER.md:679-683 fig:0_overall analogue).

Only argument marshalling and bookkeeping happen here; every simulated step runs
in liburg.so.  Miss ratios follow Eq. 3 via ``urg_miss_ratios``.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Dict, List, Optional

import numpy as np

from workloads.spec import (COLL_BINS, EDF, F_BIND, F_COLLISIONS, F_DELAY, F_EARLY_EXIT, FIFO, HRRN, LCUF, SJF,
                            EXEC_CHAIN, EXEC_TASK, STATIC, SYNC_ASYNC,
                            SYNC_BATCHED, SYNC_EACH, SYNC_OVERLAP, URGENGO, Batch, Policy, Workload,
                            collision_hist)

from .urg import DeviceWorkload


@dataclass
class Point:
    """One variant of a study: what changed, and the batch it ran."""
    label: str
    policy: Policy
    batch: Batch
    num_prio: Optional[int] = None          # workload override (binding streams)
    frees: Optional[int] = None             # workload override: the first n tasks end with cudaFree (R28)
    cores: Optional[int] = None             # workload override: CPU cores shared by the threads (R29)
    alpha: Optional[int] = None             # workload override: contention slow-down per-mille (R30)
    copies: bool = False                    # workload override: H2D/D2H memcpys around every task (R31)
    executors: Optional[int] = None         # workload override: EXEC_CHAIN / EXEC_TASK (R32)


@dataclass
class Result:
    label: str
    overall_miss: float                     # Eq. 3
    per_chain_miss: List[float]
    collisions: Dict[int, int]              # number of colliding tasks -> events (R24)
    launches: int
    steps: int
    gpu_ms: float
    extra: dict = field(default_factory=dict)


def sync_modes(base: Policy, b: Batch) -> List[Point]:
    names = [("sync (each kernel)", SYNC_EACH), ("async", SYNC_ASYNC), ("sync batched", SYNC_BATCHED),
             ("UrgenGo overlapped", SYNC_OVERLAP)]
    return [Point(n, replace(base, sync_mode=m), b) for n, m in names]


def delta_eval(base: Policy, b: Batch, values_us=(100, 250, 500, 1000, 2000, 4000)) -> List[Point]:
    return [Point(f"delta_eval {v} us", replace(base, delta_eval_ns=v * 1000), b) for v in values_us]


def num_prio(base: Policy, b: Batch, values=(1, 2, 3, 4, 5, 6)) -> List[Point]:
    return [Point(f"NUM_PRI {n}", base, b, num_prio=n) for n in values]


def ablation(base: Policy, b: Batch) -> List[Point]:
    early = base.flags & F_EARLY_EXIT
    return [Point("no binding, no delay", replace(base, flags=early), b),
            Point("binding only", replace(base, flags=early | F_BIND), b),
            Point("delay only", replace(base, flags=early | F_DELAY), b),
            Point("binding + delay", replace(base, flags=early | F_BIND | F_DELAY), b)]


def collisions(base: Policy, b: Batch) -> List[Point]:
    f = base.flags | F_COLLISIONS
    return [Point("UrgenGo without delayed launching", replace(base, flags=f & ~F_DELAY), b),
            Point("UrgenGo", replace(base, flags=f), b)]


def policies(base: Policy, b: Batch) -> List[Point]:
    out = [Point("UrgenGo", base, b), Point("FIFO (vanilla)", Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC), b),
           Point("static (PAAM-like)", Policy(kind=STATIC, flags=0, sync_mode=SYNC_ASYNC), b)]
    for n, k in (("EDF", EDF), ("SJF", SJF), ("HRRN", HRRN), ("LCUF", LCUF)):
        out.append(Point(n, Policy(kind=k, flags=0, sync_mode=base.sync_mode, delta_eval_ns=base.delta_eval_ns), b))
    return out


def cudafree(base: Policy, b: Batch, counts=(0, 1, 2, 3, 4)) -> List[Point]:
    """PAPER.md:907-911 (fig:15_vector_free): 0..4 tasks ending with cudaFree, under UrgenGo,
    static priorities and plain asynchronous launching."""
    pols = [("UrgenGo", base), ("static (PAAM-like)", Policy(kind=STATIC, flags=0, sync_mode=SYNC_ASYNC)),
            ("async (FIFO)", Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC))]
    return [Point(f"{n} cudaFree tasks, {name}", p, b, frees=n) for n in counts for name, p in pols]


def cpu_cores(base: Policy, b: Batch, counts=(1, 2, 4, 8, 0)) -> List[Point]:
    """PAPER.md:386-399 urgency-centric CPU scheduling: the chains' threads on 1..8 shared cores
    (0 = one core per thread) under UrgenGo, static priorities and FIFO (R29)."""
    pols = [("UrgenGo", base), ("static (PAAM-like)", Policy(kind=STATIC, flags=0, sync_mode=SYNC_ASYNC)),
            ("FIFO", Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC))]
    return [Point(f"{'unlimited' if n == 0 else n} cores, {name}", p, b, cores=n) for n in counts for name, p in pols]


def contention(base: Policy, b: Batch, alphas=(0, 250, 500, 1000, 2000)) -> List[Point]:
    """PAPER.md:209-212 (fig:13_cdf): co-running kernels slow each other down; miss ratios of
    UrgenGo, static priorities and FIFO as the slow-down alpha grows (R30)."""
    pols = [("UrgenGo", base), ("static (PAAM-like)", Policy(kind=STATIC, flags=0, sync_mode=SYNC_ASYNC)),
            ("FIFO", Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC))]
    return [Point(f"alpha {a} permille, {name}", p, b, alpha=a) for a in alphas for name, p in pols]


def memcpy(base: Policy, b: Batch) -> List[Point]:
    """Table 3: every task starts with a 0.3 ms H2D memcpy and ends with a 0.1 ms
    D2H memcpy on the copy engine (R31), against the same workload without copies."""
    pols = [("UrgenGo", base), ("static (PAAM-like)", Policy(kind=STATIC, flags=0, sync_mode=SYNC_ASYNC)),
            ("FIFO", Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC))]
    return [Point(f"{'with' if cp else 'no'} memcpys, {name}", p, b, copies=cp) for cp in (False, True)
            for name, p in pols]


def executors(base: Policy, b: Batch) -> List[Point]:
    """PAPER.md:272 ("each task is executed by a dedicated thread"): the chain-thread model (R6)
    against per-task executor threads with depth-1 hand-over (R32), under UrgenGo, static
    priorities and FIFO."""
    pols = [("UrgenGo", base), ("static (PAAM-like)", Policy(kind=STATIC, flags=0, sync_mode=SYNC_ASYNC)),
            ("FIFO", Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC))]
    return [Point(f"{lbl}, {name}", p, b, executors=e) for e, lbl in ((EXEC_CHAIN, "thread per chain"),
                                                                    (EXEC_TASK, "executor per task"))
            for name, p in pols]


def with_copies(w: Workload, h2d_ns: int = 300_000, d2h_ns: int = 100_000) -> Workload:
    """A copy of w whose tasks start with an H2D and end with a D2H memcpy (R31)."""
    import copy
    from workloads.spec import Kernel
    w2 = copy.deepcopy(w)
    h2d, d2h = Kernel(h2d_ns, h2d_ns, 200, 1), Kernel(d2h_ns, d2h_ns, 200, 1)
    variants = [iter(v) for v in (w2.kernel_variants or [])]
    new_variants = [[] for _ in variants]
    for ch in w2.chains:
        for t in ch.tasks:
            for it, nv in zip(variants, new_variants):   # every template variant gets the same copies (R33)
                nv += [copy.copy(h2d)] + [next(it) for _ in t.kernels] + [copy.copy(d2h)]
            t.kernels = [copy.copy(h2d)] + t.kernels + [copy.copy(d2h)]
    if variants:
        w2.kernel_variants = new_variants
    return w2


def with_frees(w: Workload, n: int) -> Workload:
    """A copy of w whose first n tasks (chain-major) end with cudaFree."""
    import copy
    w2 = copy.deepcopy(w)
    k = 0
    for ch in w2.chains:
        for t in ch.tasks:
            t.frees = k < n
            k += 1
    return w2


def utilisation(base: Policy, batches: List[Batch]) -> List[Point]:
    pols = [("UrgenGo", base), ("FIFO", Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC)),
            ("static", Policy(kind=STATIC, flags=0, sync_mode=SYNC_ASYNC))]
    out = []
    for bb in batches:
        u = 1.2082 * bb.fa_num / bb.fa_den
        for n, p in pols:
            out.append(Point(f"u={u:.2f} {n}", p, bb))
    return out


STUDIES = ("sync_modes", "delta_eval", "num_prio", "ablation", "collisions", "policies", "cudafree", "cpu_cores",
           "contention", "memcpy", "executors")


def run(w: Workload, points: List[Point], stream=None) -> List[Result]:
    """Run every point on the current CUDA device (one urg_simulate_batch per point)."""
    import torch
    out = []
    cache: Dict[tuple, DeviceWorkload] = {}
    try:
        for pt in points:
            npri = pt.num_prio if pt.num_prio is not None else w.num_prio
            key = (npri, pt.frees, pt.cores, pt.alpha, pt.copies, pt.executors)
            if key not in cache:
                ww = replace(w, num_prio=npri, cpu_cores=pt.cores if pt.cores is not None else w.cpu_cores,
                             contention_permille=pt.alpha if pt.alpha is not None else w.contention_permille,
                             executors=pt.executors if pt.executors is not None else w.executors)
                if pt.copies:
                    ww = with_copies(ww)
                cache[key] = DeviceWorkload(with_frees(ww, pt.frees) if pt.frees is not None else ww)
            dw = cache[key]
            agg = torch.zeros(dw.agg_words, dtype=torch.int64, device="cuda")
            s = stream if stream is not None else torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            dw.simulate(pt.policy, pt.batch, agg, None, stream=s)
            e1.record(s)
            dw.check(s)
            a = agg.cpu().numpy()
            per, overall = dw.miss_ratios(a)
            h = collision_hist(a, w.num_chains, w.rt_bins)
            out.append(Result(pt.label, float(overall), [float(x) for x in per],
                              {int(k): int(h[k]) for k in range(COLL_BINS) if h[k]},
                              int(a[-2]), int(a[-1]), float(e0.elapsed_time(e1))))
    finally:
        for dw in cache.values():
            dw.close()
    return out


def table(results: List[Result]) -> str:
    rows = ["| variant | Eq. 3 miss ratio | collisions (tasks: events) | launch events | GPU ms | G events/s |",
            "|---|---|---|---|---|---|"]
    for r in results:
        coll = ", ".join(f"{k}: {v}" for k, v in sorted(r.collisions.items())) or "-"
        rows.append(f"| {r.label} | {r.overall_miss:.4f} | {coll} | {r.launches} | {r.gpu_ms:.1f} | "
                    f"{r.launches / max(r.gpu_ms, 1e-9) / 1e6:.3f} |")
    return "\n".join(rows)
