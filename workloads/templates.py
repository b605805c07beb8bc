"""Workload templates: the paper-shaped 11-chain workflow, the 2-chain toy and
the hand-worked fixtures W1-W3.

Nothing here simulates anything; it only builds chain/task/kernel records.

paper11 (BASELINE.json configs[1]) -- chains C0-C10 of Table 2:
period, deadline D, E^cpu_C +- sigma and E^gpu_C +- sigma per chain.  Tasks of
each chain are the GPU tasks of Table 4 combined as in
SURVEY.md §8(c) Q17 (the combinations whose Table 4 totals reproduce Table 2's
E^gpu_C).  Table 2 totals govern: each chain's GPU time is split over its tasks
in proportion to Table 4's E_gpu and each task's kernel count is Table 4's N_k.
Per-kernel times are a truncated log-normal (most kernels < 100 us with a long
tail, Fig. fig:14_kernel_time PAPER.md:180) rescaled so the task sum is exact
in integer ns (SPEC.md:106 design decision).  CPU time per chain is split
evenly over its tasks.  Utilisations come from a fixed discrete table that
contains Table 1's 19/33/42 % rows and a ~15 % class below
the 0.1 exemption -- SURVEY.md Q20 reading.
"""
from __future__ import annotations

from typing import List, Sequence

import functools

import numpy as np

from .quantiles import inst_z_table
from .spec import MS, US, Chain, Kernel, Task, Workload

# Table 4: name -> (kernel count N_k, E_gpu ms)
TABLE4 = {
    "det3d": (41, 13.4),    # PointPillars 3D detection
    "pf": (16, 15.0),       # particle filtering
    "det2d": (323, 19.8),   # YOLOX 2D detection
    "face": (225, 7.1),     # face detection
    "sign": (65, 10.4),     # traffic-sign classification
    "seg": (63, 11.5),      # FCN segmentation
    "path": (256, 8.0),     # path finding
    "icp": (40, 21.3),      # ICP registration
    "calib": (133, 11.2),   # online calibration
    "llama": (1106, 17.8),  # LLaMA2 text generation
}

# Table 2: (period ms, D ms, Ecpu ms, Ecpu sigma, Egpu ms, Egpu sigma, tasks)
TABLE2 = [
    (150, 120, 17.4, 4.9, 28.4, 3.0, ("det3d", "pf")),             # C0
    (150, 120, 16.2, 3.2, 28.4, 3.1, ("det3d", "pf")),             # C1
    (500, 120, 21.0, 4.6, 27.0, 1.3, ("det2d", "face")),           # C2
    (200, 120, 20.2, 1.7, 30.2, 1.3, ("det2d", "sign")),           # C3
    (150, 120, 21.8, 2.7, 19.5, 2.8, ("seg", "path")),             # C4
    (200, 120, 20.2, 1.7, 30.2, 1.3, ("det2d", "sign")),           # C5
    (200, 120, 21.8, 2.7, 19.5, 2.8, ("seg", "path")),             # C6
    (500, 120, 21.0, 4.6, 27.0, 1.3, ("det2d", "face")),           # C7
    (200, 120, 21.3, 3.9, 19.7, 2.9, ("icp", "path")),             # C8
    (500, 120, 11.2, 1.4, 46.1, 4.2, ("det3d", "icp", "calib")),   # C9
    (5000, 200, 17.8, 4.6, 6.7, 2.9, ("llama",)),                  # C10
]

# Discrete utilisation table (per-mille, probability) -- SURVEY.md Q20 reading.
UTIL_TABLE = ((50, 0.15), (190, 0.15), (330, 0.20), (420, 0.20), (600, 0.15), (800, 0.10), (1000, 0.05))


def _ns(ms: float) -> int:
    return int(round(ms * MS))


def split_exact(total: int, weights: Sequence[float]) -> List[int]:
    """Integer split of ``total`` proportional to ``weights``; the remainder goes to the last part."""
    w = np.asarray(weights, dtype=np.float64)
    parts = [int(np.floor(total * x / w.sum())) for x in w[:-1]]
    parts.append(total - sum(parts))
    return parts


def synth_kernel_times(n: int, total_ns: int, rng: np.random.Generator, sigma: float = 1.2) -> List[int]:
    """n positive integer durations summing exactly to total_ns (truncated log-normal, rescaled)."""
    if n == 1:
        return [total_ns]
    z = np.clip(rng.standard_normal(n), -3.0, 3.0)
    x = np.exp(sigma * z)
    d = np.maximum(1, np.floor(x / x.sum() * total_ns)).astype(np.int64)
    # final-element adjustment on the largest kernel keeps every duration >= 1
    j = int(np.argmax(d))
    d[j] += total_ns - int(d.sum())
    assert d[j] >= 1 and int(d.sum()) == total_ns
    return [int(v) for v in d]


def paper11(template_seed: int = 0x5EED0002, chains: Sequence[int] = tuple(range(11))) -> Workload:
    rng = np.random.default_rng(template_seed)
    util_vals = np.array([u for u, _ in UTIL_TABLE])
    util_p = np.array([p for _, p in UTIL_TABLE])
    out = []
    for ci, (period, dl, ecpu, scpu, egpu, sgpu, names) in enumerate(TABLE2):
        gpu_parts = split_exact(_ns(egpu), [TABLE4[n][1] for n in names])
        cpu_parts = split_exact(_ns(ecpu), [1.0] * len(names))
        tasks = []
        for name, g_ns, c_ns in zip(names, gpu_parts, cpu_parts):
            nk = TABLE4[name][0]
            durs = synth_kernel_times(nk, g_ns, rng)
            utils = rng.choice(util_vals, size=nk, p=util_p)
            ks = [Kernel(d, d, int(u)) for d, u in zip(durs, utils)]
            tasks.append(Task(c_ns, c_ns, ks))
        if ci in chains:
            out.append(Chain(period * MS, dl * MS, 0, tasks,
                             cpu_sigma_ppm=int(round(scpu / ecpu * 1e6)),
                             gpu_sigma_ppm=int(round(sgpu / egpu * 1e6))))
    return Workload(chains=out, inst_quantiles_q16=inst_z_table())


def paper11_variants(num_variants: int = 64, template_seed: int = 0x5EED0002,
                     chains: Sequence[int] = tuple(range(11))) -> Workload:
    """paper11 with num_variants kernel-record sets (SURVEY.md §8(d) cfg 2: "64 templates, scenario s
    uses template s mod 64"; R33): set v is the kernel synthesis of template seed
    template_seed + v -- same chains, tasks, kernel counts and per-task totals, different per-kernel
    durations and utilisations.  Set 0 is paper11(template_seed)."""
    w = paper11(template_seed, chains)
    w.kernel_variants = [[Kernel(*r) for r in _kernel_rows(template_seed + v, tuple(chains))]
                         for v in range(1, num_variants)]
    return w


@functools.lru_cache(maxsize=256)
def _kernel_rows(template_seed: int, chains: tuple) -> tuple:
    return tuple((k.nominal_ns, k.estimate_ns, k.util_permille, k.flags)
                 for ch in paper11(template_seed, chains).chains for t in ch.tasks for k in t.kernels)


def toy2() -> Workload:
    """BASELINE.json configs[0]: 2 chains (1 tight, 1 loose), 3 tasks x 5 kernels, 2 streams.

    Parameters from SURVEY.md §8(d) cfg 1: chain 0 P=100 ms D=25 ms, CPU 1 ms per
    task, kernels [1.0,0.5,2.0,0.5,1.0] ms with u [600,300,900,50,600]; chain 1
    P=250 ms D=250 ms, CPU 2 ms per task, kernels [4,4,8,4,4] ms at u=800;
    lambda = sigma = 20 us, no AKB cost, no jitter, factors 1.0.
    """
    k0 = [(1.0, 600), (0.5, 300), (2.0, 900), (0.5, 50), (1.0, 600)]
    k1 = [(4.0, 800), (4.0, 800), (8.0, 800), (4.0, 800), (4.0, 800)]
    t0 = [Task(1 * MS, 1 * MS, [Kernel(_ns(d), _ns(d), u) for d, u in k0]) for _ in range(3)]
    t1 = [Task(2 * MS, 2 * MS, [Kernel(_ns(d), _ns(d), u) for d, u in k1]) for _ in range(3)]
    return Workload(chains=[Chain(100 * MS, 25 * MS, 0, t0), Chain(250 * MS, 250 * MS, 0, t1)],
                    num_prio=2, launch_ns=20 * US, launch_akb_ns=0, sync_lo_ns=20 * US,
                    sync_hi_ns=20 * US, jitter_ns=0)


def w1() -> Workload:
    """Fixture W1: two chains, lambda = sigma = 0, NUM_PRI = 2, one instance each."""
    a = Chain(1000 * MS, 8 * MS, 0, [Task(1 * MS, 1 * MS, [Kernel(2 * MS, 2 * MS, 1000), Kernel(2 * MS, 2 * MS, 1000)])])
    b = Chain(1000 * MS, 100 * MS, 0, [Task(1_500_000, 1_500_000, [Kernel(5 * MS, 5 * MS, 1000)])])
    return Workload(chains=[a, b], num_prio=2, launch_ns=0, launch_akb_ns=0, sync_lo_ns=0, sync_hi_ns=0, jitter_ns=0)


def w2() -> Workload:
    """Fixture W2: one chain, CPU 1 ms, 8 kernels x 0.2 ms, lambda 0.1 ms, sigma 0.05 ms."""
    ks = [Kernel(200 * US, 200 * US, 1000) for _ in range(8)]
    return Workload(chains=[Chain(1000 * MS, 100 * MS, 0, [Task(1 * MS, 1 * MS, ks)])], num_prio=6,
                    launch_ns=100 * US, launch_akb_ns=0, sync_lo_ns=50 * US, sync_hi_ns=50 * US, jitter_ns=0)


def w3() -> Workload:
    """Fixture W3: one chain, D' = 4.5 ms, 2 tasks of (CPU 1 ms + one kernel estimated 1 ms); k0 actually 1.8 ms."""
    t0 = Task(1 * MS, 1 * MS, [Kernel(1_800_000, 1 * MS, 1000)])
    t1 = Task(1 * MS, 1 * MS, [Kernel(1 * MS, 1 * MS, 1000)])
    return Workload(chains=[Chain(1000 * MS, 4_500_000, 0, [t0, t1])], num_prio=6,
                    launch_ns=0, launch_akb_ns=0, sync_lo_ns=0, sync_hi_ns=0, jitter_ns=0)


def w4() -> Workload:
    """Fixture W4 (tests/golden/w4.json): three chains for the kernel-collision metric (R24)."""
    a = Chain(1000 * MS, 6 * MS, 0, [Task(1 * MS, 1 * MS, [Kernel(1 * MS, 1 * MS, 1000), Kernel(1 * MS, 1 * MS, 1000)])])
    b = Chain(1000 * MS, 100 * MS, 0, [Task(500 * US, 500 * US, [Kernel(4 * MS, 4 * MS, 1000)])])
    b2 = Chain(1000 * MS, 100 * MS, 0, [Task(600 * US, 600 * US, [Kernel(4 * MS, 4 * MS, 1000)])])
    return Workload(chains=[a, b, b2], num_prio=2, launch_ns=0, launch_akb_ns=0, sync_lo_ns=0, sync_hi_ns=0,
                    jitter_ns=0)


def w6(two_chains: bool = True) -> Workload:
    """Fixture W6 (tests/golden/w6.json): cudaFree device barriers (R28)."""
    a = Chain(1000 * MS, 100 * MS, 0, [Task(1 * MS, 1 * MS, [Kernel(2 * MS, 2 * MS, 500)], frees=True)])
    b = Chain(1000 * MS, 100 * MS, 0, [Task(500 * US, 500 * US, [Kernel(5 * MS, 5 * MS, 500), Kernel(1 * MS, 1 * MS, 500)])])
    return Workload(chains=[a, b] if two_chains else [a], num_prio=2, launch_ns=0, launch_akb_ns=0, sync_lo_ns=0,
                    sync_hi_ns=0, jitter_ns=0, free_ns=188 * US)


def w7(cores: int = 1) -> Workload:
    """Fixture W7 (tests/golden/w7.json): two chains sharing CPU cores (R29)."""
    a = Chain(1000 * MS, 20 * MS, 0, [Task(4 * MS, 4 * MS, [Kernel(1 * MS, 1 * MS, 1000)])])
    b = Chain(1000 * MS, 6 * MS, 1 * MS, [Task(2 * MS, 2 * MS, [Kernel(1 * MS, 1 * MS, 1000)])])
    return Workload(chains=[a, b], num_prio=2, launch_ns=0, launch_akb_ns=0, sync_lo_ns=0, sync_hi_ns=0,
                    jitter_ns=0, cpu_cores=cores)


def w8(alpha_permille: int = 600) -> Workload:
    """Fixture W8 (tests/golden/w8.json): kernel contention slow-down (R30)."""
    a = Chain(1000 * MS, 100 * MS, 0, [Task(500 * US, 500 * US, [Kernel(4 * MS, 4 * MS, 500)])])
    b = Chain(1000 * MS, 100 * MS, 0, [Task(1 * MS, 1 * MS, [Kernel(2 * MS, 2 * MS, 500)])])
    return Workload(chains=[a, b], num_prio=2, launch_ns=0, launch_akb_ns=0, sync_lo_ns=0, sync_hi_ns=0,
                    jitter_ns=0, contention_permille=alpha_permille)


def contention_pair(co_run: bool = True, alpha_permille: int = 0, template_seed: int = 0x5EED0007) -> Workload:
    """Fig. fig:13_cdf set-up: 2D detection (YOLOX, Table 4: 323 kernels,
    19.8 ms) alone or sharing the GPU with 3D detection (PointPillars: 41 kernels, 13.4 ms).
    Chain 0 = 2D detection with the tighter deadline (the higher static priority), 2 ms CPU
    segment; chain 1 = 3D detection, 2 ms CPU segment; both every 50 ms with 15 ms jitter."""
    rng = np.random.default_rng(template_seed)
    util_vals = np.array([u for u, _ in UTIL_TABLE])
    util_p = np.array([p for _, p in UTIL_TABLE])
    chains = []
    for name, dl in (("det2d", 60), ("det3d", 120)):
        nk, egpu = TABLE4[name]
        durs = synth_kernel_times(nk, _ns(egpu), rng)
        utils = rng.choice(util_vals, size=nk, p=util_p)
        ks = [Kernel(d, d, int(u)) for d, u in zip(durs, utils)]
        chains.append(Chain(50 * MS, dl * MS, 0, [Task(2 * MS, 2 * MS, ks)]))
    return Workload(chains=chains if co_run else chains[:1], num_prio=6, jitter_ns=15 * MS,
                    contention_permille=alpha_permille)


def w9(copies: bool = True) -> Workload:
    """Fixture W9 (tests/golden/w9.json): memcpy operations on the copy engine (R31).
    With copies=False the same operations are plain kernels at u 500."""
    f = 1 if copies else 0
    a = Chain(1000 * MS, 100 * MS, 0, [Task(1 * MS, 1 * MS, [Kernel(1 * MS, 1 * MS, 500, f), Kernel(2 * MS, 2 * MS, 500)])])
    b = Chain(1000 * MS, 100 * MS, 0, [Task(500 * US, 500 * US, [Kernel(2 * MS, 2 * MS, 500, f), Kernel(1 * MS, 1 * MS, 500)])])
    return Workload(chains=[a, b], num_prio=2, launch_ns=0, launch_akb_ns=0, sync_lo_ns=0, sync_hi_ns=0, jitter_ns=0)


def w10() -> Workload:
    """Fixture W10 (tests/golden/w10.json): a zero-cost, already-satisfied OVERLAP sync (PAPER.md:504-509,
    sigma = 0 at the low end of P:494's range made exact) -- the same-t continuation of DESIGN.md R21.
    Chain A overlaps its batches; chain B is urgent and becomes AKB-active at the very time A's
    satisfied sync returns."""
    a = Chain(1000 * MS, 100 * MS, 0, [Task(1 * MS, 1 * MS, [Kernel(50 * US, 600 * US, 100),
                                                            Kernel(200 * US, 600 * US, 100),
                                                            Kernel(200 * US, 600 * US, 500)])])
    b = Chain(1000 * MS, 4 * MS, 0, [Task(1_100_000, 1_100_000, [Kernel(1 * MS, 1 * MS, 100)])])
    return Workload(chains=[a, b], num_prio=2, launch_ns=100 * US, launch_akb_ns=0, sync_lo_ns=0, sync_hi_ns=0,
                    jitter_ns=0)


W11_ESTIMATES_MS = (49, 58, 52, 36, 53, 44)


def w11() -> Workload:
    """Fixture W11 (tests/golden/w11.json): UrgenGo's rank normalisation with NUM_PRI = 6 inside a
    simulation ("normalize ... to (1, NUM_PRI-1)").  Six chains bind
    one after another (CPU segments of 1..6 ms) while the earlier ones stay AKB-active; kernel
    estimates are chosen so the laxities at binding are 50, 40, 45, 60, 42, 50 ms.  Each kernel
    takes 300 permille, so only three run at once and the levels decide the later dispatch order."""
    chains = [Chain(1000 * MS, 100 * MS, 0, [Task((i + 1) * MS, 0, [Kernel(50 * MS, e * MS, 300)])])
              for i, e in enumerate(W11_ESTIMATES_MS)]
    return Workload(chains=chains, num_prio=6, launch_ns=0, launch_akb_ns=0, sync_lo_ns=0, sync_hi_ns=0,
                    jitter_ns=0)
