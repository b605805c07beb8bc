"""Plain input records for a batched UrgenGo policy simulation.

This module is the *input side* shared by the CPU oracle (``oracle/``) and the
CUDA path (``paper_2509_12207_b200/``).  It holds data only: chains, tasks,
kernels, device/launch parameters, policy knobs and batch parameters.  It
contains none of the method's arithmetic (no urgency, no suffix sums, no
random draws, no scheduling) -- each side implements that itself.

The shapes follow the paper's task-chain model:
  * a chain C has a period and an end-to-end deadline D, and is a sequence of
    tasks (§1; Table 2);
  * a task is one CPU segment followed by one GPU segment of kernels launched
    in order on one stream (§2, §4.1);
  * a kernel is a lookup-table record: profiled execution time and GPU
    utilisation (Table 1).
All times are integer nanoseconds; utilisation is integer per-mille.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

# ---- policy / mode identifiers (values of the C-ABI enums in include/urg.h) ----
FIFO, STATIC, URGENGO = 0, 1, 2
EDF, SJF, HRRN, LCUF = 3, 4, 5, 6   # classical policies of the policy study (R27)
F_BIND, F_DELAY, F_EARLY_EXIT = 1, 2, 4
F_COLLISIONS = 8           # count kernel collisions of urgent kernels (metric only; R24)
F_ALL = F_BIND | F_DELAY | F_EARLY_EXIT
SYNC_ASYNC, SYNC_EACH, SYNC_BATCHED, SYNC_OVERLAP = 0, 1, 2, 3
EXEC_CHAIN, EXEC_TASK = 0, 1   # one thread per chain (R6) / one executor per task (R32)

MS = 1_000_000
US = 1_000


@dataclass
class Kernel:
    nominal_ns: int            # profiled execution time E^gpu_k (actual before per-scenario factors)
    estimate_ns: int           # lookup-table estimate ~E^gpu_k used by Eq. 2
    util_permille: int         # U_k in per-mille of the GPU (Table 1 "U_k (%)" x 10)
    flags: int = 0             # bit 0: a memcpy on the copy engine, not a kernel (Table 3; R31)


@dataclass
class Task:
    cpu_nominal_ns: int        # CPU segment actual time (before per-scenario factor)
    cpu_estimate_ns: int       # ~E^cpu_j used by Eq. 2
    kernels: List[Kernel]
    frees: bool = False        # the task ends with cudaFree: a device-wide barrier (R28)


@dataclass
class Chain:
    period_ns: int
    deadline_ns: int
    offset_ns: int
    tasks: List[Task]
    cpu_sigma_ppm: int = 0     # per-instance CPU time spread (Table 2 "+-"), parts per million of the mean
    gpu_sigma_ppm: int = 0     # per-instance GPU time spread (Table 2 "+-")


@dataclass
class Workload:
    chains: List[Chain]
    num_prio: int = 6                  # NUM_PRI stream priorities
    launch_ns: int = 21_672            # lambda: CPU cost of one launch, 7 ms / 323 kernels
    launch_akb_ns: int = 500           # AKB update cost
    sync_lo_ns: int = 10 * US          # sigma range, 10-200 us per sync call
    sync_hi_ns: int = 200 * US
    jitter_ns: int = 15 * MS           # arrival jitter
    inst_quantiles_q16: Optional[np.ndarray] = None   # int32[4096] truncated-normal z quantiles, Q16.16
    kern_quantiles_q16: Optional[np.ndarray] = None   # uint32[4096] per-kernel factor quantiles, Q16.16
    rt_bin_ns: int = 1 * MS
    rt_bins: int = 1024
    free_ns: int = 188 * US            # cudaFree cost on an idle device (Table 5; R28)
    cpu_cores: int = 0                 # cores shared by the chains' threads, 0 = one each (8; R29)
    contention_permille: int = 0       # kernel slow-down per co-running utilisation (R30)
    executors: int = EXEC_CHAIN        # EXEC_TASK: one thread per task, depth-1 hand-over (R32)
    # template variants (R33): kernel-record sets 1..V-1, each a chain-major list of
    # total_kernels() records of the same structure; scenario s uses set s mod V (set 0 = the chains')
    kernel_variants: Optional[List[List[Kernel]]] = None

    @property
    def num_chains(self) -> int:
        return len(self.chains)

    def total_kernels(self) -> int:
        return sum(len(t.kernels) for c in self.chains for t in c.tasks)

    @property
    def num_variants(self) -> int:
        return 1 + len(self.kernel_variants or [])

    def flat(self) -> dict:
        """Flatten to SoA numpy arrays (chains, then tasks in chain order, then kernels)."""
        ch_period, ch_deadline, ch_offset, ch_ntasks, ch_csig, ch_gsig = [], [], [], [], [], []
        t_cpu_nom, t_cpu_est, t_nk, t_flags = [], [], [], []
        k_nom, k_est, k_util, k_flags = [], [], [], []
        for c in self.chains:
            ch_period.append(c.period_ns); ch_deadline.append(c.deadline_ns); ch_offset.append(c.offset_ns)
            ch_ntasks.append(len(c.tasks)); ch_csig.append(c.cpu_sigma_ppm); ch_gsig.append(c.gpu_sigma_ppm)
            for t in c.tasks:
                t_cpu_nom.append(t.cpu_nominal_ns); t_cpu_est.append(t.cpu_estimate_ns); t_nk.append(len(t.kernels))
                t_flags.append(1 if t.frees else 0)
                for k in t.kernels:
                    k_nom.append(k.nominal_ns); k_est.append(k.estimate_ns)
                    k_util.append(k.util_permille); k_flags.append(k.flags)
        n0 = len(k_nom)
        for var in self.kernel_variants or []:
            assert len(var) == n0, "every kernel variant has one record per kernel of the chains"
            for k in var:
                k_nom.append(k.nominal_ns); k_est.append(k.estimate_ns)
                k_util.append(k.util_permille); k_flags.append(k.flags)
        return dict(
            ch_period=np.asarray(ch_period, np.int64), ch_deadline=np.asarray(ch_deadline, np.int64),
            ch_offset=np.asarray(ch_offset, np.int64), ch_ntasks=np.asarray(ch_ntasks, np.uint32),
            ch_cpu_sigma=np.asarray(ch_csig, np.uint32), ch_gpu_sigma=np.asarray(ch_gsig, np.uint32),
            t_cpu_nom=np.asarray(t_cpu_nom, np.uint32), t_cpu_est=np.asarray(t_cpu_est, np.uint32),
            t_nk=np.asarray(t_nk, np.uint32), t_flags=np.asarray(t_flags, np.uint32),
            k_nom=np.asarray(k_nom, np.uint32), k_est=np.asarray(k_est, np.uint32),
            k_util=np.asarray(k_util, np.uint16), k_flags=np.asarray(k_flags, np.uint16),
        )


@dataclass
class Policy:
    kind: int = URGENGO
    flags: int = F_ALL
    sync_mode: int = SYNC_OVERLAP
    delta_eval_ns: int = 500 * US      # Delta_eval = 0.5 ms
    lax_threshold_ns: int = 20 * MS    # L_th = 1/TH_urgent; configs override
    sleep_ns: int = 1 * MS             # delay-loop sleep
    util_exempt_permille: int = 100    # U < 0.1 never delayed
    noise_permille: int = 0            # urgency-estimation noise, uniform per task instance (R25)
    cpu_ma_window: int = 0             # CPU-segment moving-average window W (R26), 0 = profiled


@dataclass
class Batch:
    seed: int = 0
    scenario_begin: int = 0
    scenario_count: int = 1
    horizon_ns: int = 1_000 * MS
    fa_num: int = 1
    fa_den: int = 1
    fd_num: int = 1
    fd_den: int = 1
    ftight_permille: int = 0
    tight_explicit: int = 0            # 1: use tight_mask instead of the per-scenario draw
    tight_mask: int = 0


RECORD_WORDS = 8   # per scenario, per chain: total, miss, early, unfinished, launches, rt_hash, sum_rt_lo, sum_rt_hi
REC_TOTAL, REC_MISS, REC_EARLY, REC_UNFIN, REC_LAUNCH, REC_HASH, REC_SUMRT_LO, REC_SUMRT_HI = range(8)
AGG_COUNTERS = 5   # per chain: total, miss, early, unfinished, sum_rt
RATIO_BINS = 101
COLL_BINS = 33     # kernel-collision histogram, bin = number of colliding tasks (2..32)


def agg_words(num_chains: int, rt_bins: int) -> int:
    """int64 words of the aggregate buffer: per chain [5 counters | rt_bins | 101 ratio bins], then the
    33-bin kernel-collision histogram, then 2 event counters (launch events, loop steps)."""
    return num_chains * (AGG_COUNTERS + rt_bins + RATIO_BINS) + COLL_BINS + 2


def collision_hist(agg, num_chains: int, rt_bins: int):
    """View of the collision histogram inside an aggregate buffer (index = number of colliding tasks)."""
    o = num_chains * (AGG_COUNTERS + rt_bins + RATIO_BINS)
    return agg[o: o + COLL_BINS]
