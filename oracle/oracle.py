"""ctypes wrapper of the CPU oracle (oracle/urg_oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, never by the product package.
The shared object is compiled on demand with gcc (plain C, -O2, no CUDA).
"""
from __future__ import annotations

import ctypes as ct
import os
import subprocess
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from workloads.spec import RECORD_WORDS, Batch, Policy, Workload, agg_words

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "urg_oracle.c")
_LIB = os.path.join(_HERE, "liburg_oracle.so")

TRACE_KINDS = {1: "STEP", 2: "INST_START", 3: "TASK_START", 4: "EVAL", 5: "DELAY", 6: "BIND", 7: "ENQUEUE",
               8: "DISPATCH", 9: "RETIRE", 10: "SYNC_CALL", 11: "SYNC_RET", 12: "FREE_CLOSE",
               13: "INST_DONE", 14: "EARLY_EXIT", 15: "COLLISION", 16: "FREE_CALL", 17: "FREE_START",
               18: "FREE_RET", 19: "CPU_RUN", 20: "CPU_STOP",
               21: "PUBLISH", 22: "TAKE"}
TRACE_CODES = {v: k for k, v in TRACE_KINDS.items()}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-Wno-unused-parameter",
                               "-shared", "-fPIC", _SRC, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


class OrcInput(ct.Structure):
    _fields_ = [
        ("num_chains", ct.c_uint32),
        ("ch_period", ct.c_void_p), ("ch_deadline", ct.c_void_p), ("ch_offset", ct.c_void_p),
        ("ch_ntasks", ct.c_void_p), ("ch_cpu_sigma", ct.c_void_p), ("ch_gpu_sigma", ct.c_void_p),
        ("t_cpu_nom", ct.c_void_p), ("t_cpu_est", ct.c_void_p), ("t_nk", ct.c_void_p), ("t_flags", ct.c_void_p),
        ("k_nom", ct.c_void_p), ("k_est", ct.c_void_p), ("k_util", ct.c_void_p), ("k_flags", ct.c_void_p),
        ("num_prio", ct.c_uint32),
        ("launch_ns", ct.c_int64), ("launch_akb_ns", ct.c_int64), ("sync_lo_ns", ct.c_int64),
        ("sync_hi_ns", ct.c_int64), ("jitter_ns", ct.c_int64),
        ("inst_q16", ct.c_void_p), ("kern_q16", ct.c_void_p),
        ("rt_bin_ns", ct.c_int64), ("rt_bins", ct.c_uint32), ("free_ns", ct.c_int64), ("cpu_cores", ct.c_uint32),
        ("contention_permille", ct.c_uint32), ("task_exec", ct.c_uint32),
        ("num_variants", ct.c_uint32),
        ("kind", ct.c_uint32), ("flags", ct.c_uint32), ("sync_mode", ct.c_uint32),
        ("delta_eval_ns", ct.c_int64), ("lax_threshold_ns", ct.c_int64), ("sleep_ns", ct.c_int64),
        ("util_exempt_permille", ct.c_uint32),
        ("noise_permille", ct.c_uint32), ("cpu_ma_window", ct.c_uint32),
        ("seed", ct.c_uint64), ("scenario_begin", ct.c_uint64), ("scenario_count", ct.c_uint64),
        ("horizon_ns", ct.c_int64),
        ("fa_num", ct.c_uint32), ("fa_den", ct.c_uint32), ("fd_num", ct.c_uint32), ("fd_den", ct.c_uint32),
        ("ftight_permille", ct.c_uint32), ("tight_explicit", ct.c_uint32), ("tight_mask", ct.c_uint32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ct.CDLL(build())
        _lib.orc_run.restype = ct.c_int
        _lib.orc_run.argtypes = [ct.POINTER(OrcInput), ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_int64,
                                 ct.POINTER(ct.c_int64)]
        _lib.orc_calibrate.restype = ct.c_int64
        _lib.orc_calibrate.argtypes = [ct.POINTER(OrcInput), ct.c_int64, ct.POINTER(ct.c_int64)]
        _lib.orc_eq2_laxity.restype = ct.c_int64
        _lib.orc_eq2_laxity.argtypes = [ct.c_int64, ct.c_int64, ct.c_void_p, ct.c_uint32, ct.c_uint32,
                                        ct.c_void_p, ct.c_uint32, ct.c_uint32, ct.c_int64]
        _lib.orc_urgency_key.restype = ct.c_int64
        _lib.orc_urgency_key.argtypes = [ct.c_int64]
        _lib.orc_is_urgent.restype = ct.c_int
        _lib.orc_is_urgent.argtypes = [ct.c_int64, ct.c_int64]
        _lib.orc_rank.restype = None
        _lib.orc_rank.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_uint32, ct.c_void_p]
        _lib.orc_normalise_level.restype = ct.c_uint32
        _lib.orc_normalise_level.argtypes = [ct.c_uint32, ct.c_uint32, ct.c_uint32]
        _lib.orc_plan_batches.restype = None
        _lib.orc_plan_batches.argtypes = [ct.c_void_p, ct.c_uint32, ct.c_int64, ct.c_void_p]
        _lib.orc_overall_miss_ratio.restype = ct.c_double
        _lib.orc_overall_miss_ratio.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_uint32]
        _lib.orc_philox4x32_10.restype = None
        _lib.orc_philox4x32_10.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_void_p]
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _make_input(w: Workload, p: Policy, b: Batch):
    f = w.flat()
    keep = dict(f)
    inst = None if w.inst_quantiles_q16 is None else np.ascontiguousarray(w.inst_quantiles_q16, np.int32)
    kern = None if w.kern_quantiles_q16 is None else np.ascontiguousarray(w.kern_quantiles_q16, np.uint32)
    keep["inst"], keep["kern"] = inst, kern
    s = OrcInput(
        num_chains=w.num_chains,
        ch_period=_ptr(f["ch_period"]), ch_deadline=_ptr(f["ch_deadline"]), ch_offset=_ptr(f["ch_offset"]),
        ch_ntasks=_ptr(f["ch_ntasks"]), ch_cpu_sigma=_ptr(f["ch_cpu_sigma"]), ch_gpu_sigma=_ptr(f["ch_gpu_sigma"]),
        t_cpu_nom=_ptr(f["t_cpu_nom"]), t_cpu_est=_ptr(f["t_cpu_est"]), t_nk=_ptr(f["t_nk"]), t_flags=_ptr(f["t_flags"]),
        k_nom=_ptr(f["k_nom"]), k_est=_ptr(f["k_est"]), k_util=_ptr(f["k_util"]), k_flags=_ptr(f["k_flags"]),
        num_prio=w.num_prio, launch_ns=w.launch_ns, launch_akb_ns=w.launch_akb_ns,
        sync_lo_ns=w.sync_lo_ns, sync_hi_ns=w.sync_hi_ns, jitter_ns=w.jitter_ns,
        inst_q16=_ptr(inst), kern_q16=_ptr(kern), rt_bin_ns=w.rt_bin_ns, rt_bins=w.rt_bins, free_ns=w.free_ns,
        cpu_cores=w.cpu_cores, contention_permille=w.contention_permille, task_exec=w.executors,
        num_variants=w.num_variants,
        kind=p.kind, flags=p.flags, sync_mode=p.sync_mode, delta_eval_ns=p.delta_eval_ns,
        lax_threshold_ns=p.lax_threshold_ns, sleep_ns=p.sleep_ns, util_exempt_permille=p.util_exempt_permille,
        noise_permille=p.noise_permille, cpu_ma_window=p.cpu_ma_window,
        seed=b.seed, scenario_begin=b.scenario_begin, scenario_count=b.scenario_count, horizon_ns=b.horizon_ns,
        fa_num=b.fa_num, fa_den=b.fa_den, fd_num=b.fd_num, fd_den=b.fd_den,
        ftight_permille=b.ftight_permille, tight_explicit=b.tight_explicit, tight_mask=b.tight_mask,
    )
    return s, keep


@dataclass
class OracleResult:
    records: np.ndarray      # [count, C, 8] uint32
    agg: np.ndarray          # int64[agg_words]
    trace: Optional[np.ndarray]
    seconds: float

    @property
    def launches(self) -> int:
        return int(self.agg[-2])

    @property
    def steps(self) -> int:
        return int(self.agg[-1])


def run(w: Workload, p: Policy, b: Batch, trace_cap: int = 0) -> OracleResult:
    s, keep = _make_input(w, p, b)
    C = w.num_chains
    rec = np.zeros((b.scenario_count, C, RECORD_WORDS), np.uint32)
    agg = np.zeros(agg_words(C, w.rt_bins), np.int64)
    tr = np.zeros((trace_cap, 6), np.int64) if trace_cap else None
    tlen = ct.c_int64(0)
    t0 = time.perf_counter()
    rc = lib().orc_run(ct.byref(s), rec.ctypes.data, agg.ctypes.data, _ptr(tr), trace_cap, ct.byref(tlen))
    dt = time.perf_counter() - t0
    if rc != 0:
        raise ValueError(f"oracle rejected input (rc={rc})")
    del keep
    return OracleResult(rec, agg, None if tr is None else tr[: tlen.value].copy(), dt)


def calibration_samples(w: Workload, p: Policy, b: Batch, window_ns: int = 30_000_000_000):
    """Per-scenario calibration samples (laxities, in sampling order): list of int64 arrays."""
    s, keep = _make_input(w, p, b)
    f = lib().orc_calibration_samples
    f.restype = ct.c_int
    f.argtypes = [ct.POINTER(OrcInput), ct.c_int64, ct.c_void_p, ct.c_int64, ct.c_void_p]
    end = min(b.horizon_ns, window_ns)
    cap = end // 1_000_000 + 2
    L = np.zeros((b.scenario_count, cap), np.int64)
    n = np.zeros(b.scenario_count, np.int64)
    rc = f(ct.byref(s), window_ns, L.ctypes.data, cap, n.ctypes.data)
    del keep
    if rc != 0:
        raise ValueError(f"oracle rejected input (rc={rc})")
    return [L[j, : n[j]].copy() for j in range(b.scenario_count)]


def calibrate(w: Workload, p: Policy, b: Batch, window_ns: int = 30_000_000_000):
    """L_th from the samples of every scenario of `b`, pooled."""
    s, keep = _make_input(w, p, b)
    n = ct.c_int64(0)
    lth = lib().orc_calibrate(ct.byref(s), window_ns, ct.byref(n))
    del keep
    return int(lth), int(n.value)


# ---- thin access to the oracle's pure functions (for the pins) ----
def eq2_laxity(t_arr, D, est_gpu, n, est_cpu, m, t) -> int:
    g = np.ascontiguousarray(est_gpu, np.uint32)
    c = np.ascontiguousarray(est_cpu, np.uint32)
    return int(lib().orc_eq2_laxity(t_arr, D, g.ctypes.data, len(g), n, c.ctypes.data, len(c), m, t))


def urgency_key(L: int) -> int:
    return int(lib().orc_urgency_key(L))


def is_urgent(L: int, lth: int) -> bool:
    return bool(lib().orc_is_urgent(L, lth))


def rank(keys, chains) -> np.ndarray:
    k = np.ascontiguousarray(keys, np.int64)
    c = np.ascontiguousarray(chains, np.uint32)
    out = np.zeros(len(k), np.uint32)
    lib().orc_rank(k.ctypes.data, c.ctypes.data, len(k), out.ctypes.data)
    return out


def normalise_level(r: int, n_r: int, num_prio: int) -> int:
    return int(lib().orc_normalise_level(r, n_r, num_prio))


def plan_batches(est, delta_eval_ns: int) -> np.ndarray:
    e = np.ascontiguousarray(est, np.uint32)
    out = np.zeros(len(e), np.uint8)
    lib().orc_plan_batches(e.ctypes.data, len(e), delta_eval_ns, out.ctypes.data)
    return out


def overall_miss_ratio(miss, total) -> float:
    m = np.ascontiguousarray(miss, np.uint64)
    t = np.ascontiguousarray(total, np.uint64)
    return float(lib().orc_overall_miss_ratio(m.ctypes.data, t.ctypes.data, len(m)))


def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(c.ctypes.data, k.ctypes.data, out.ctypes.data)
    return out


def nearest_rank_lth(laxities, pct: int = 95) -> int:
    a = np.ascontiguousarray(laxities, np.int64).copy()
    f = lib().orc_nearest_rank_lth
    f.restype = ct.c_int64
    f.argtypes = [ct.c_void_p, ct.c_int64, ct.c_int64]
    return int(f(a.ctypes.data, len(a), pct))


def classical_rank(kind: int, tarr, D, R, G, Pp, self_idx: int, t: int) -> int:
    """Rank of item self_idx (chain id = index) under a classical policy (R27)."""
    f = lib().orc_classical_rank
    f.restype = ct.c_uint32
    f.argtypes = [ct.c_uint32] + [ct.c_void_p] * 5 + [ct.c_uint32, ct.c_uint32, ct.c_int64]
    arrs = [np.ascontiguousarray(x, np.int64) for x in (tarr, D, R, G, Pp)]
    return int(f(kind, *[a.ctypes.data for a in arrs], len(arrs[0]), self_idx, t))
