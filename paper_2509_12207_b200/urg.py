"""Thin ctypes binding of liburg.so (include/urg.h).  Argument marshalling only:
every step of the simulation runs in the CUDA kernel.  There is no CPU fallback:
if the library is missing this module raises.
"""
from __future__ import annotations

import ctypes as ct
import os
from typing import Optional

import numpy as np

from workloads.spec import Batch, Policy, Workload

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liburg.so")

URG_OK, URG_EINVAL, URG_ERANGE, URG_ENOMEM, URG_ECUDA, URG_EINTERNAL = 0, -1, -2, -3, -4, -5


class UrgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"urg status {status}: {msg}")
        self.status = status


class KernelDesc(ct.Structure):
    _fields_ = [("nominal_ns", ct.c_uint32), ("estimate_ns", ct.c_uint32),
                ("util_permille", ct.c_uint16), ("flags", ct.c_uint16)]


class TaskDesc(ct.Structure):
    _fields_ = [("cpu_nominal_ns", ct.c_uint32), ("cpu_estimate_ns", ct.c_uint32),
                ("num_kernels", ct.c_uint32), ("kernels", ct.POINTER(KernelDesc)), ("flags", ct.c_uint32)]


class ChainDesc(ct.Structure):
    _fields_ = [("period_ns", ct.c_int64), ("deadline_ns", ct.c_int64), ("offset_ns", ct.c_int64),
                ("num_tasks", ct.c_uint32), ("tasks", ct.POINTER(TaskDesc)),
                ("cpu_sigma_ppm", ct.c_uint32), ("gpu_sigma_ppm", ct.c_uint32)]


class WorkloadDesc(ct.Structure):
    _fields_ = [("num_chains", ct.c_uint32), ("chains", ct.POINTER(ChainDesc)), ("num_prio", ct.c_uint32),
                ("launch_ns", ct.c_int64), ("launch_akb_ns", ct.c_int64),
                ("sync_lo_ns", ct.c_int64), ("sync_hi_ns", ct.c_int64), ("jitter_ns", ct.c_int64),
                ("inst_quantiles_q16", ct.c_void_p), ("kern_quantiles_q16", ct.c_void_p),
                ("rt_bin_ns", ct.c_int64), ("rt_bins", ct.c_uint32), ("free_ns", ct.c_int64),
                ("cpu_cores", ct.c_uint32), ("contention_permille", ct.c_uint32), ("executors", ct.c_uint32),
                ("num_variants", ct.c_uint32), ("variant_kernels", ct.c_void_p)]

# urg_kernel_desc as a numpy record (12 B: u32 nominal, u32 estimate, u16 util, u16 flags)
_KDESC = np.dtype([("nominal_ns", "<u4"), ("estimate_ns", "<u4"), ("util_permille", "<u2"), ("flags", "<u2")])


class PolicyS(ct.Structure):
    _fields_ = [("kind", ct.c_uint32), ("flags", ct.c_uint32), ("sync_mode", ct.c_uint32),
                ("delta_eval_ns", ct.c_int64), ("lax_threshold_ns", ct.c_int64), ("sleep_ns", ct.c_int64),
                ("util_exempt_permille", ct.c_uint32), ("noise_permille", ct.c_uint32),
                ("cpu_ma_window", ct.c_uint32)]


class BatchS(ct.Structure):
    _fields_ = [("seed", ct.c_uint64), ("scenario_begin", ct.c_uint64), ("scenario_count", ct.c_uint64),
                ("horizon_ns", ct.c_int64), ("fa_num", ct.c_uint32), ("fa_den", ct.c_uint32),
                ("fd_num", ct.c_uint32), ("fd_den", ct.c_uint32), ("ftight_permille", ct.c_uint32),
                ("tight_explicit", ct.c_uint32), ("tight_mask", ct.c_uint32)]


class OutputsS(ct.Structure):
    _fields_ = [("records", ct.c_void_p), ("agg", ct.c_void_p)]


SYMBOLS = ["urg_create_workload", "urg_destroy_workload", "urg_agg_words", "urg_template_bytes", "urg_simulate_batch",
           "urg_simulate_batch_host", "urg_check", "urg_miss_ratios", "urg_last_error",
           "urg_calibration_words", "urg_calibrate"]

DEBUG_LIB_PATH = os.path.join(_HERE, "liburg_debug.so")
_lib = None
_lib_debug = None


def lib():
    """Load liburg.so (built by paper_2509_12207_b200.build / __graft_entry__.build)."""
    global _lib
    if _lib is None:
        # URG_LIB selects another build of the same library (liburg_stats.so, the profiling variant)
        _lib = _load(os.environ.get("URG_LIB") or LIB_PATH)
    return _lib


def lib_debug():
    """Load liburg_debug.so: the same kernels compiled with -DURG_DEBUG (device invariant checks and
    the one-scenario event trace).  A separate handle beside liburg.so; tests only."""
    global _lib_debug
    if _lib_debug is None:
        _lib_debug = _load(DEBUG_LIB_PATH)
        assert _lib_debug.urg_debug_build() == 1, "liburg_debug.so is not the debug build"
    return _lib_debug


def _load(path):
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                           "(the CUDA path has no CPU fallback)")
    if True:
        L = ct.CDLL(path)
        L.urg_create_workload.restype = ct.c_int
        L.urg_create_workload.argtypes = [ct.POINTER(WorkloadDesc), ct.POINTER(ct.c_void_p)]
        L.urg_destroy_workload.restype = None
        L.urg_destroy_workload.argtypes = [ct.c_void_p]
        L.urg_agg_words.restype = ct.c_uint64
        L.urg_agg_words.argtypes = [ct.c_void_p]
        L.urg_template_bytes.restype = ct.c_uint64
        L.urg_template_bytes.argtypes = [ct.c_void_p]
        L.urg_calibration_words.restype = ct.c_uint64
        L.urg_calibration_words.argtypes = [ct.c_void_p, ct.POINTER(BatchS), ct.c_int64]
        L.urg_calibrate.restype = ct.c_int
        L.urg_calibrate.argtypes = [ct.c_void_p, ct.POINTER(PolicyS), ct.POINTER(BatchS), ct.c_int64, ct.c_void_p,
                                    ct.c_uint64, ct.c_void_p, ct.c_void_p]
        for f in (L.urg_simulate_batch, L.urg_simulate_batch_host):
            f.restype = ct.c_int
            f.argtypes = [ct.c_void_p, ct.POINTER(PolicyS), ct.POINTER(BatchS), ct.POINTER(OutputsS), ct.c_void_p]
        L.urg_check.restype = ct.c_int
        L.urg_check.argtypes = [ct.c_void_p, ct.c_void_p, ct.POINTER(ct.c_int64)]
        L.urg_miss_ratios.restype = ct.c_int
        L.urg_miss_ratios.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.POINTER(ct.c_double)]
        L.urg_last_error.restype = ct.c_char_p
        L.urg_last_error.argtypes = []
        if hasattr(L, "urg_debug_stats"):
            L.urg_debug_stats.restype = ct.c_int
            L.urg_debug_stats.argtypes = [ct.c_void_p, ct.c_void_p]
        L.urg_debug_philox.restype = ct.c_int
        L.urg_debug_philox.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_void_p, ct.c_int, ct.c_void_p]
        L.urg_debug_set_trace.restype = ct.c_int
        L.urg_debug_set_trace.argtypes = [ct.c_void_p, ct.c_uint64, ct.c_uint64]
        L.urg_debug_build.restype = ct.c_int
        L.urg_debug_build.argtypes = []
    return L


def _check(status: int, L=None):
    if status != URG_OK:
        raise UrgError(status, (L or lib()).urg_last_error().decode())


def policy_struct(p: Policy) -> PolicyS:
    return PolicyS(p.kind, p.flags, p.sync_mode, p.delta_eval_ns, p.lax_threshold_ns, p.sleep_ns,
                   p.util_exempt_permille, p.noise_permille, p.cpu_ma_window)


def batch_struct(b: Batch) -> BatchS:
    return BatchS(b.seed, b.scenario_begin, b.scenario_count, b.horizon_ns, b.fa_num, b.fa_den, b.fd_num,
                  b.fd_den, b.ftight_permille, b.tight_explicit, b.tight_mask)


RECORD_WORDS_ = 8   # urg_outputs.records: 8 uint32 per (scenario, chain), include/urg.h


def _current_device() -> int:
    """The CUDA device urg_create_workload bound the workload to (cudaGetDevice at create)."""
    try:
        import torch
        return torch.cuda.current_device()
    except Exception:
        return 0


def _stream_handle(stream) -> Optional[int]:
    if stream is None:
        return None
    return int(getattr(stream, "cuda_stream", stream))


class DeviceWorkload:
    """urg_workload handle: the template resident in HBM (urg_create_workload)."""

    def __init__(self, w: Workload, debug: bool = False):
        """debug=True: the workload lives in liburg_debug.so (device invariant checks, event trace)."""
        self.spec = w
        self.L = lib_debug() if debug else lib()
        keep = []
        chains = (ChainDesc * w.num_chains)()
        for ci, ch in enumerate(w.chains):
            tasks = (TaskDesc * len(ch.tasks))()
            for ti, t in enumerate(ch.tasks):
                ks = (KernelDesc * len(t.kernels))(*[KernelDesc(k.nominal_ns, k.estimate_ns, k.util_permille, k.flags)
                                                     for k in t.kernels])
                keep.append(ks)
                tasks[ti] = TaskDesc(t.cpu_nominal_ns, t.cpu_estimate_ns, len(t.kernels), ks, 1 if t.frees else 0)
            keep.append(tasks)
            chains[ci] = ChainDesc(ch.period_ns, ch.deadline_ns, ch.offset_ns, len(ch.tasks), tasks,
                                   ch.cpu_sigma_ppm, ch.gpu_sigma_ppm)
        inst = None if w.inst_quantiles_q16 is None else np.ascontiguousarray(w.inst_quantiles_q16, np.int32)
        kern = None if w.kern_quantiles_q16 is None else np.ascontiguousarray(w.kern_quantiles_q16, np.uint32)
        var = None
        if w.kernel_variants:   # template variants 1..V-1 (R33), chain-major records
            var = np.array([(k.nominal_ns, k.estimate_ns, k.util_permille, k.flags)
                            for v in w.kernel_variants for k in v], dtype=_KDESC)
        self.desc = WorkloadDesc(w.num_chains, chains, w.num_prio, w.launch_ns, w.launch_akb_ns, w.sync_lo_ns,
                                 w.sync_hi_ns, w.jitter_ns, None if inst is None else inst.ctypes.data,
                                 None if kern is None else kern.ctypes.data, w.rt_bin_ns, w.rt_bins, w.free_ns,
                                 w.cpu_cores, w.contention_permille, w.executors, w.num_variants,
                                 None if var is None else var.ctypes.data)
        self._keep = (keep, chains, inst, kern, var)
        h = ct.c_void_p()
        self._chk(self.L.urg_create_workload(ct.byref(self.desc), ct.byref(h)))
        self.handle = h
        self.device = _current_device()
        self.num_chains = w.num_chains
        self.agg_words = int(self.L.urg_agg_words(h))
        self.template_bytes = int(self.L.urg_template_bytes(h))

    def _chk(self, status):
        _check(status, self.L)

    def close(self):
        if getattr(self, "handle", None):
            self.L.urg_destroy_workload(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- device buffers (torch tensors on the workload's CUDA device) --
    def _check_device_buffers(self, b: Batch, agg, records):
        """The kernel writes 8 words per (scenario, chain) into records and int64 atomics into agg:
        refuse buffers it would overrun or misread (wrong dtype, size, layout or device)."""
        import torch
        dev = torch.device("cuda", self.device)
        if not (isinstance(agg, torch.Tensor) and agg.dtype == torch.int64 and agg.is_contiguous()
                and agg.device == dev and agg.numel() == self.agg_words):
            raise ValueError(f"agg must be a contiguous int64 tensor of {self.agg_words} words on {dev}")
        if records is not None:
            need = b.scenario_count * self.num_chains * RECORD_WORDS_
            if not (isinstance(records, torch.Tensor) and records.dtype in (torch.int32, getattr(torch, "uint32", None))
                    and records.is_contiguous() and records.device == dev and records.numel() >= need):
                raise ValueError(f"records must be a contiguous 32-bit tensor of >= {need} words on {dev}")

    def simulate(self, p: Policy, b: Batch, agg, records=None, stream=None):
        """urg_simulate_batch: asynchronous on `stream`; adds into `agg` (int64 device tensor)."""
        self._check_device_buffers(b, agg, records)
        o = OutputsS(None if records is None else records.data_ptr(), agg.data_ptr())
        self._chk(self.L.urg_simulate_batch(self.handle, ct.byref(policy_struct(p)), ct.byref(batch_struct(b)),
                                        ct.byref(o), _stream_handle(stream)))

    # -- host buffers (numpy) --
    def simulate_host(self, p: Policy, b: Batch, agg: np.ndarray, records: Optional[np.ndarray] = None,
                      stream=None):
        """urg_simulate_batch_host: synchronous; agg (int64[agg_words]) is added into."""
        if not (isinstance(agg, np.ndarray) and agg.dtype == np.int64 and agg.flags.c_contiguous
                and agg.size == self.agg_words):
            raise ValueError(f"agg must be a C-contiguous int64 array of {self.agg_words} words")
        if records is not None:
            need = b.scenario_count * self.num_chains * RECORD_WORDS_
            if not (isinstance(records, np.ndarray) and records.dtype in (np.uint32, np.int32)
                    and records.flags.c_contiguous and records.size >= need):
                raise ValueError(f"records must be a C-contiguous 32-bit array of >= {need} words")
        o = OutputsS(None if records is None else records.ctypes.data, agg.ctypes.data)
        self._chk(self.L.urg_simulate_batch_host(self.handle, ct.byref(policy_struct(p)), ct.byref(batch_struct(b)),
                                             ct.byref(o), _stream_handle(stream)))

    def calibrate(self, p: Policy, b: Batch, window_ns: int = 30_000_000_000, stream=None):
        """urg_calibrate: L_th = 1/TH_urgent from the batch's pooled samples.
        Returns (L_th, number of samples, per-scenario sample lists)."""
        import torch
        bs = batch_struct(b)
        words = int(self.L.urg_calibration_words(self.handle, ct.byref(bs), window_ns))
        scratch = torch.zeros(words, dtype=torch.int64, device="cuda")
        res = torch.zeros(2, dtype=torch.int64, device="cuda")
        self._chk(self.L.urg_calibrate(self.handle, ct.byref(policy_struct(p)), ct.byref(bs), window_ns,
                                   scratch.data_ptr(), words, res.data_ptr(), _stream_handle(stream)))
        self.check(stream)
        r = res.cpu().numpy()
        sc = scratch.cpu().numpy()
        cnt = b.scenario_count
        cap = (min(b.horizon_ns, window_ns) // 1_000_000) + 2
        rows = [sc[cnt + j * cap: cnt + j * cap + int(sc[j])] for j in range(cnt)]
        return int(r[0]), int(r[1]), rows

    def trace(self, p: Policy, b: Batch, scenario: int, cap_rows: int = 1 << 20, stream=None):
        """Debug build only: simulate batch b and return the event trace of global scenario
        `scenario` as int64 rows (t, kind, lane, instance, a, b) (urg_debug_set_trace), with the
        batch's aggregates.  Rows of one lane are in its program order; lanes interleave."""
        import torch
        if self.L.urg_debug_build() != 1:
            raise RuntimeError("event traces need the debug build: DeviceWorkload(w, debug=True)")
        buf = torch.zeros(1 + 6 * cap_rows, dtype=torch.int64, device="cuda")
        agg = torch.zeros(self.agg_words, dtype=torch.int64, device="cuda")
        self._chk(self.L.urg_debug_set_trace(buf.data_ptr(), cap_rows, scenario))
        try:
            self.simulate(p, b, agg, None, stream=stream)
            self.check(stream)
        finally:
            self._chk(self.L.urg_debug_set_trace(None, 0, 0))
        h = buf.cpu().numpy()
        n = int(h[0])
        if n > cap_rows:
            raise RuntimeError(f"trace overflow: {n} rows > cap {cap_rows}")
        return h[1: 1 + 6 * n].reshape(n, 6).copy(), agg.cpu().numpy()

    def check(self, stream=None) -> None:
        s = ct.c_int64(0)
        self._chk(self.L.urg_check(self.handle, _stream_handle(stream), ct.byref(s)))

    def miss_ratios(self, agg_host: np.ndarray):
        per = np.zeros(self.num_chains, np.float64)
        ov = ct.c_double(0.0)
        a = np.ascontiguousarray(agg_host, np.int64)
        self._chk(self.L.urg_miss_ratios(self.handle, a.ctypes.data, per.ctypes.data, ct.byref(ov)))
        return per, ov.value


def philox_device(ctr, key, stream=None):
    """Device Philox4x32-10 of n (ctr, key) pairs (test hook for the known-answer vectors)."""
    import torch
    c = torch.as_tensor(np.ascontiguousarray(ctr, np.uint32).view(np.int32)).cuda()
    k = torch.as_tensor(np.ascontiguousarray(key, np.uint32).view(np.int32)).cuda()
    out = torch.zeros_like(c)
    n = c.shape[0]
    _check(lib().urg_debug_philox(c.data_ptr(), k.data_ptr(), out.data_ptr(), n, _stream_handle(stream)))
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint32)
