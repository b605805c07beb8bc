"""Build liburg.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

The simulation kernel (csrc/urg_sim.cuh) has one instantiation per (policy kind,
UrgenGo flags, per-kernel factor table, latency/throughput build); csrc/urg_sim_part.cu
is compiled once per slice of those rows, the objects in parallel, then linked with the
dispatch table (urg_sim.cu) and the C ABI (urg_api.cu) into one shared library.
"""
from __future__ import annotations

import os
import subprocess
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
PART_SRC = os.path.join(CSRC, "urg_sim_part.cu")
SOURCES = [os.path.join(CSRC, f) for f in ("urg_sim.cu", "urg_api.cu", "urg_sim_part.cu")]
HEADERS = [os.path.join(CSRC, f) for f in ("urg_layout.h", "urg_sim.cuh")] + \
          [os.path.join(os.path.dirname(HERE), "include", "urg.h")]
OUT = os.path.join(HERE, "liburg.so")
STATS_OUT = os.path.join(HERE, "liburg_stats.so")   # profiling variant (-DURG_STATS event-loop counters)
DEBUG_OUT = os.path.join(HERE, "liburg_debug.so")   # debug variant (-DURG_DEBUG: device invariants, event trace)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
ROWS = 38                                            # URG_SIM_ROWS in urg_sim.cuh
PARTS = [(r, r + 2) for r in range(0, 18, 2)] + [(18, 26), (26, 34), (34, 36), (36, 38)]   # urg_sim_part0..12


def needs_build(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return r.stderr


def _compile_all(out: str, defines, verbose: bool) -> str:
    extra = [f"-D{d}" for d in defines]
    with tempfile.TemporaryDirectory(prefix="urg_build_") as tmpd:
        jobs = []
        for k, (lo, hi) in enumerate(PARTS):
            o = os.path.join(tmpd, f"part{k}.o")
            jobs.append(([NVCC, *CFLAGS, *extra, f"-DURG_PART_LO={lo}", f"-DURG_PART_HI={hi}",
                          f"-DURG_PART_FN=urg_sim_part{k}", "-c", PART_SRC, "-o", o], o))
        for src in ("urg_sim.cu", "urg_api.cu"):
            o = os.path.join(tmpd, src.replace(".cu", ".o"))
            jobs.append(([NVCC, *CFLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", o], o))
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            logs = list(ex.map(lambda j: _run(j[0]), jobs))
        tmp = out + f".{os.getpid()}.tmp"
        _run([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *[o for _, o in jobs], "-o", tmp])
        os.replace(tmp, out)
    if verbose:
        print("\n".join(logs))
    return out


def build(force: bool = False, verbose: bool = False, stats: bool = False, debug: bool = False) -> str:
    out = STATS_OUT if stats else DEBUG_OUT if debug else OUT
    if force or needs_build(out):
        _compile_all(out, ["URG_STATS"] if stats else ["URG_DEBUG"] if debug else [], verbose)
    return out


def build_variant(name: str, defines) -> str:
    """An experiment build liburg_<name>.so with extra -D flags (A/B timing via URG_LIB)."""
    return _compile_all(os.path.join(HERE, f"liburg_{name}.so"), list(defines), False)


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(OUT)
