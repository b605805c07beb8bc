"""Build liburg.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(CSRC, f) for f in ("urg_sim.cu", "urg_api.cu")]
HEADERS = [os.path.join(CSRC, "urg_layout.h"), os.path.join(os.path.dirname(HERE), "include", "urg.h")]
OUT = os.path.join(HERE, "liburg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def needs_build(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


STATS_OUT = os.path.join(HERE, "liburg_stats.so")   # profiling variant (-DURG_STATS event-loop counters)


def build(force: bool = False, verbose: bool = False, stats: bool = False) -> str:
    out = STATS_OUT if stats else OUT
    if force or needs_build(out):
        tmp = out + f".{os.getpid()}.tmp"
        extra = ["-DURG_STATS"] if stats else []
        r = subprocess.run([NVCC, *FLAGS, *extra, *SOURCES, "-o", tmp], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(r.stderr)
        os.replace(tmp, out)
    return out


def build_variant(name: str, defines) -> str:
    """An experiment build liburg_<name>.so with extra -D flags (A/B timing via URG_LIB)."""
    out = os.path.join(HERE, f"liburg_{name}.so")
    tmp = out + f".{os.getpid()}.tmp"
    r = subprocess.run([NVCC, *FLAGS, *[f"-D{d}" for d in defines], *SOURCES, "-o", tmp], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(OUT)
