"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, exports every
symbol include/urg.h declares, and rejects malformed descriptors with a field
locus before touching the GPU.  No compute calls (no GPU here)."""
import ctypes as ct
import os
import re

import pytest

from workloads import paper11, toy2
from workloads.spec import Chain, Kernel, Task, Workload

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2509_12207_b200 import build as B
    B.build()
    from paper_2509_12207_b200.urg import lib
    return lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "urg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(urg_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    syms = declared_symbols()
    assert {"urg_create_workload", "urg_simulate_batch", "urg_miss_ratios"} <= set(syms)
    for s in syms:
        assert hasattr(L, s), s


def test_sass_is_sm100a():
    import subprocess
    from paper_2509_12207_b200 import build as B
    B.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.OUT], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _create(w):
    from paper_2509_12207_b200.urg import DeviceWorkload, UrgError
    with pytest.raises(UrgError) as e:
        DeviceWorkload(w)
    return e.value


def test_validation_loci(L):
    w = toy2()
    w.chains[1].tasks[2].kernels[3].nominal_ns = 0
    e = _create(w)
    assert e.status == -1 and "chains[1].tasks[2].kernels[3].nominal_ns" in str(e)
    w = toy2()
    w.chains[0].tasks[1].kernels[0].util_permille = 1001
    assert "chains[0].tasks[1].kernels[0].util_permille" in str(_create(w))
    w = toy2()
    w.chains[0].period_ns = 0
    assert "chains[0].period_ns" in str(_create(w))
    w = toy2()
    w.chains[1].tasks = []
    assert "chains[1].num_tasks" in str(_create(w))
    w = toy2()
    w.num_prio = 9
    assert "num_prio" in str(_create(w))
    w = Workload(chains=[paper11().chains[0]] * 33)
    e = _create(w)
    assert e.status == -2 and "exceeds 32" in str(e)
    w = Workload(chains=[])
    assert "num_chains" in str(_create(w))


def test_task_executor_limits(L):
    """Per-task executors (R32): one lane per task, so at most 32 tasks; unknown modes refused."""
    from workloads.spec import EXEC_TASK
    w = paper11()                      # 22 tasks: accepted
    w.executors = EXEC_TASK
    w.chains = w.chains + w.chains[:6]   # 34 tasks
    e = _create(w)
    assert e.status == -2 and "per-task executors" in str(e)
    w = paper11()
    w.executors = 2
    assert "executors" in str(_create(w))


def test_template_variant_validation(L):
    """Template variants (R33): records validated with their locus; memcpy flags are structural."""
    from workloads.spec import Kernel as K
    w = toy2()
    n = w.total_kernels()
    w.kernel_variants = [[K(1000, 1000, 500) for _ in range(n)] for _ in range(2)]
    w.kernel_variants[1][7] = K(0, 1000, 500)
    e = _create(w)
    assert e.status == -1 and "variant_kernels[2][7].nominal_ns" in str(e)
    w.kernel_variants[1][7] = K(1000, 1000, 500, 1)
    assert "variant_kernels[2][7].flags" in str(_create(w))


def test_cudafree_needs_positive_cost(L):
    from workloads import w6
    w = w6(False)
    w.free_ns = 0
    e = _create(w)
    assert e.status == -1 and "free_ns must be > 0" in str(e)


def test_template_over_shared_memory_budget(L):
    """A template larger than the shared-memory budget is refused with URG_ERANGE before any
    device work (SURVEY.md §8(b) 'template larger than the smem budget -> URG_ERANGE')."""
    tasks = [Task(1000, 1000, [Kernel(1000, 1000, 500)])] * 10_500   # 10.5k task records x 16 B > 160 KB
    w = Workload(chains=[Chain(100_000_000, 50_000_000, 0, tasks)])
    e = _create(w)
    assert e.status == -2 and "shared memory" in str(e)


def test_header_documents_every_entry_point():
    """Each entry point declared in include/urg.h has a comment block citing the paper or the
    design document (argument meaning, layout, ownership and errors live there)."""
    src = open(os.path.join(ROOT, "include", "urg.h")).read()
    for sym in declared_symbols():
        i = src.index(sym + "(")
        block = src[max(0, i - 1500):i]
        assert "/*" in block, sym
    assert src.count("PAPER.md") >= 10
