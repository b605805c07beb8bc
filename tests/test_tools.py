"""Host-side logic of the measurement tools (no GPU)."""
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load(name):
    spec = importlib.util.spec_from_file_location(name, os.path.join(ROOT, "tools", f"{name}.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_parity_sample_follows_baseline_plan():
    """configs[2]-[4] check the first 256, the last 256 and every 9973rd index."""
    m = _load("run_configs")
    s = m.sample_indices(0, 1_000_000, full=False)
    assert s[:256] == list(range(256)) and s[-256:] == list(range(1_000_000 - 256, 1_000_000))
    assert all(i in s for i in range(0, 1_000_000, 9973))
    assert len(s) == len(set(s)) == 256 + 256 + len([i for i in range(256, 1_000_000 - 256) if i % 9973 == 0])
    assert m.sample_indices(5, 300, full=False) == list(range(5, 305))
    assert m.sample_indices(10, 7, full=True) == list(range(10, 17))
