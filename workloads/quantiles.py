"""Quantile tables for per-scenario execution-time factors (input data, host-built).

Both simulators draw a 32-bit counter-based random word and index one of these
4096-entry tables with its top 12 bits; the tables themselves are plain input
data, built here once in double precision and shipped as integers so that the
CPU oracle and the GPU path see identical bits.

* ``inst_z_table``: quantiles of a standard normal truncated at +-3 sigma, in
  Q16.16 (int32).  The per-instance factor is 1 + z * sigma_rel, sigma_rel being
  Table 2's "+-" spread over the mean (read as one standard
  deviation, truncated at 3 sigma -- SPEC.md:108 design decision).
* ``pareto_table``: Pareto(alpha=1.5) per-kernel factor truncated at 64x and
  normalised to mean 1, in Q16.16 (uint32) -- the heavy-tail stress of
  BASELINE.json configs[3] ("kernel-duration jitter stress").
"""
from __future__ import annotations

import numpy as np
from scipy.stats import norm

TABLE_SIZE = 4096


def _midpoints() -> np.ndarray:
    return (np.arange(TABLE_SIZE, dtype=np.float64) + 0.5) / TABLE_SIZE


def inst_z_table(trunc: float = 3.0) -> np.ndarray:
    u = _midpoints()
    lo, hi = norm.cdf(-trunc), norm.cdf(trunc)
    z = norm.ppf(lo + u * (hi - lo))
    return np.round(z * 65536.0).astype(np.int32)


def pareto_table(alpha: float = 1.5, cap: float = 64.0) -> np.ndarray:
    u = _midpoints()
    x = np.minimum((1.0 - u) ** (-1.0 / alpha), cap)
    x = x / x.mean()
    return np.round(x * 65536.0).astype(np.uint32)


def unit_table() -> np.ndarray:
    return np.full(TABLE_SIZE, 65536, dtype=np.uint32)
