"""The five BASELINE.json configs as (workload, policies, batch) input recipes.

Seeds: 0x5EED0000 + config id.  L_th (= 1/TH_urgent) for the
paper-shaped configs is the value ``oracle/calibrate.py`` derives with the
SURVEY.md Q5 recipe and writes to ``calibrated.json``; the
GPU path only reads the stored number.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field, replace
from typing import Callable, Dict, List

from .quantiles import pareto_table
from .spec import (F_ALL, FIFO, MS, STATIC, SYNC_ASYNC, SYNC_OVERLAP, URGENGO, Batch, Policy,
                   Workload)
from .templates import paper11_variants, toy2

_CAL = os.path.join(os.path.dirname(__file__), "calibrated.json")


def calibrated_lth(name: str, default: int = 20 * MS) -> int:
    if os.path.exists(_CAL):
        with open(_CAL) as f:
            return int(json.load(f).get(name, default))
    return default


def urgengo(lth: int) -> Policy:
    return Policy(kind=URGENGO, flags=F_ALL, sync_mode=SYNC_OVERLAP, lax_threshold_ns=lth)


def fifo() -> Policy:
    return Policy(kind=FIFO, flags=0, sync_mode=SYNC_ASYNC)


def static() -> Policy:
    return Policy(kind=STATIC, flags=0, sync_mode=SYNC_ASYNC)


@dataclass
class Config:
    name: str
    workload: Callable[[], Workload]
    policies: Dict[str, Policy]
    batch: Batch
    note: str = ""
    sweep: List[Batch] = field(default_factory=list)


def _cfg1() -> Config:
    return Config("toy2", toy2, {"urgengo": Policy(kind=URGENGO, flags=F_ALL, sync_mode=SYNC_OVERLAP,
                                                   lax_threshold_ns=10 * MS),
                                 "fifo": fifo(), "static": static()},
                  Batch(seed=0x5EED0001, scenario_count=1, horizon_ns=1000 * MS),
                  "configs[0]: 2 chains, 3 tasks x 5 kernels, 2 streams, 1 s, 1 scenario")


def paper11_64():
    """The Table-2 workload with 64 template variants: scenario s uses template s mod 64
    (SURVEY.md §8(d) cfg 2; R33).  Template 0 is paper11(0x5EED0002)."""
    return paper11_variants(64)


def _cfg2() -> Config:
    lth = calibrated_lth("paper11")
    return Config("paper11", paper11_64, {"urgengo": urgengo(lth), "fifo": fifo(), "static": static()},
                  Batch(seed=0x5EED0002, scenario_count=1000, horizon_ns=10_000 * MS, ftight_permille=400),
                  "configs[1]: 11 chains (Table 2), 10 s horizon, 1k randomized scenarios")


def _cfg3() -> Config:
    lth = calibrated_lth("paper11")
    # utilisation u = sum_c Egpu_c / P'_c is 1.2082 at f_a = 1 (Table 2); f_a = u / 1.2082 (rational)
    sweep = [Batch(seed=0x5EED0003, scenario_count=100_000, horizon_ns=10_000 * MS, ftight_permille=400,
                   fa_num=u10 * 1000, fa_den=12082) for u10 in range(5, 13)]
    return Config("usweep", paper11_64, {"urgengo": urgengo(lth), "fifo": fifo(), "static": static()},
                  sweep[0], "configs[2]: utilisation sweep 0.5-1.2 x 100k scenarios", sweep)


def _paper11_heavy() -> Workload:
    w = paper11_64()
    w.kern_quantiles_q16 = pareto_table()
    return w


def _cfg4() -> Config:
    lth = calibrated_lth("paper11")
    return Config("jitter", _paper11_heavy, {"urgengo": urgengo(lth), "fifo": fifo()},
                  Batch(seed=0x5EED0004, scenario_count=1_000_000, horizon_ns=60_000 * MS, ftight_permille=400),
                  "configs[3]: heavy-tailed kernel times (Pareto 1.5, cap 64x), 1M scenarios, 60 s")


def _cfg5() -> Config:
    lth = calibrated_lth("paper11")
    return Config("scaleout", paper11_64, {"urgengo": urgengo(lth)},
                  Batch(seed=0x5EED0005, scenario_count=100_000_000, horizon_ns=1_000 * MS, ftight_permille=400),
                  "configs[4]: 100M scenarios, 1 s horizon, sharded over GPUs")


CONFIGS = {"toy2": _cfg1, "paper11": _cfg2, "usweep": _cfg3, "jitter": _cfg4, "scaleout": _cfg5}


def get_config(name: str) -> Config:
    return CONFIGS[name]()


def with_batch(b: Batch, **kw) -> Batch:
    return replace(b, **kw)
