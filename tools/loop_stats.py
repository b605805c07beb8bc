"""Event-loop counters of one bench-sized launch (profiling build liburg_stats.so).
usage: python tools/loop_stats.py [config] [policy] [scenarios]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_12207_b200 import build as B  # noqa: E402

os.environ["URG_LIB"] = B.build(stats=True)
import numpy as np  # noqa: E402
import torch  # noqa: E402
from dataclasses import replace  # noqa: E402
from paper_2509_12207_b200.urg import DeviceWorkload, lib  # noqa: E402
from workloads import get_config  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "paper11")
pol = sys.argv[2] if len(sys.argv) > 2 else "urgengo"
b = cfg.batch
if len(sys.argv) > 3:
    b = replace(b, scenario_count=int(sys.argv[3]))
with DeviceWorkload(cfg.workload()) as dw:
    agg = torch.zeros(dw.agg_words, dtype=torch.int64, device="cuda")
    dw.simulate(cfg.policies[pol], b, agg)
    torch.cuda.synchronize()
    out = np.zeros(4, np.uint64)
    assert lib().urg_debug_stats(dw.handle, out.ctypes.data) == 0
    a = agg.cpu().numpy()
single, multi, disp, rebase = (int(x) for x in out)
steps, launches = int(a[-1]), int(a[-2])
print(f"{cfg.name}/{pol}: steps {steps} launches {launches} | single-chain steps {single} multi-chain {multi} "
      f"| Phase C runs {disp} ({disp / max(steps, 1):.3f}/step) | rebases {rebase}")
