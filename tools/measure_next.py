"""Throughput of the §8(f) NEXT rows on the GPU next to the CPU oracle (profiles/<tag>_next.json).
usage: python tools/measure_next.py TAG"""
import json
import os
import sys
import time
from dataclasses import replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2509_12207_b200.urg import DeviceWorkload  # noqa: E402
from workloads import get_config  # noqa: E402
from workloads.spec import F_COLLISIONS, Policy  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
cfg = get_config("paper11")
w, base, b = cfg.workload(), cfg.policies["urgengo"], cfg.batch
out = {"workload": "paper11 (configs[1]) 1000 scenarios x 10 s", "rows": {}}
dw = DeviceWorkload(w)


def gpu_sim(p, reps=3, d=None):
    d = d or dw
    agg = torch.zeros(d.agg_words, dtype=torch.int64, device="cuda")
    ts = []
    for _ in range(reps + 1):
        agg.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); d.simulate(p, b, agg); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    d.check()
    ms = sorted(ts[1:])[len(ts[1:]) // 2]
    return int(agg[-2].item()), ms


def cpu_sim(p, n=2, wx=None):
    r = O.run(wx or w, p, replace(b, scenario_count=n))
    return r.launches, r.seconds


variants = {
    "UrgenGo (base)": base,
    "UrgenGo + collision metric (R24)": replace(base, flags=base.flags | F_COLLISIONS),
    "UrgenGo + 30% estimation noise (R25)": replace(base, noise_permille=300),
    "UrgenGo + W=8 CPU moving average (R26)": replace(base, cpu_ma_window=8),
}
for name, p in variants.items():
    L, ms = gpu_sim(p)
    cl, cs = cpu_sim(p)
    out["rows"][name] = {"gpu_launch_events_per_s": L / ms * 1e3, "gpu_ms": ms, "launch_events": L,
                         "oracle_1core_launch_events_per_s": cl / cs}
    print(name, out["rows"][name], flush=True)

# rows that change the workload (extended-model build)
from paper_2509_12207_b200 import sweep as SW  # noqa: E402
from workloads.spec import EXEC_TASK  # noqa: E402

wvars = {
    "EDF (R27)": (w, Policy(kind=3, flags=0, sync_mode=base.sync_mode)),
    "cudaFree at the end of 2 tasks (R28)": (SW.with_frees(w, 2), base),
    "8 shared CPU cores (R29)": (replace(w, cpu_cores=8), base),
    "contention alpha 500 permille (R30)": (replace(w, contention_permille=500), base),
    "H2D/D2H memcpys around every task (R31)": (SW.with_copies(w), base),
    "per-task executors (R32)": (replace(w, executors=EXEC_TASK), base),
}
for name, (wx, p) in wvars.items():
    d = DeviceWorkload(wx)
    L, ms = gpu_sim(p, d=d)
    d.close()
    cl, cs = cpu_sim(p, wx=wx)
    out["rows"][name] = {"gpu_launch_events_per_s": L / ms * 1e3, "gpu_ms": ms, "launch_events": L,
                         "oracle_1core_launch_events_per_s": cl / cs}
    print(name, out["rows"][name], flush=True)

# TH_urgent calibration (urg_calibrate) over the whole batch, 30 s window (= the 10 s horizon)
torch.cuda.synchronize()
t0 = time.perf_counter()
lth, n, _ = dw.calibrate(base, b)
dt = time.perf_counter() - t0
t1 = time.perf_counter()
olth, on = O.calibrate(w, base, replace(b, scenario_count=2))
odt = time.perf_counter() - t1
out["rows"]["TH_urgent calibration (urg_calibrate)"] = {
    "gpu_scenarios_per_s": b.scenario_count / dt, "gpu_s": dt, "lth_ns_1000_scenarios": lth, "samples": n,
    "oracle_1core_scenarios_per_s": 2 / odt, "note": "GPU time is host wall clock incl. scratch allocation and D2H"}
print(out["rows"]["TH_urgent calibration (urg_calibrate)"])
dw.close()
with open(os.path.join(ROOT, "profiles", f"{tag}_next.json"), "w") as f:
    json.dump(out, f, indent=1)
