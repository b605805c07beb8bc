"""A/B timing of library variants on one workload (each in a fresh process via URG_LIB).
usage: python tools/ab.py CONFIG POLICY SCENARIOS lib1.so lib2.so ...
Prints ms per launch (median of 3) and checks every variant's records equal the first's."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, ROOT)
from dataclasses import replace
from paper_2509_12207_b200.urg import DeviceWorkload
from workloads import get_config
from workloads.spec import RECORD_WORDS
cfg = get_config(CFG); b = replace(cfg.batch, scenario_count=NS) if NS else cfg.batch
w = cfg.workload(); p = cfg.policies[POL]
dw = DeviceWorkload(w)
agg = torch.zeros(dw.agg_words, dtype=torch.int64, device="cuda")
rec = torch.zeros((b.scenario_count, w.num_chains, RECORD_WORDS), dtype=torch.int32, device="cuda")
ts = []
for i in range(4):
    agg.zero_(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); dw.simulate(p, b, agg, rec); e1.record(); torch.cuda.synchronize()
    if i: ts.append(e0.elapsed_time(e1))
dw.check()
np.save(OUT, rec.cpu().numpy())
print(json.dumps({"ms": sorted(ts)[1], "launches": int(agg[-2].item()), "steps": int(agg[-1].item())}))
'''
cfg, pol, ns = sys.argv[1], sys.argv[2], int(sys.argv[3])
libs = sys.argv[4:]
ref = None
import numpy as np  # noqa: E402
for i, lib in enumerate(libs):
    out = f"/tmp/ab_rec_{i}.npy"
    code = CHILD.replace("ROOT", repr(ROOT)).replace("CFG", repr(cfg)).replace("POL", repr(pol)) \
                .replace("NS", str(ns)).replace("OUT", repr(out))
    env = dict(os.environ, URG_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
    if r.returncode != 0:
        print(lib, "FAILED", r.stderr[-800:])
        continue
    d = json.loads(r.stdout.strip().splitlines()[-1])
    rec = np.load(out)
    same = True if ref is None else bool(np.array_equal(rec, ref))
    if ref is None:
        ref = rec
    print(f"{os.path.basename(lib):28s} {d['ms']:9.2f} ms  launches {d['launches']}  steps {d['steps']}  "
          f"{d['launches'] / d['ms'] / 1e6:.3f} G/s  same_as_first={same}", flush=True)
