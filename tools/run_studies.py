"""Run the design-option studies (paper_2509_12207_b200.sweep) on the GPU and write
profiles/<tag>_studies.{json,md}.  usage: python tools/run_studies.py TAG [scenarios] [usweep_scenarios]"""
import json
import os
import sys
import time
from dataclasses import asdict, replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_12207_b200 import sweep as SW  # noqa: E402
from workloads import get_config  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
SU = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
cfg = get_config("paper11")
w = cfg.workload()
base = cfg.policies["urgengo"]
b = replace(cfg.batch, scenario_count=S)
out, md = {}, [f"# Design-option studies on B200 ({tag})", "",
               f"paper11 workload (BASELINE.json configs[1]), {S} seeded scenarios x {b.horizon_ns / 1e9:.0f} s "
               f"per point, UrgenGo base policy (OVERLAP, L_th = {base.lax_threshold_ns} ns) unless stated. "
               "Miss ratios are Eq. 3 over the batch's aggregate counters; every point is one "
               "urg_simulate_batch launch.", ""]
studies = {
    "sync_modes (PAPER.md:793-796)": SW.sync_modes(base, b),
    "delta_eval (PAPER.md:798-800)": SW.delta_eval(base, b),
    "num_prio (PAPER.md:779-780)": SW.num_prio(base, b),
    "ablation (PAPER.md:774-776)": SW.ablation(base, b),
    "collisions (PAPER.md:790-791)": SW.collisions(base, b),
    "policies (PAPER.md:782-784)": SW.policies(base, b),
    "cudaFree (PAPER.md:907-911)": SW.cudafree(base, b),
    "CPU cores (PAPER.md:386-399)": SW.cpu_cores(base, b),
    "contention (PAPER.md:209-212)": SW.contention(base, b),
    "memcpy (Table 3, PAPER.md:374)": SW.memcpy(base, b),
    "executors (PAPER.md:272)": SW.executors(base, b),
}
cfg3 = get_config("usweep")
studies["utilisation sweep (configs[2])"] = SW.utilisation(base, [replace(x, scenario_count=SU) for x in cfg3.sweep])
for name, pts in studies.items():
    t0 = time.time()
    res = SW.run(w, pts)
    out[name] = [asdict(r) for r in res]
    md += [f"## {name}", "", SW.table(res), "", f"(wall {time.time() - t0:.1f} s)", ""]
    print(name, "done", flush=True)
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
with open(os.path.join(ROOT, "profiles", f"{tag}_studies.json"), "w") as f:
    json.dump(out, f, indent=1)
with open(os.path.join(ROOT, "profiles", f"{tag}_studies.md"), "w") as f:
    f.write("\n".join(md) + "\n")
print("\n".join(md))
