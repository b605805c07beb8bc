"""Write workloads/calibrated.json: L_th = 1/TH_urgent for the paper-shaped configs.

TH_urgent is "the 95th percentile urgency" of "the highest urgency value among
all active kernels in AKB", recorded periodically.  The
oracle runs scenario 0 of configs[1] (paper11, seed 0x5EED0002) under the full
UrgenGo policy with the threshold disabled, samples every 1 ms of the first
min(H, 30 s), and returns the laxity of the nearest-rank 95th percentile
(Q5).  Only the oracle is called; the GPU path reads the number.

Usage: python -m oracle.calibrate
"""
import json
import os
from dataclasses import replace

from oracle import oracle as O
from workloads.configs import get_config

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "workloads", "calibrated.json")


def main():
    cfg = get_config("paper11")
    b = replace(cfg.batch, scenario_count=1)          # scenario 0 of configs[1] (Q5)
    lth, n = O.calibrate(cfg.workload(), cfg.policies["urgengo"], b, window_ns=30_000_000_000)
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    out.update({"paper11": lth, "_samples": {"paper11": n},
                "_how": "python -m oracle.calibrate (PAPER.md:464-465, DESIGN.md Q5)"})
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
