"""Run the BASELINE.json configurations at full size on the GPU and check sampled scenarios
against the CPU oracle (BASELINE.md "CPU baseline plan": configs[0]-[1] every scenario,
configs[2]-[4] the first 256, the last 256 and every 9973rd scenario index).

usage: python tools/run_configs.py TAG [--configs toy2,paper11,usweep,jitter,scaleout]
                                       [--scaleout-count N] [--chunk N]
Writes profiles/<TAG>_configs.json and prints a markdown table.
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time
from dataclasses import replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

_W = {}


def _init(names):
    from oracle import oracle as O
    from workloads import get_config
    O.lib()
    for n in names:
        _W[n] = get_config(n)


def _oracle_one(args):
    name, pol, bd, s = args
    from oracle import oracle as O
    from workloads.spec import Batch
    cfg = _W[name]
    b = Batch(**bd)
    r = O.run(cfg.workload(), cfg.policies[pol], replace(b, scenario_begin=s, scenario_count=1))
    return s, r.records[0]


def sample_indices(begin, count, full):
    if full:
        return list(range(begin, begin + count))
    idx = set(range(begin, begin + min(256, count)))
    idx |= set(range(begin + max(0, count - 256), begin + count))
    idx |= set(range(begin, begin + count, 9973))
    return sorted(idx)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--configs", default="toy2,paper11,usweep,jitter,scaleout")
    ap.add_argument("--scaleout-count", type=int, default=100_000_000)
    ap.add_argument("--chunk", type=int, default=2_000_000)
    a = ap.parse_args()
    import numpy as np
    import torch
    from paper_2509_12207_b200.urg import DeviceWorkload
    from workloads import get_config
    from workloads.spec import RECORD_WORDS
    from bench import Clocks
    names = a.configs.split(",")
    cores = len(os.sched_getaffinity(0))
    pool = mp.get_context("fork").Pool(cores, initializer=_init, initargs=(names,))
    out, md = [], ["| config | point | policy | scenarios | launch events | GPU s | G events/s | Eq. 3 miss ratio | "
                   "oracle-checked scenarios | mismatches | SM MHz (median/max), throttle |",
          "|---|---|---|---|---|---|---|---|---|---|---|"]
    for name in names:
        cfg = get_config(name)
        w = cfg.workload()
        batches = cfg.sweep or [cfg.batch]
        full = name in ("toy2", "paper11")
        with DeviceWorkload(w) as dw:
            for bi, b in enumerate(batches):
                if name == "scaleout":
                    b = replace(b, scenario_count=a.scaleout_count)
                for pol in cfg.policies:
                    p = cfg.policies[pol]
                    want = sample_indices(b.scenario_begin, b.scenario_count, full)
                    jobs = pool.map_async(_oracle_one, [(name, pol, b.__dict__, s) for s in want], chunksize=4)
                    agg = torch.zeros(dw.agg_words, dtype=torch.int64, device="cuda")
                    got = {}
                    t0 = time.perf_counter()
                    gpu_s = 0.0
                    clk = Clocks(torch.cuda.current_device()).__enter__()   # SM clocks / throttle reasons
                    for lo in range(0, b.scenario_count, a.chunk):
                        n = min(a.chunk, b.scenario_count - lo)
                        cb = replace(b, scenario_begin=b.scenario_begin + lo, scenario_count=n)
                        rec = torch.zeros((n, w.num_chains, RECORD_WORDS), dtype=torch.int32, device="cuda")
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        dw.simulate(p, cb, agg, rec)
                        e1.record()
                        torch.cuda.synchronize()
                        gpu_s += e0.elapsed_time(e1) / 1e3
                        sel = [s for s in want if cb.scenario_begin <= s < cb.scenario_begin + n]
                        if sel:
                            r = rec[torch.tensor([s - cb.scenario_begin for s in sel], device="cuda")].cpu().numpy()
                            for s, x in zip(sel, r.view(np.uint32)):
                                got[s] = x
                        del rec
                    clk.__exit__(None, None, None)
                    clocks = clk.summary()
                    dw.check()
                    a_host = agg.cpu().numpy()
                    per, overall = dw.miss_ratios(a_host)
                    mism = [s for s, orec in jobs.get() if not np.array_equal(orec, got[s])]
                    launches = int(a_host[-2])
                    row = {"config": name, "point": bi, "fa": f"{b.fa_num}/{b.fa_den}", "policy": pol,
                           "scenarios": b.scenario_count, "horizon_s": b.horizon_ns / 1e9, "launch_events": launches,
                           "loop_steps": int(a_host[-1]), "gpu_s": gpu_s, "wall_s": time.perf_counter() - t0,
                           "launch_events_per_s": launches / gpu_s, "eq3_miss_ratio": overall,
                           "per_chain_miss_ratio": [float(x) for x in per], "oracle_checked": len(want),
                           "mismatches": mism[:16], "clocks": clocks}
                    out.append(row)
                    md.append(f"| {name} | {bi} (f_a {b.fa_num}/{b.fa_den}) | {pol} | {b.scenario_count} | {launches:.4g} | "
                              f"{gpu_s:.2f} | {launches / gpu_s / 1e9:.2f} | {overall:.4f} | {len(want)} | {len(mism)} | "
                              f"{clocks['sm_mhz']}/{clocks['sm_max_mhz']} {','.join(clocks['reasons']) or '-'} |")
                    print(md[-1], flush=True)
    pool.close()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{a.tag}_configs.json"), "w") as f:
        json.dump(out, f, indent=1)
    with open(os.path.join(ROOT, "profiles", f"{a.tag}_configs.md"), "w") as f:
        f.write(f"# BASELINE.json configurations at full size on one B200 ({a.tag})\n\n"
                "GPU: `urg_simulate_batch` in chunks of at most 2M scenarios, device-timed.  Oracle: "
                "configs[0]-[1] every scenario, configs[2]-[4] the first 256, the last 256 and every "
                "9973rd scenario index, per-scenario records compared bit for bit (BASELINE.md).  SM clocks "
                "sampled with nvidia-smi every 100 ms while each row's GPU runs were in flight.\n\n")
        f.write("\n".join(md) + "\n")


if __name__ == "__main__":
    main()
