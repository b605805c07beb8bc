"""Key metrics of one `ncu --set full` capture (.ncu-rep) as JSON, and the bench's DRAM traffic
per launch (profiles/traffic.json, bench.py's `roofline.traffic`).

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.json [--traffic CONFIG POLICY]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "launch__registers_per_thread", "sass__inst_executed_local_loads", "sass__inst_executed_local_stores",
        "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__shared_mem_per_block_dynamic"]
STALLS = "smsp__average_warps_issue_stalled_"
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TUNIT = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}   # -> ms


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for h, u, v in zip(head, units, vals):
        if h in KEYS or (h.startswith(STALLS) and h.endswith("_per_issue_active.ratio")):
            res[h] = [v, u]
    return res


def kernel_ms(res):
    v, u = res["gpu__time_duration.sum"]
    return float(v.replace(",", "")) * TUNIT.get(u, 1.0)


def dram_bytes(res):
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        v, u = res[k]
        tot += float(v.replace(",", "")) * UNIT.get(u, 1)
    return int(round(tot))


if __name__ == "__main__":
    rep, dst = sys.argv[1], sys.argv[2]
    res = summary(rep)
    with open(dst, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))
    if "--traffic" in sys.argv:
        i = sys.argv.index("--traffic")
        cfg, pol = sys.argv[i + 1], sys.argv[i + 2]
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        tp = os.path.join(root, "profiles", "traffic.json")
        t = json.load(open(tp)) if os.path.exists(tp) else {}
        t.setdefault(cfg, {})[pol] = {
            "bytes_per_launch": dram_bytes(res), "kernel_ms": kernel_ms(res),
            "source": f"{os.path.relpath(dst, root)}: dram__bytes_read.sum + dram__bytes_write.sum and "
                      "gpu__time_duration.sum of one urg_sim_kernel launch of bench.py's step (ncu)"}
        with open(tp, "w") as f:
            json.dump(t, f, indent=1)
        print("traffic", t[cfg][pol])
