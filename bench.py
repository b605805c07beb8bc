"""bench.py -- batched UrgenGo launch-policy simulation on B200 (the driver's contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl urg|reference] [--config paper11]

One step = one pass of the whole hot path (plus the
§8(e) allreduce when N > 1) over one batch: urg_simulate_batch on the config's
scenarios (weak scaling: every rank simulates its own `scenario_count` global
scenarios), then the int64 aggregate allreduce.  Rank 0 prints ONE JSON line.

The default workload is BASELINE.json configs[1] ("paper11": 11 Table-2 chains,
~100s of kernels per task, 10 s horizon, 1k seeded scenarios per GPU).  L2 is
flushed (a 256 MiB write) between timed steps; inputs are tiny (a ~100 KB
template), so the flush is what keeps steps cold.

`cpu_baseline` (and `--impl reference`) run the CPU oracle (oracle/, test
infrastructure) unchanged over a bounded sample of the same scenarios on the
host cores -- one oracle process per core over disjoint scenarios -- and the
cpu_baseline leg also compares the oracle's per-scenario records with the GPU's
for that sample (bit-exact parity on the bench's own launch configuration).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "simulated launch events/s"
UNIT = "launch events/s"

# Algorithmic warp-instructions of the event loop: per loop step
# (one distinct event time of one scenario) and per launch event, all of them and the
# ALU-pipe ones (integer compare/add/select/shift/logic; the rest are warp collectives,
# loads, branches and the two IMAD.WIDE of the duration).  The bound is the ALU pipe:
# one warp-instruction per 2 cycles per scheduler (B300_MICROARCH.md "alu-pipe rt_SMSP=2";
# ncu: 80-84 % busy in the throughput build), so peak = SMs x 4 x 0.5 x sm_max_mhz; the
# issue peak (1 warp-instruction/clk/scheduler) is reported beside it.
ALG_INST_PER_STEP = 24
ALG_INST_PER_LAUNCH = 40
ALG_ALU_PER_STEP = 18
ALG_ALU_PER_LAUNCH = 34
SMSP_PER_SM = 4
ALU_RT_CYCLES = 2


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ----------------------------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline and --impl reference): one process per core, disjoint scenarios
# ----------------------------------------------------------------------------------------------
_W = None


def _oracle_init(cfg_name, pol_name):
    global _W
    from oracle import oracle as O
    from workloads import get_config
    cfg = get_config(cfg_name)
    O.lib()
    _W = (O, cfg.workload(), cfg.policies[pol_name], cfg.batch)


def _oracle_job(args):
    begin, count, horizon = args
    from dataclasses import replace
    O, w, p, b = _W
    bb = replace(b, scenario_begin=begin, scenario_count=count, horizon_ns=horizon)
    r = O.run(w, p, bb)
    return begin, r.records, int(r.agg[-2]), r.seconds


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_pool(cfg_name, pol_name, cores, method="fork"):
    import multiprocessing as mp
    ctx = mp.get_context(method)
    return ctx.Pool(cores, initializer=_oracle_init, initargs=(cfg_name, pol_name))


def oracle_sample(pool, begins, horizon):
    """Run the oracle on scenarios `begins` (one scenario per job); wall time over the pool."""
    t0 = time.perf_counter()
    res = pool.map(_oracle_job, [(s, 1, horizon) for s in begins], chunksize=1)
    dt = time.perf_counter() - t0
    return res, dt


# ----------------------------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, r[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------------------------
def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="urg", choices=["urg", "reference"])
    ap.add_argument("--config", default="paper11")
    ap.add_argument("--policy", default="urgengo")
    ap.add_argument("--scenarios", type=int, default=0, help="override scenarios per GPU (default: the config's)")
    ap.add_argument("--horizon-ms", type=int, default=0, help="override the horizon")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-throughput", action="store_true", help="skip the configs[4] throughput-regime line item")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU work of the cpu_baseline sample")
    return ap.parse_args()


def workload_batch(a):
    from dataclasses import replace
    from workloads import get_config
    cfg = get_config(a.config)
    b = cfg.batch
    if a.scenarios:
        b = replace(b, scenario_count=a.scenarios)
    if a.horizon_ms:
        b = replace(b, horizon_ns=a.horizon_ms * 1_000_000)
    return cfg, cfg.workload(), cfg.policies[a.policy], b


def config_json(cfg, w, b, a, n):
    return {"workload": f"{cfg.name} (BASELINE.json {cfg.note.split(':')[0]})", "policy": a.policy,
            "chains": w.num_chains, "kernels_per_template": w.total_kernels(),
            "template_variants": w.num_variants,
            "scenarios_per_gpu": b.scenario_count, "scenarios_total": b.scenario_count * n,
            "horizon_s": b.horizon_ns / 1e9, "seed": hex(b.seed), "l2": "flushed (256 MiB write) between steps",
            "parallelism": f"scenario shards x{n}"}


def run_reference(a):
    """--impl reference: the CPU oracle as it stands, on the host cores, over bounded samples."""
    rank = _env_int("RANK", 0)
    n = a.gpus
    if rank != 0:
        return
    cfg, w, p, b = workload_batch(a)
    cores = _cores()
    pool = oracle_pool(a.config, a.policy, cores)
    per_step = cores   # one full-horizon scenario per core per step
    total_launch, total_t, times = 0, 0.0, []
    for i in range(a.warmup + a.steps):
        begins = [(i * per_step + j) % max(b.scenario_count, 1) + b.scenario_begin for j in range(per_step)]
        res, dt = oracle_sample(pool, begins, b.horizon_ns)
        if i >= a.warmup:
            total_launch += sum(r[2] for r in res)
            total_t += dt
            times.append(dt)
    pool.close()
    v = total_launch / total_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": n, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * total_t / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded)",
            "config": config_json(cfg, w, b, a, 1),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{per_step} full-horizon scenarios per step (one per core), "
                                       f"{cores} oracle processes, CPU {_cpu_model()}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import ctypes as ct

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2509_12207_b200.dist import allreduce_agg
    from paper_2509_12207_b200.urg import DeviceWorkload, OutputsS, batch_struct, lib, policy_struct
    from dataclasses import replace
    from workloads import get_config
    from workloads.spec import RECORD_WORDS

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    want_cpu = rank == 0 and world == 1 and not a.no_cpu_baseline
    # the oracle pool is started only after the GPU legs (an idle pool forked at start-up was
    # measured to slow the e2e leg 2-3x on some hosts), spawned so no child inherits CUDA state
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (the product path has no CPU fallback)")
    # one process per GPU; URG_BENCH_BACKEND=gloo (test only) lets several ranks share one
    # device so the N > 1 path can be exercised on a single-GPU box
    backend = os.environ.get("URG_BENCH_BACKEND", "nccl")
    dev = local % torch.cuda.device_count() if backend != "nccl" else local
    torch.cuda.set_device(dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    n = world

    cfg, w, p, b0 = workload_batch(a)
    S = b0.scenario_count
    b = replace(b0, scenario_begin=b0.scenario_begin + rank * S)     # weak scaling: own global scenarios
    stream = torch.cuda.current_stream()
    dw = DeviceWorkload(w)
    agg = torch.zeros(dw.agg_words, dtype=torch.int64, device="cuda")
    rec = torch.zeros((S, w.num_chains, RECORD_WORDS), dtype=torch.int32, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        agg.zero_()
        if ev:
            ev[1].record(stream)
        dw.simulate(p, b, agg, rec, stream=stream)
        if ev:
            ev[2].record(stream)
        allreduce_agg(agg)
        if ev:
            ev[3].record(stream)

    for _ in range(a.warmup):
        flush.fill_(1)
        step()
    dw.check(stream)
    torch.cuda.synchronize()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(a.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(dev) as clk:
        for i in range(a.steps):
            flush.fill_(i & 0xFF)            # L2 flush outside the timed events
            step(evs[i])
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    dw.check(stream)
    step_ms = [e[0].elapsed_time(e[3]) for e in evs]
    kern_ms = [e[1].elapsed_time(e[2]) for e in evs]
    t_local = sum(step_ms) / 1e3
    k_local = sum(kern_ms) / 1e3 / a.steps
    tt = torch.tensor([t_local, k_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_max, k_max = tt.tolist()
    a_host = agg.cpu().numpy()
    launches_all = int(a_host[-2])        # after the allreduce: every rank's launch events
    steps_all = int(a_host[-1])
    scen_all = S * n
    value = launches_all * a.steps / t_max
    clocks = clk.summary()

    # ---- e2e: the public API with HOST buffers, template upload included, every step ----
    # pinned host buffers: the step's device->host result copies are DMA from/to page-locked memory
    host_agg = torch.zeros(dw.agg_words, dtype=torch.int64, pin_memory=True).numpy()
    host_rec = torch.zeros((S, w.num_chains, RECORD_WORDS), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    L = lib()
    ps, bs = policy_struct(p), batch_struct(b)
    o = OutputsS(host_rec.ctypes.data, host_agg.ctypes.data)
    h2d = dw.template_bytes
    d2h = host_agg.nbytes + host_rec.nbytes
    e2e_t = []
    for i in range(max(1, min(a.steps, 3)) + 1):
        flush.fill_(1)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        hw = ct.c_void_p()
        assert L.urg_create_workload(ct.byref(dw.desc), ct.byref(hw)) == 0, L.urg_last_error()
        host_agg[:] = 0
        t1 = time.perf_counter()
        st = L.urg_simulate_batch_host(hw, ct.byref(ps), ct.byref(bs), ct.byref(o), ct.c_void_p(stream.cuda_stream))
        assert st == 0, L.urg_last_error()
        t2 = time.perf_counter()
        ht = torch.from_numpy(host_agg.copy())
        if world > 1:     # the same single collective, on host-returned results
            ht = ht.cuda()
            dist.all_reduce(ht)
            ht = ht.cpu()
        L.urg_destroy_workload(hw)
        dt = time.perf_counter() - t0
        if os.environ.get("URG_BENCH_DEBUG"):
            print(f"e2e step {i}: {dt * 1e3:.1f} ms (create {1e3 * (t1 - t0):.1f}, simulate {1e3 * (t2 - t1):.1f})",
                  file=sys.stderr, flush=True)
        if i > 0:
            e2e_t.append(dt)
    tt = torch.tensor([sum(e2e_t) / len(e2e_t)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    e2e_step = tt.item()
    assert np.array_equal(host_rec, rec.cpu().numpy().view(np.uint32)), "host-buffer path differs from device path"

    # ---- roofline: ALU-pipe-bound event loop ----
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    peak_mhz = clocks["sm_max_mhz"] or 1965.0
    # per-rank algorithmic instruction count of one launch of urg_sim_kernel
    launches_rank, steps_rank = launches_all / n, steps_all / n
    alg_inst = steps_rank * ALG_INST_PER_STEP + launches_rank * ALG_INST_PER_LAUNCH
    alg_alu = steps_rank * ALG_ALU_PER_STEP + launches_rank * ALG_ALU_PER_LAUNCH
    achieved = alg_alu / k_max / 1e9              # G ALU-pipe warp-inst/s
    peak = sms * SMSP_PER_SM * peak_mhz * 1e6 / ALU_RT_CYCLES / 1e9
    issue_achieved = alg_inst / k_max / 1e9
    issue_peak = sms * SMSP_PER_SM * peak_mhz * 1e6 / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(cfg.name, {}).get(a.policy)
        except (OSError, ValueError):
            traffic = None

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": 1e3 * t_max / a.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic (seeded Philox scenarios of the Table-2 workload)",
            "config": config_json(cfg, w, b0, a, n),
            "scenarios_per_s": scen_all * a.steps / t_max,
            "launch_events_per_step": launches_all, "loop_steps_per_step": steps_all,
            "kernel_ms": 1e3 * k_max,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gwarp-inst/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "urg_sim_kernel",
                         "issue": {"achieved": issue_achieved, "peak": issue_peak, "frac": issue_achieved / issue_peak},
                         "note": f"algorithmic ALU-pipe warp-inst = {ALG_ALU_PER_STEP}/loop step + "
                                 f"{ALG_ALU_PER_LAUNCH}/launch event (DESIGN.md §7); peak = ALU pipe, {sms} SMs x 4 "
                                 f"schedulers x 1/{ALU_RT_CYCLES} warp-inst/clk x {peak_mhz:.0f} MHz; 'issue' = all "
                                 f"{ALG_INST_PER_STEP}/{ALG_INST_PER_LAUNCH} algorithmic warp-inst against the issue peak"},
            "e2e": {"value": launches_all / e2e_step, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": a.steps,
            "clocks": clocks}

    # ---- throughput regime beside the headline (not the metric's workload): configs[4]'s
    #      workload at a size that fills the GPU, the throughput build, device-timed ----
    if not a.no_throughput and a.config == "paper11":
        tcfg = get_config("scaleout")
        tw = tcfg.workload()
        tS = 300_000
        tb = replace(tcfg.batch, scenario_begin=rank * tS, scenario_count=tS)
        tdw = DeviceWorkload(tw)
        tagg = torch.zeros(tdw.agg_words, dtype=torch.int64, device="cuda")
        tdw.simulate(tcfg.policies["urgengo"], tb, tagg, stream=stream)          # warm-up
        tt_ms = []
        for _ in range(2):
            tagg.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            tdw.simulate(tcfg.policies["urgengo"], tb, tagg, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            tt_ms.append(e0.elapsed_time(e1))
        tdw.check(stream)
        tl, tsteps = int(tagg[-2].item()), int(tagg[-1].item())
        tdw.close()
        x = torch.tensor([max(tt_ms)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
        line["throughput_regime"] = {
            "workload": f"scaleout (BASELINE.json configs[4]) workload, {tS} scenarios x 1 s per GPU, UrgenGo; "
                        "throughput build (two scenarios per warp); reported beside the headline, not the metric",
            "value": tl * n / (x.item() / 1e3), "unit": UNIT, "ms_per_launch": x.item(),
            "launch_events_per_gpu": tl,
            # the same ALU-pipe roofline as the headline's (algorithmic ALU-pipe warp-inst / kernel time)
            "roofline": {"bound": "alu", "unit": "Gwarp-inst/s", "peak": peak,
                         "achieved": (tsteps * ALG_ALU_PER_STEP + tl * ALG_ALU_PER_LAUNCH) / (x.item() / 1e3) / 1e9,
                         "frac": (tsteps * ALG_ALU_PER_STEP + tl * ALG_ALU_PER_LAUNCH) / (x.item() / 1e3) / 1e9 / peak}}

    # ---- cpu_baseline: the oracle, unchanged, on a bounded sample (rank 0, N = 1 only) ----
    if want_cpu:
        cores = _cores()
        pool = oracle_pool(a.config, a.policy, cores, "spawn")
        one, _ = oracle_sample(pool, [b.scenario_begin] * cores, b.horizon_ns)  # warm every worker
        dt1 = max(r[3] for r in one)                                            # size the sample
        per_core = max(1, int(a.cpu_seconds / max(dt1, 1e-3)))
        m = min(S, cores * per_core)
        begins = [b.scenario_begin + i for i in range(m)]
        res, dt = oracle_sample(pool, begins, b.horizon_ns)
        pool.close()
        g = rec.cpu().numpy().view(np.uint32)
        mism = [s for s, r, _, _ in res if not np.array_equal(r[0], g[s - b.scenario_begin])]
        ol = sum(r[2] for r in res)
        line["cpu_baseline"] = {"value": ol / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": f"scenarios {begins[0]}..{begins[-1]} ({m} of {S}) at the full horizon, "
                                          f"one oracle process per core; CPU {_cpu_model()}",
                                "single_core_value": ol / sum(r[3] for r in res)}
        line["parity_sample"] = {"scenarios": m, "bit_exact": not mism, "mismatches": mism[:8]}

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    dw.close()


if __name__ == "__main__":
    main()
