"""bench.py -- batched UrgenGo launch-policy simulation on B200 (the driver's contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl urg|reference] [--config jitter]
                    [--scaling weak|strong]

The headline workload is BASELINE.json configs[3] ("jitter": 11 Table-2 chains, 64 template
variants, heavy-tailed Pareto(1.5) kernel times, 60 s horizon, 1M seeded scenarios, UrgenGo) --
the largest configuration one GPU holds.  The whole configuration is timed: its scenarios are
split into K contiguous slices and one step = one pass of the hot path (SURVEY.md §8(a) rows
A0-A12, plus the §8(e) allreduce of the step's int64 aggregates when N > 1) over one slice:
urg_simulate_batch on that slice, then the allreduce.  W warm-up steps run first on scenarios
outside the configuration (the same kernel build).  L2 is flushed (a 256 MiB write) between
steps, outside the timed events.

Multi-GPU: one process per GPU (torchrun).  --scaling weak (default): every rank simulates the
configuration's size on its own global scenario indices; --scaling strong: the configuration's
scenarios are partitioned over the ranks.  `value` = launch events of all
ranks / the max over ranks of the summed step times.

Beside the headline the line carries: `latency_regime` (configs[1], 1000 scenarios x 10 s, the
latency build) and `throughput_regime` (configs[4]'s workload, 300k scenarios x 1 s per GPU),
both device-timed; `e2e` (the public C ABI with HOST buffers, template upload and result copies
inside the timed region, over the first three slices); `roofline` (ALU pipe, issue and HBM
views of the simulation kernel); `cpu_baseline` + `parity_sample` (the CPU oracle, unchanged,
on BASELINE.md's sample of the configuration -- the first 256, the last 256 and every 9973rd
scenario -- on the host cores, compared record by record with the GPU's records).
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
HBM_FALLBACK_GBS = 6650.0     # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
BASELINE_SAMPLE_STRIDE = 9973  # first 256, last 256 and every 9973rd scenario


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    except (OSError, ValueError):
        return {"hbm_gbs": HBM_FALLBACK_GBS}, "fallback (B200_PROFILING.md)"


def baseline_sample(begin: int, count: int):
    """BASELINE.md's deterministic sample of a configuration's scenario indices."""
    idx = set(range(begin, begin + min(256, count)))
    idx |= set(range(begin + max(0, count - 256), begin + count))
    idx |= set(range(begin, begin + count, BASELINE_SAMPLE_STRIDE))
    return sorted(idx)


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
def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20, help="timed steps = slices of the configuration")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="urg", choices=["urg", "reference"])
    ap.add_argument("--config", default="jitter")
    ap.add_argument("--policy", default="urgengo")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--scenarios", type=int, default=0, help="override the configuration's scenario count")
    ap.add_argument("--horizon-ms", type=int, default=0, help="override the horizon")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-regimes", action="store_true", help="skip the latency / throughput regime items")
    ap.add_argument("--e2e-steps", type=int, default=3, help="slices timed through the host-buffer C ABI")
    return ap.parse_args(argv)


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


def config_json(cfg, w, b, a, n, per_rank):
    return {"workload": f"{cfg.name} (BASELINE.json {cfg.note})", "policy": a.policy,
            "chains": w.num_chains, "kernels_per_template": w.total_kernels(),
            "template_variants": w.num_variants, "kernel_factor_table": w.kern_quantiles_q16 is not None,
            "scenarios_config": b.scenario_count, "scenarios_per_gpu": per_rank,
            "scenarios_total": per_rank * n if a.scaling == "weak" else b.scenario_count,
            "slices": a.steps, "horizon_s": b.horizon_ns / 1e9, "seed": hex(b.seed),
            "l2": "flushed (256 MiB write) between steps", "scaling": a.scaling,
            "parallelism": f"scenario shards x{n}"}


def run_reference(a):
    """--impl reference: the CPU oracle as it stands, on the host cores, over bounded samples of
    the same configuration (one full-horizon scenario per core per step)."""
    rank = _env_int("RANK", 0)
    n = a.gpus
    if rank != 0:
        return
    cfg, w, p, b = workload_batch(a)
    cores = _cores()
    pool = oracle_pool(a.config, a.policy, cores)
    per_step = cores
    total_launch, total_t = 0, 0.0
    for i in range(a.warmup + a.steps):
        begins = [b.scenario_begin + (i * per_step + j) % max(b.scenario_count, 1) for j in range(per_step)]
        res, dt = oracle_sample(pool, begins, b.horizon_ns)
        if i >= a.warmup:
            total_launch += sum(r[2] for r in res)
            total_t += dt
    pool.close()
    v = total_launch / total_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": n, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * total_t / a.steps, "higher_is_better": True,
            "scaling": a.scaling, "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded)",
            "config": config_json(cfg, w, b, a, 1, b.scenario_count),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{per_step} full-horizon scenarios of the configuration per step (one per "
                                       f"core), {cores} oracle processes, CPU {_cpu_model()}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def _alu_roofline(steps, launches, seconds, sms, mhz):
    alu = (steps * ALG_ALU_PER_STEP + launches * ALG_ALU_PER_LAUNCH) / seconds / 1e9
    inst = (steps * ALG_INST_PER_STEP + launches * ALG_INST_PER_LAUNCH) / seconds / 1e9
    peak = sms * SMSP_PER_SM * mhz * 1e6 / ALU_RT_CYCLES / 1e9
    issue_peak = sms * SMSP_PER_SM * mhz * 1e6 / 1e9
    return {"bound": "alu", "achieved": alu, "peak": peak, "unit": "Gwarp-inst/s", "frac": alu / peak,
            "issue": {"achieved": inst, "peak": issue_peak, "frac": inst / issue_peak}}


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import ctypes as ct

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2509_12207_b200.dist import allreduce_agg, job_range, reduce_job, slices
    from paper_2509_12207_b200.urg import DeviceWorkload, OutputsS, batch_struct, lib, policy_struct
    from dataclasses import replace
    from workloads import get_config
    from workloads.spec import RECORD_WORDS

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    want_cpu = rank == 0 and world == 1 and not a.no_cpu_baseline
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (the product path has no CPU fallback)")
    # one process per GPU; URG_BENCH_BACKEND=gloo (test only) lets several ranks share one
    # device so the N > 1 path can be exercised on a single-GPU box
    backend = os.environ.get("URG_BENCH_BACKEND", "nccl")
    dev = local % torch.cuda.device_count() if backend != "nccl" else local
    torch.cuda.set_device(dev)
    comm = {"backend": None, "nranks": 1}
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
        comm = {"backend": dist.get_backend(), "nranks": dist.get_world_size()}
        print(f"[bench] rank {rank}: {comm['backend']} communicator, nranks={comm['nranks']}, device cuda:{dev}",
              file=sys.stderr, flush=True)
    n = world
    red_dev = "cuda" if comm["backend"] == "nccl" else "cpu"

    cfg, w, p, b0 = workload_batch(a)
    lo, S = job_range(rank, world, b0.scenario_begin, b0.scenario_count, a.scaling)
    plan = slices(lo, S, a.steps)
    wcount = min(max(c for _, c in plan), 8192)          # warm-up: the timed steps' kernel build
    warm_lo = b0.scenario_begin + (world if a.scaling == "weak" else 1) * b0.scenario_count + rank * a.warmup * wcount
    warm = [(warm_lo + i * wcount, wcount) for i in range(a.warmup)]
    stream = torch.cuda.current_stream()
    dw = DeviceWorkload(w)
    C = w.num_chains
    agg_step = torch.zeros(dw.agg_words, dtype=torch.int64, device="cuda")
    agg_total = torch.zeros(dw.agg_words, dtype=torch.int64, device="cuda")
    rec = torch.zeros((max(S, 1), C, RECORD_WORDS), dtype=torch.int32, device="cuda")   # the job's records
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def step(begin, count, ev=None, out_rec=None):
        if ev:
            ev[0].record(stream)
        agg_step.zero_()
        if ev:
            ev[1].record(stream)
        dw.simulate(p, replace(b0, scenario_begin=begin, scenario_count=count), agg_step, out_rec, stream=stream)
        if ev:
            ev[2].record(stream)
        allreduce_agg(agg_step)
        agg_total.add_(agg_step)
        if ev:
            ev[3].record(stream)

    wrec = torch.zeros((max(wcount, 1), C, RECORD_WORDS), dtype=torch.int32, device="cuda")
    for wb, wc in warm:
        flush.fill_(1)
        step(wb, wc, out_rec=wrec)
    dw.check(stream)
    torch.cuda.synchronize()
    agg_total.zero_()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(a.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(dev) as clk:
        for i, (sb, sc) in enumerate(plan):
            flush.fill_(i & 0xFF)            # L2 flush outside the timed events
            step(sb, sc, evs[i], rec[sb - lo: sb - lo + sc] if sc else None)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    dw.check(stream)
    step_ms = [e[0].elapsed_time(e[3]) for e in evs]
    kern_ms = [e[1].elapsed_time(e[2]) for e in evs]
    a_host = agg_total.cpu().numpy()                   # every rank's events (reduced per step)
    launches_all, steps_all = int(a_host[-2]), int(a_host[-1])
    _, _, t_max = reduce_job(0, 0, sum(step_ms) / 1e3, red_dev)
    _, _, k_max = reduce_job(0, 0, sum(kern_ms) / 1e3, red_dev)
    value = launches_all / t_max
    clocks = clk.summary()
    # the aggregates are the records' sums (R23): a cross-check over the whole job on this rank
    rec_np = rec.cpu().numpy().view(np.uint32)[:S]
    local_launch = int(rec_np[:, :, 4].astype(np.int64).sum())
    l_sum, _, _ = reduce_job(local_launch, 0, 0.0, red_dev)
    agg_consistent = l_sum == launches_all

    # ---- e2e: the public API with HOST buffers, template upload included, every step ----
    L = lib()
    ps = policy_struct(p)
    e2e_plan = plan[: max(1, min(a.e2e_steps, len(plan)))]
    e_count = max(c for _, c in e2e_plan)
    host_agg = torch.zeros(dw.agg_words, dtype=torch.int64, pin_memory=True).numpy()
    host_rec = torch.zeros((max(e_count, 1), C, RECORD_WORDS), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    h2d = dw.template_bytes
    e2e_t, e2e_launch, d2h, e2e_same = 0.0, 0, 0, True
    for i, (sb, sc) in enumerate([e2e_plan[0]] + e2e_plan):       # the first call warms the host path
        flush.fill_(1)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        bs = batch_struct(replace(b0, scenario_begin=sb, scenario_count=sc))
        o = OutputsS(host_rec.ctypes.data, host_agg.ctypes.data)
        t0 = time.perf_counter()
        hw = ct.c_void_p()
        assert L.urg_create_workload(ct.byref(dw.desc), ct.byref(hw)) == 0, L.urg_last_error()
        host_agg[:] = 0
        st = L.urg_simulate_batch_host(hw, ct.byref(ps), ct.byref(bs), ct.byref(o), ct.c_void_p(stream.cuda_stream))
        assert st == 0, L.urg_last_error()
        ht = torch.from_numpy(host_agg.copy())
        if world > 1:     # the same single collective, on host-returned results
            ht = ht.to(red_dev)
            dist.all_reduce(ht)
            ht = ht.cpu()
        L.urg_destroy_workload(hw)
        dt = time.perf_counter() - t0
        if i > 0:
            e2e_t += dt
            e2e_launch += int(ht[-2].item())
            d2h += host_agg.nbytes + sc * C * RECORD_WORDS * 4
            e2e_same = e2e_same and np.array_equal(host_rec[:sc], rec_np[sb - lo: sb - lo + sc])
    _, _, e2e_max = reduce_job(0, 0, e2e_t, red_dev)
    ne = len(e2e_plan)

    # ---- roofline of the simulation kernel ----
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    peak_mhz = clocks["sm_max_mhz"] or 1965.0
    launches_rank, steps_rank = launches_all / n, steps_all / n       # per-rank averages
    roof = _alu_roofline(steps_rank, launches_rank, k_max, sms, peak_mhz)
    peaks, peaks_src = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", HBM_FALLBACK_GBS))
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        tr = json.load(open(tp)).get(cfg.name, {}).get(a.policy)
        if isinstance(tr, dict):
            traffic = tr
    except (OSError, ValueError):
        traffic = None
    roof["kernel"] = "urg_sim_kernel"
    roof["traffic"] = None if traffic is None else traffic.get("bytes_per_launch")
    # algorithmic HBM bytes of one launch: the slice's records (32 B per scenario and chain) and
    # its aggregate words written, the template variants' kernel records read once
    alg_bytes = (S / a.steps) * C * RECORD_WORDS * 4 + dw.agg_words * 8 + dw.template_bytes
    roof["hbm"] = {"algorithmic_bytes_per_launch": alg_bytes, "achieved": alg_bytes / (k_max / a.steps) / 1e9,
                   "peak": hbm_peak, "unit": "GB/s", "peak_source": peaks_src}
    roof["hbm"]["frac"] = roof["hbm"]["achieved"] / hbm_peak
    if traffic is not None:
        dram_gbs = traffic["bytes_per_launch"] / (traffic["kernel_ms"] / 1e3) / 1e9
        roof["hbm"]["dram_measured"] = {"bytes_per_launch": traffic["bytes_per_launch"], "GB/s": dram_gbs,
                                        "frac": dram_gbs / hbm_peak, "source": traffic.get("source")}
    roof["note"] = (f"algorithmic ALU-pipe warp-inst = {ALG_ALU_PER_STEP}/loop step + {ALG_ALU_PER_LAUNCH}/launch "
                    f"event (DESIGN.md §7); peak = ALU pipe, {sms} SMs x 4 schedulers x 1/{ALU_RT_CYCLES} "
                    f"warp-inst/clk x {peak_mhz:.0f} MHz; 'issue' = all {ALG_INST_PER_STEP}/{ALG_INST_PER_LAUNCH} "
                    "algorithmic warp-inst against the issue peak; 'hbm' = algorithmic bytes per launch "
                    "(records + aggregates written, kernel records read) and ncu DRAM bytes, against the "
                    "measured copy bandwidth")

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": 1e3 * t_max / a.steps, "higher_is_better": True, "scaling": a.scaling,
            "vs_baseline": None, "dtype": "int64",
            "data": "synthetic (seeded Philox scenarios of the Table-2 workload, 64 template variants)",
            "config": config_json(cfg, w, b0, a, n, S),
            "scenarios_per_s": (S * n if a.scaling == "weak" else b0.scenario_count) / t_max,
            "launch_events": launches_all, "loop_steps": steps_all, "kernel_ms_per_step": 1e3 * k_max / a.steps,
            "agg_consistent_with_records": agg_consistent,
            "roofline": roof,
            "e2e": {"value": e2e_launch / e2e_max, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h // ne, "steps": ne,
                    "path": "urg_create_workload + urg_simulate_batch_host (pinned host buffers) + "
                            f"urg_destroy_workload per step, the first {ne} slices",
                    "records_equal_device_path": bool(e2e_same)},
            "gpu_launches": a.steps,
            "comm": comm,
            "clocks": clocks}

    # ---- regimes beside the headline (not the metric's workload), device-timed ----
    if not a.no_regimes:
        def regime(name, pol, count, horizon_ns, reps):
            rc = get_config(name)
            rw = rc.workload()
            rlo, rS = job_range(rank, world, rc.batch.scenario_begin, count, a.scaling)
            rb = replace(rc.batch, scenario_begin=rlo, scenario_count=rS, horizon_ns=horizon_ns)
            rdw = DeviceWorkload(rw)
            ragg = torch.zeros(rdw.agg_words, dtype=torch.int64, device="cuda")
            rdw.simulate(rc.policies[pol], rb, ragg, stream=stream)          # warm-up
            ms = []
            for _ in range(reps):
                flush.fill_(1)
                ragg.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                rdw.simulate(rc.policies[pol], rb, ragg, stream=stream)
                e1.record(stream)
                torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
            rdw.check(stream)
            rl, rs = int(ragg[-2].item()), int(ragg[-1].item())
            rdw.close()
            tl, ts, tmax = reduce_job(rl, rs, statistics.median(ms) / 1e3, red_dev)
            return {"value": tl / tmax, "unit": UNIT, "ms_per_launch": 1e3 * tmax, "launch_events": tl,
                    "roofline": _alu_roofline(ts / n, tl / n, tmax, sms, peak_mhz)}

        lr = regime("paper11", "urgengo", 1000, 10_000_000_000, 5)
        lr["workload"] = ("paper11 (BASELINE.json configs[1]): 1000 scenarios x 10 s per GPU, UrgenGo; "
                          "latency build (fewer warps than schedulers x 2)")
        line["latency_regime"] = lr
        tr_ = regime("scaleout", "urgengo", 300_000, 1_000_000_000, 2)
        tr_["workload"] = ("scaleout (BASELINE.json configs[4]) workload, 300k scenarios x 1 s per GPU, UrgenGo; "
                           "throughput build (two scenarios per warp)")
        line["throughput_regime"] = tr_

    # ---- cpu_baseline + parity: the oracle, unchanged, on BASELINE.md's sample (rank 0, N = 1) ----
    if want_cpu:
        cores = _cores()
        sample = baseline_sample(lo, S)
        pool = oracle_pool(a.config, a.policy, cores, "spawn")
        oracle_sample(pool, [sample[0]] * cores, min(b0.horizon_ns, 1_000_000_000))   # start every worker
        res, dt = oracle_sample(pool, sample, b0.horizon_ns)
        pool.close()
        mism = [s for s, r, _, _ in res if not np.array_equal(r[0], rec_np[s - lo])]
        ol = sum(r[2] for r in res)
        line["cpu_baseline"] = {"value": ol / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": f"BASELINE.md sample of the configuration: {len(sample)} scenarios (the first "
                                          f"256, the last 256, every {BASELINE_SAMPLE_STRIDE}th) at the full horizon, "
                                          f"one oracle process per core; CPU {_cpu_model()}",
                                "seconds": dt, "single_core_value": ol / sum(r[3] for r in res)}
        line["parity_sample"] = {"scenarios": len(sample), "bit_exact": not mism, "mismatches": mism[:8]}

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    dw.close()


if __name__ == "__main__":
    main()
