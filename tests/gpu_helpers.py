"""Shared helpers for the -m gpu tests: run the CUDA path through the C ABI."""
import numpy as np

from workloads.spec import RECORD_WORDS, agg_words


def gpu_run(w, p, b, records=True, stream=None):
    import torch

    from paper_2509_12207_b200.urg import DeviceWorkload

    with DeviceWorkload(w) as dw:
        agg = torch.zeros(dw.agg_words, dtype=torch.int64, device="cuda")
        rec = torch.zeros((max(b.scenario_count, 1), w.num_chains, RECORD_WORDS), dtype=torch.int32,
                          device="cuda") if records else None
        dw.simulate(p, b, agg, rec, stream=stream)
        dw.check(stream)
        torch.cuda.synchronize()
        a = agg.cpu().numpy()
        r = rec.cpu().numpy().view(np.uint32)[: b.scenario_count] if records else None
    return r, a


def assert_same(oracle_res, gpu_rec, gpu_agg, ctx=""):
    o_rec, o_agg = oracle_res.records, oracle_res.agg
    if gpu_rec is not None and not np.array_equal(o_rec, gpu_rec):
        diff = np.argwhere(o_rec != gpu_rec)
        s, c, wd = diff[0]
        raise AssertionError(f"{ctx}: record mismatch at scenario {s} chain {c} word {wd}: "
                             f"oracle {o_rec[s, c].tolist()} gpu {gpu_rec[s, c].tolist()} ({len(diff)} words differ)")
    if not np.array_equal(o_agg, gpu_agg):
        idx = np.flatnonzero(o_agg != gpu_agg)
        raise AssertionError(f"{ctx}: aggregate mismatch at words {idx[:8].tolist()}: oracle "
                             f"{o_agg[idx[:8]].tolist()} gpu {gpu_agg[idx[:8]].tolist()}")


def agg_from_records(rec: np.ndarray, C: int, rt_bins: int) -> np.ndarray:
    """Counters and miss-ratio bins of the aggregate recomputed from per-scenario records."""
    stride = 5 + rt_bins + 101
    out = np.zeros(agg_words(C, rt_bins), np.int64)
    r = rec.astype(np.int64)
    for c in range(C):
        out[c * stride + 0] = r[:, c, 0].sum()
        out[c * stride + 1] = r[:, c, 1].sum()
        out[c * stride + 2] = r[:, c, 2].sum()
        out[c * stride + 3] = r[:, c, 3].sum()
        out[c * stride + 4] = (r[:, c, 6] | (r[:, c, 7] << 32)).sum()
        tot, miss = r[:, c, 0], r[:, c, 1]
        ok = tot > 0
        bins = (100 * miss[ok]) // tot[ok]
        np.add.at(out, c * stride + 5 + rt_bins + bins, 1)
    out[-2] = r[:, :, 4].sum()
    return out
