// urg_api.cu -- host side of liburg.so: the C ABI declared in include/urg.h.
//
// Validates descriptors (errors name the offending field), packs the workload
// template into the device blob (urg_layout.h), owns its HBM copy, and launches
// the simulation kernel (urg_sim.cu) on the caller's stream.  No simulation
// arithmetic happens here: every step of the path runs in the kernel.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/urg.h"
#include "urg_layout.h"

typedef void (*urg_sim_fn)(const uint8_t *blob, const UrgSimParams P, uint32_t *records, unsigned long long *agg,
                           unsigned long long *work, long long *err);
const void *urg_sim_kernel_for(uint32_t kind, uint32_t flags, bool kern_q, bool wide, bool cal, bool ext,
                               bool pk, bool small);   // urg_sim.cu
extern "C" __global__ void urg_cal_hist_kernel(const int64_t *buf, uint64_t count, uint64_t cap, long long *ws,
                                               int pass);
extern "C" __global__ void urg_cal_pick_kernel(long long *ws, int pass, int pct, long long *result);
extern "C" __global__ void urg_philox_kat_kernel(const uint4 *ctr, const uint2 *key, uint4 *out, int n);

struct urg_workload {
    uint32_t num_chains, num_prio, rt_bins;
    int64_t launch_ns, launch_akb_ns, sync_lo_ns, sync_hi_ns, jitter_ns, rt_bin_ns;
    std::vector<int64_t> period, deadline;
    std::vector<uint8_t> blob;        // host copy of the packed template
    uint8_t *d_blob = nullptr;        // HBM copy
    unsigned long long *d_work = nullptr;   // per-launch scenario counter
    long long *d_err = nullptr;       // [code, scenario]
    int device = 0;
    int num_sms = 148;
    bool has_kern_q = false;          // per-kernel factor table present (selects the kernel instantiation)
    uint32_t max_tasks = 0;           // most tasks of any chain (CPU predictor state size, R26)
    bool has_free = false;            // some task ends with cudaFree (R28)
    int64_t free_ns = 0;
    uint32_t cpu_cores = 0;           // cores shared by the chains' threads, 0 = one each (R29)
    uint32_t alpha_pm = 0;            // contention slow-down (R30)
    bool has_copy = false;            // some operation is a memcpy (R31)
    uint32_t num_lanes = 0;           // simulated threads: chains, or tasks under per-task executors (R32)
    bool task_exec = false;
    uint32_t num_variants = 1, nk_total = 0;   // template variants (R33) and kernels per variant
    UrgKernRec *d_kern = nullptr;     // HBM: [num_variants][nk_total] kernel records
    UrgVarRec *d_var = nullptr;       // HBM: [num_variants][num_lanes] estimate totals
    uint64_t kern_bytes = 0;
};

static thread_local std::string g_err;

// debug-build event trace (urg_debug_set_trace; liburg_debug.so records, the product build ignores it)
static struct { int64_t *buf; uint64_t cap, scenario; } g_trace = {nullptr, 0, 0};

// cudaFuncSetAttribute (dynamic shared memory, carveout) is process-global per kernel function:
// the attribute set of one launch and its <<<>>> stay together under this lock, so two host
// threads launching the same instantiation with different geometries cannot interleave.
static std::mutex g_launch_mu;

static urg_status fail(urg_status st, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

static urg_status cuda_fail(cudaError_t e, const char *what)
{
    return fail(URG_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CUDA_TRY(x, what)                                  \
    do {                                                   \
        cudaError_t e_ = (x);                              \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

extern "C" const char *urg_last_error(void) { return g_err.c_str(); }

static uint32_t align16(uint32_t x) { return (x + 15u) & ~15u; }

extern "C" urg_status urg_create_workload(const urg_workload_desc *d, urg_workload **out)
{
    g_err.clear();
    if (!out) return fail(URG_EINVAL, "out must not be NULL");
    *out = nullptr;
    if (!d) return fail(URG_EINVAL, "desc must not be NULL");
    if (d->num_chains == 0) return fail(URG_EINVAL, "num_chains must be >= 1");
    if (d->num_chains > 32) return fail(URG_ERANGE, "num_chains = %u exceeds 32 (one warp lane per chain)", d->num_chains);
    if (!d->chains) return fail(URG_EINVAL, "chains must not be NULL");
    if (d->num_prio < 1 || d->num_prio > 8) return fail(URG_EINVAL, "num_prio must be in 1..8");
    if (d->launch_ns < 0) return fail(URG_EINVAL, "launch_ns must be >= 0");
    if (d->launch_akb_ns < 0) return fail(URG_EINVAL, "launch_akb_ns must be >= 0");
    if (d->sync_lo_ns < 0 || d->sync_hi_ns < d->sync_lo_ns)
        return fail(URG_EINVAL, "sync range must satisfy 0 <= sync_lo_ns <= sync_hi_ns");
    if (d->sync_hi_ns >= 0xFFFFFFFFLL) return fail(URG_ERANGE, "sync_hi_ns must be < 2^32 - 1 (the kernel keeps sync costs in 32 bits)");
    if (d->jitter_ns < 0 || d->jitter_ns >= 0xFFFFFFFFLL) return fail(URG_EINVAL, "jitter_ns must be in [0, 2^32 - 1)");
    if (d->rt_bin_ns <= 0) return fail(URG_EINVAL, "rt_bin_ns must be > 0");
    if (d->rt_bins < 1 || d->rt_bins > (1u << 20)) return fail(URG_EINVAL, "rt_bins must be in 1..2^20");
    if (d->free_ns < 0 || d->free_ns >= (1LL << 40)) return fail(URG_EINVAL, "free_ns must be in [0, 2^40)");
    if (d->cpu_cores > 32) return fail(URG_EINVAL, "cpu_cores must be <= 32 (0 = one core per chain thread)");
    if (d->contention_permille > 100000) return fail(URG_EINVAL, "contention_permille must be <= 100000");
    if (d->executors > URG_EXEC_TASK) return fail(URG_EINVAL, "executors must be URG_EXEC_CHAIN or URG_EXEC_TASK");
    const uint32_t n_var = d->num_variants ? d->num_variants : 1u;
    if (n_var > 65536) return fail(URG_EINVAL, "num_variants must be <= 65536");
    if (n_var > 1 && !d->variant_kernels) return fail(URG_EINVAL, "variant_kernels must not be NULL when num_variants > 1");

    uint32_t n_tasks = 0, n_kern = 0;
    for (uint32_t c = 0; c < d->num_chains && d->chains; ++c)
        for (uint32_t j = 0; j < d->chains[c].num_tasks && d->chains[c].tasks; ++j)
            if ((d->chains[c].tasks[j].flags & 1u) && d->free_ns <= 0)
                return fail(URG_EINVAL, "chains[%u].tasks[%u] ends with cudaFree: free_ns must be > 0", c, j);
    for (uint32_t c = 0; c < d->num_chains; ++c) {
        const urg_chain_desc &ch = d->chains[c];
        if (ch.period_ns <= 0) return fail(URG_EINVAL, "chains[%u].period_ns must be > 0", c);
        if (ch.deadline_ns <= 0) return fail(URG_EINVAL, "chains[%u].deadline_ns must be > 0", c);
        if (ch.offset_ns < 0) return fail(URG_EINVAL, "chains[%u].offset_ns must be >= 0", c);
        if (ch.period_ns >= (1LL << 40) || ch.deadline_ns >= (1LL << 40) || ch.offset_ns >= (1LL << 40))
            return fail(URG_ERANGE, "chains[%u]: period/deadline/offset must be < 2^40 ns", c);
        if (ch.num_tasks < 1) return fail(URG_EINVAL, "chains[%u].num_tasks must be >= 1", c);
        if (!ch.tasks) return fail(URG_EINVAL, "chains[%u].tasks must not be NULL", c);
        for (uint32_t j = 0; j < ch.num_tasks; ++j) {
            const urg_task_desc &t = ch.tasks[j];
            if (t.num_kernels < 1) return fail(URG_EINVAL, "chains[%u].tasks[%u].num_kernels must be >= 1", c, j);
            if (t.flags > 1) return fail(URG_EINVAL, "chains[%u].tasks[%u].flags has unknown bits", c, j);
            if (!t.kernels) return fail(URG_EINVAL, "chains[%u].tasks[%u].kernels must not be NULL", c, j);
            for (uint32_t k = 0; k < t.num_kernels; ++k) {
                const urg_kernel_desc &kd = t.kernels[k];
                if (kd.nominal_ns == 0)
                    return fail(URG_EINVAL, "chains[%u].tasks[%u].kernels[%u].nominal_ns must be > 0", c, j, k);
                if (kd.util_permille > 1000)
                    return fail(URG_EINVAL, "chains[%u].tasks[%u].kernels[%u].util_permille must be <= 1000", c, j, k);
                if (kd.flags > 1)
                    return fail(URG_EINVAL, "chains[%u].tasks[%u].kernels[%u].flags has unknown bits", c, j, k);
            }
            n_kern += t.num_kernels;
        }
        n_tasks += ch.num_tasks;
    }
    // template variants (R33): every set has the chains' structure; memcpy flags are structural
    if ((uint64_t)n_var * n_kern >= (1ull << 31))
        return fail(URG_ERANGE, "num_variants x kernels = %llu kernel records exceeds 2^31",
                    (unsigned long long)n_var * n_kern);
    for (uint32_t v = 1, g = 0; v < n_var; ++v, g = 0)
        for (uint32_t c = 0; c < d->num_chains; ++c)
            for (uint32_t j = 0; j < d->chains[c].num_tasks; ++j)
                for (uint32_t k = 0; k < d->chains[c].tasks[j].num_kernels; ++k, ++g) {
                    const urg_kernel_desc &kd = d->variant_kernels[(uint64_t)(v - 1) * n_kern + g];
                    if (kd.nominal_ns == 0)
                        return fail(URG_EINVAL, "variant_kernels[%u][%u].nominal_ns must be > 0", v, g);
                    if (kd.util_permille > 1000)
                        return fail(URG_EINVAL, "variant_kernels[%u][%u].util_permille must be <= 1000", v, g);
                    if (kd.flags != d->chains[c].tasks[j].kernels[k].flags)
                        return fail(URG_EINVAL, "variant_kernels[%u][%u].flags must equal the chains' kernel flags",
                                    v, g);
                }
    const bool te = d->executors == URG_EXEC_TASK;
    const uint32_t n_lanes = te ? n_tasks : d->num_chains;
    if (n_lanes > 32)
        return fail(URG_ERANGE, "per-task executors: %u tasks exceed 32 (one warp lane per executor thread)", n_lanes);

    // ---- pack the blob ----
    UrgBlobHeader h = {};
    h.magic = URG_BLOB_MAGIC;
    h.num_chains = n_lanes;
    h.num_tasks = n_tasks;
    h.num_kernels = n_kern;
    uint32_t off = align16(sizeof(UrgBlobHeader));
    h.off_chains = off; off = align16(off + n_lanes * (uint32_t)sizeof(UrgChainRec));
    h.off_tasks = off;  off = align16(off + n_tasks * (uint32_t)sizeof(UrgTaskRec));
    h.off_kerns = 0;    // kernel records are read from global memory (R33), not staged
    if (d->inst_quantiles_q16) { h.off_inst_q = off; off = align16(off + URG_QTABLE * 4); }
    if (d->kern_quantiles_q16) { h.off_kern_q = off; off = align16(off + URG_QTABLE * 4); }
    h.total_bytes = off;
    if (off > URG_MAX_BLOB_BYTES)
        return fail(URG_ERANGE, "template needs %u bytes of shared memory, more than the %u-byte budget", off,
                    URG_MAX_BLOB_BYTES);

    urg_workload *w = new urg_workload();
    w->num_chains = d->num_chains; w->num_prio = d->num_prio; w->rt_bins = d->rt_bins;
    w->launch_ns = d->launch_ns; w->launch_akb_ns = d->launch_akb_ns;
    w->sync_lo_ns = d->sync_lo_ns; w->sync_hi_ns = d->sync_hi_ns;
    w->jitter_ns = d->jitter_ns; w->rt_bin_ns = d->rt_bin_ns;
    w->has_kern_q = d->kern_quantiles_q16 != nullptr;
    w->free_ns = d->free_ns;
    w->cpu_cores = d->cpu_cores;
    w->alpha_pm = d->contention_permille;
    w->num_lanes = n_lanes; w->task_exec = te;
    w->num_variants = n_var; w->nk_total = n_kern;
    std::vector<UrgKernRec> krs((size_t)n_var * n_kern);
    std::vector<UrgVarRec> vrs((size_t)n_var * n_lanes);
    w->blob.assign(off, 0);
    memcpy(w->blob.data(), &h, sizeof h);
    UrgChainRec *chs = (UrgChainRec *)(w->blob.data() + h.off_chains);
    UrgTaskRec *tks = (UrgTaskRec *)(w->blob.data() + h.off_tasks);
    uint32_t tb = 0, kb = 0, lane = 0;
    for (uint32_t c = 0; c < d->num_chains; ++c) {
        const urg_chain_desc &ch = d->chains[c];
        uint32_t n_local = 0;
        for (uint32_t j = 0; j < ch.num_tasks; ++j) n_local += ch.tasks[j].num_kernels;
        // one thread record per chain, or per task of the chain (R32), chain-major
        for (uint32_t j = 0, k_first = 0; j < (te ? ch.num_tasks : 1u); k_first += ch.tasks[j].num_kernels, ++j) {
            UrgChainRec &r = chs[lane++];
            r.period_ns = ch.period_ns; r.deadline_ns = ch.deadline_ns; r.offset_ns = ch.offset_ns;
            r.num_tasks = ch.num_tasks; r.task_base = tb; r.num_kernels = n_local;
            r.kern_base = kb; r.cpu_sigma_ppm = ch.cpu_sigma_ppm; r.gpu_sigma_ppm = ch.gpu_sigma_ppm;
            r.chain_id = c; r.stage = te ? j : 0; r.stage_end = te ? j + 1 : ch.num_tasks; r.k_first = k_first;
            r.cpu_est_total = 0;
            for (uint32_t q = r.stage; q < ch.num_tasks; ++q) r.cpu_est_total += ch.tasks[q].cpu_estimate_ns;
        }
        uint32_t local = 0;
        for (uint32_t j = 0; j < ch.num_tasks; ++j) {
            const urg_task_desc &t = ch.tasks[j];
            tks[tb + j] = UrgTaskRec{t.cpu_nominal_ns, t.cpu_estimate_ns, t.num_kernels, t.flags};
            if (t.flags & 1u) w->has_free = true;
            for (uint32_t k = 0; k < t.num_kernels; ++k)
            {
                krs[kb + local + k] = UrgKernRec{t.kernels[k].nominal_ns, t.kernels[k].estimate_ns,
                                                 t.kernels[k].util_permille, t.kernels[k].flags};
                if (t.kernels[k].flags & 1u) w->has_copy = true;
            }
            local += t.num_kernels;
        }
        if (ch.num_tasks > w->max_tasks) w->max_tasks = ch.num_tasks;
        for (uint32_t v = 1; v < n_var; ++v)
            for (uint32_t k = 0; k < local; ++k) {
                const urg_kernel_desc &kd = d->variant_kernels[(uint64_t)(v - 1) * n_kern + kb + k];
                krs[(size_t)v * n_kern + kb + k] = UrgKernRec{kd.nominal_ns, kd.estimate_ns, kd.util_permille, kd.flags};
            }
        tb += ch.num_tasks; kb += local;
        w->period.push_back(ch.period_ns);
        w->deadline.push_back(ch.deadline_ns);
    }
    // per (variant, thread) estimate totals: Eq. 2's kernel sum from the thread's first kernel, and the
    // chain's total (LCUF, R27)
    for (uint32_t v = 0; v < n_var; ++v)
        for (uint32_t l = 0; l < n_lanes; ++l) {
            const UrgChainRec &r = chs[l];
            int64_t g = 0, gc = 0;
            for (uint32_t k = 0; k < r.num_kernels; ++k) {
                const int64_t e = krs[(size_t)v * n_kern + r.kern_base + k].estimate_ns;
                gc += e;
                if (k >= r.k_first) g += e;
            }
            vrs[(size_t)v * n_lanes + l] = UrgVarRec{g, gc};
        }
    if (d->inst_quantiles_q16) memcpy(w->blob.data() + h.off_inst_q, d->inst_quantiles_q16, URG_QTABLE * 4);
    if (d->kern_quantiles_q16) memcpy(w->blob.data() + h.off_kern_q, d->kern_quantiles_q16, URG_QTABLE * 4);

    cudaError_t e;
    if ((e = cudaGetDevice(&w->device)) != cudaSuccess) { delete w; return cuda_fail(e, "cudaGetDevice"); }
    cudaDeviceGetAttribute(&w->num_sms, cudaDevAttrMultiProcessorCount, w->device);
    if ((e = cudaMalloc(&w->d_blob, off)) != cudaSuccess) { delete w; return fail(URG_ENOMEM, "cudaMalloc(blob)"); }
    if ((e = cudaMalloc(&w->d_work, 64)) != cudaSuccess) { cudaFree(w->d_blob); delete w; return fail(URG_ENOMEM, "cudaMalloc(work)"); }
    w->d_err = (long long *)(w->d_work + 2);
    w->kern_bytes = (uint64_t)krs.size() * sizeof(UrgKernRec);
    if ((e = cudaMalloc(&w->d_kern, w->kern_bytes)) != cudaSuccess ||
        (e = cudaMalloc(&w->d_var, vrs.size() * sizeof(UrgVarRec))) != cudaSuccess) {
        cudaFree(w->d_blob); cudaFree(w->d_work); cudaFree(w->d_kern); delete w;
        return fail(URG_ENOMEM, "cudaMalloc(kernel records)");
    }
    if ((e = cudaMemcpy(w->d_blob, w->blob.data(), off, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(w->d_kern, krs.data(), w->kern_bytes, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(w->d_var, vrs.data(), vrs.size() * sizeof(UrgVarRec), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemset(w->d_work, 0, 64)) != cudaSuccess) {
        cudaFree(w->d_blob); cudaFree(w->d_work); cudaFree(w->d_kern); cudaFree(w->d_var); delete w;
        return cuda_fail(e, "copying the template to the device");
    }
    *out = w;
    return URG_OK;
}

extern "C" void urg_destroy_workload(urg_workload *w)
{
    if (!w) return;
    cudaFree(w->d_blob);
    cudaFree(w->d_work);
    cudaFree(w->d_kern);
    cudaFree(w->d_var);
    delete w;
}

extern "C" uint64_t urg_agg_words(const urg_workload *w)
{
    return w ? (uint64_t)w->num_chains * (5 + w->rt_bins + 101) + URG_COLL_BINS + 2 : 0;
}

extern "C" uint64_t urg_template_bytes(const urg_workload *w)
{
    return w ? (uint64_t)w->blob.size() + w->kern_bytes : 0;
}

static urg_status validate_call(const urg_workload *w, const urg_policy *p, const urg_batch *b)
{
    if (!w || !p || !b) return fail(URG_EINVAL, "workload, policy and batch must not be NULL");
    if (p->kind > URG_LCUF) return fail(URG_EINVAL, "policy.kind must be 0..6");
    if (p->flags > 15) return fail(URG_EINVAL, "policy.flags has unknown bits");
    if (p->sync_mode > URG_SYNC_OVERLAP) return fail(URG_EINVAL, "policy.sync_mode must be 0..3");
    if (p->delta_eval_ns <= 0) return fail(URG_EINVAL, "policy.delta_eval_ns must be > 0");
    if (p->sleep_ns <= 0) return fail(URG_EINVAL, "policy.sleep_ns must be > 0");
    if (p->noise_permille > 1000) return fail(URG_EINVAL, "policy.noise_permille must be <= 1000");
    if (p->cpu_ma_window > 64) return fail(URG_EINVAL, "policy.cpu_ma_window must be <= 64");
    if (w->task_exec && p->cpu_ma_window)
        return fail(URG_EINVAL, "policy.cpu_ma_window must be 0 with per-task executors (DESIGN.md R32)");
    if (b->fa_num == 0 || b->fa_den == 0) return fail(URG_EINVAL, "batch.fa_num and batch.fa_den must be > 0");
    if (b->fd_num == 0 || b->fd_den == 0) return fail(URG_EINVAL, "batch.fd_num and batch.fd_den must be > 0");
    if (b->ftight_permille > 1000) return fail(URG_EINVAL, "batch.ftight_permille must be <= 1000");
    if (b->horizon_ns < 0 || b->horizon_ns >= (1LL << 44)) return fail(URG_ERANGE, "batch.horizon_ns must be in [0, 2^44)");
    if (b->scenario_begin + b->scenario_count > (1ULL << 32) || b->scenario_begin >= (1ULL << 32))
        return fail(URG_ERANGE, "batch: scenario indices must stay below 2^32");
    for (uint32_t c = 0; c < w->num_chains; ++c) {
        const int64_t Pp = w->period[c] * (int64_t)b->fa_den / (int64_t)b->fa_num;   // < 2^72? guarded below
        if ((double)w->period[c] * b->fa_den > 4.0e18 || (double)w->deadline[c] * b->fd_num > 4.0e18)
            return fail(URG_ERANGE, "chains[%u]: period*fa_den or deadline*fd_num overflows int64", c);
        if (Pp <= w->jitter_ns) return fail(URG_EINVAL, "chains[%u]: scaled period P' = %lld must exceed jitter_ns", c, (long long)Pp);
        if (w->deadline[c] * (int64_t)b->fd_num / (int64_t)b->fd_den >= (1LL << 44))
            return fail(URG_ERANGE, "chains[%u]: scaled deadline must be < 2^44 ns", c);
    }
    return URG_OK;
}

static void fill_params(const urg_workload *w, const urg_policy *p, const urg_batch *b, UrgSimParams &P)
{
    memset(&P, 0, sizeof P);
    P.num_chains = w->num_chains; P.num_lanes = w->num_lanes; P.task_exec = w->task_exec ? 1u : 0u;
    P.kern = w->d_kern; P.var = w->d_var; P.nk_total = w->nk_total; P.num_variants = w->num_variants;
    P.num_prio = w->num_prio; P.rt_bins = w->rt_bins;
    P.agg_stride = 5 + w->rt_bins + 101;
    P.launch_ns = w->launch_ns; P.launch_akb_ns = w->launch_akb_ns;
    P.sync_lo_ns = w->sync_lo_ns; P.sync_hi_ns = w->sync_hi_ns;
    P.jitter_ns = w->jitter_ns; P.rt_bin_ns = w->rt_bin_ns;
    P.kind = p->kind; P.flags = p->flags; P.sync_mode = p->sync_mode; P.util_exempt = p->util_exempt_permille;
    P.delta_eval_ns = p->delta_eval_ns; P.lax_threshold_ns = p->lax_threshold_ns; P.sleep_ns = p->sleep_ns;
    P.noise_pm = p->noise_permille; P.ma_w = p->cpu_ma_window;
    P.has_free = w->has_free ? 1u : 0u; P.free_ns = w->free_ns; P.cpu_cores = w->cpu_cores; P.alpha_pm = w->alpha_pm;
    P.has_copy = w->has_copy ? 1u : 0u;
    P.seed = b->seed; P.scenario_begin = b->scenario_begin; P.scenario_count = b->scenario_count;
    P.horizon_ns = b->horizon_ns;
    P.fa_num = b->fa_num; P.fa_den = b->fa_den; P.fd_num = b->fd_num; P.fd_den = b->fd_den;
    P.ftight_permille = b->ftight_permille; P.tight_explicit = b->tight_explicit; P.tight_mask = b->tight_mask;
    P.trace_buf = g_trace.buf; P.trace_cap = g_trace.cap; P.trace_scn = g_trace.scenario;
    P.busy_launch_ns = w->launch_ns + (p->kind == URG_URGENGO ? w->launch_akb_ns : 0);
    auto d32 = [](int64_t d) -> uint32_t { return d >= (int64_t)0x80000000LL ? 0x80000000u : (uint32_t)d; };
    P.busy_launch_d32 = d32(P.busy_launch_ns);
    P.sleep_d32 = d32(p->sleep_ns);
    P.lth_excl = p->lax_threshold_ns < 0 ? 0ull : (uint64_t)p->lax_threshold_ns + 1ull;
}

// Launch geometry: one warp per scenario in flight, persistent CTAs pulling scenarios
// from an atomic counter.  Few scenarios: spread them one warp each over all SMs
// (the batch is latency-bound: fewer warps per scheduler, same per-scenario time).
// Many scenarios: the largest CTA the kernel allows, as many CTAs per SM as
// registers and shared memory (the staged template is per CTA) let reside.
static urg_status geometry(const urg_workload *w, const void *fn, uint64_t count, uint32_t smem_fixed,
                           uint32_t per_lane, int &warps, int &ctas, uint32_t &smem)
{
    cudaFuncAttributes fa;
    CUDA_TRY(cudaFuncGetAttributes(&fa, fn), "cudaFuncGetAttributes");
    int max_w = fa.maxThreadsPerBlock / 32;
    if (max_w > 32) max_w = 32;
    const uint64_t need = (count + (uint64_t)w->num_sms - 1) / (uint64_t)w->num_sms;   // warps per SM to hold all
    warps = (int)(need < (uint64_t)max_w ? need : (uint64_t)max_w);
    if (const char *ew = getenv("URG_WARPS_PER_CTA")) warps = atoi(ew);
    if (warps < 1) warps = 1;
    if (warps > max_w) warps = max_w;
    smem = smem_fixed + (uint32_t)warps * 32u * per_lane;
    CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
             "cudaFuncSetAttribute(smem)");
    int per_sm = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, warps * 32, smem), "cudaOccupancy");
    if (per_sm < 1) return fail(URG_ERANGE, "urg_sim_kernel cannot reside on an SM with %u B of shared memory", smem);
    const uint64_t blocks_needed = (count + warps - 1) / warps;
    const uint64_t resident = (uint64_t)w->num_sms * (uint64_t)per_sm;
    ctas = (int)(blocks_needed < resident ? blocks_needed : resident);
    if (ctas < 1) ctas = 1;
    {   // leave the rest of the SM's 256 KB to L1: the kernel records of the template variants are
        // read through it (R33); shared memory only for the CTAs an SM actually holds
        const uint64_t per_sm_used = ((uint64_t)ctas + w->num_sms - 1) / w->num_sms;
        uint64_t pct = (100ull * per_sm_used * (smem + 1024u) + 228u * 1024u - 1) / (228u * 1024u);
        if (pct > 100) pct = 100;
        CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)pct),
                 "cudaFuncSetAttribute(carveout)");
    }
    return URG_OK;
}

// Parameters, kernel instantiation and geometry of one simulation launch.  Shared memory:
// the template blob, its mbarrier, then per lane the Phase B snapshot (16 B) and, with the
// CPU predictor (R26), max_tasks x (W + 2) words of predictor state.
static urg_status prepare_launch(const urg_workload *w, const urg_policy *p, const urg_batch *b, bool wide, bool cal,
                                 UrgSimParams &P, urg_sim_fn &fn, int &warps, int &ctas)
{
    fill_params(w, p, b, P);
    // the extended-model build only when the batch uses noise, the CPU predictor or cudaFree
    bool ext = (p->kind == URG_URGENGO && p->noise_permille) || (p->kind >= URG_URGENGO && p->cpu_ma_window) ||
               w->has_free || w->cpu_cores > 0 || w->alpha_pm > 0 || w->has_copy || w->task_exec;
    if (const char *ee = getenv("URG_EXT")) ext = ext || atoi(ee) != 0;   // test hook: force the extended build
    // two scenarios per warp in the throughput core build when the chains fit a half warp
    bool pk = wide && !cal && !ext && w->num_chains <= 16;
    if (const char *ep = getenv("URG_PACK")) pk = pk && atoi(ep) != 0;          // test hook: disable packing
    // the small latency core build (255-register cap) when the batch needs at most 8 warps per SM
    bool small = !wide && !cal && !ext && b->scenario_count <= (uint64_t)w->num_sms * 8u;
    if (const char *es = getenv("URG_SMALL")) small = small && atoi(es) != 0;    // test hook: disable it
    fn = (urg_sim_fn)urg_sim_kernel_for(p->kind, p->kind == URG_URGENGO ? p->flags : 0, w->has_kern_q, wide && !cal,
                                        cal, ext, pk, small);
    if (!fn) return fail(URG_EINTERNAL, "no kernel instantiation for kind %u flags %u", p->kind, p->flags);
    P.blob_bytes = (uint32_t)w->blob.size();
    P.mbar_offset = align16(P.blob_bytes);
    P.snap_offset = align16(P.mbar_offset + 16);
    uint32_t per_lane = URG_SNAP_BYTES_PER_LANE;
    if (p->kind >= URG_URGENGO && P.ma_w) {   // UrgenGo and the R27 policies estimate remaining work
        P.ma_max_tasks = w->max_tasks;
        P.ma_slot = w->max_tasks * (P.ma_w + 2);
        per_lane += P.ma_slot * 4u;
    }
    urg_status st = geometry(w, (const void *)fn, pk ? (b->scenario_count + 1) / 2 : b->scenario_count,
                             P.snap_offset, per_lane, warps, ctas, P.smem_bytes);
    if (st != URG_OK) return st;
    P.ma_offset = P.snap_offset + (uint32_t)warps * 32u * URG_SNAP_BYTES_PER_LANE;
    return URG_OK;
}

extern "C" urg_status urg_simulate_batch(const urg_workload *w, const urg_policy *p, const urg_batch *b,
                                         const urg_outputs *o, void *cuda_stream)
{
    g_err.clear();
    urg_status st = validate_call(w, p, b);
    if (st != URG_OK) return st;
    if (!o || !o->agg) return fail(URG_EINVAL, "outputs.agg must not be NULL");
    if (b->scenario_count == 0) return URG_OK;
    cudaStream_t s = (cudaStream_t)cuda_stream;
    // throughput build once the batch needs more than 16 warps per SM (bench: paper11's 1000
    // scenarios use the latency build, configs[2]-[4]'s 1e5-1e8 the throughput build)
    bool wide = b->scenario_count > (uint64_t)w->num_sms * 16u;
    if (const char *ev = getenv("URG_WIDE")) wide = atoi(ev) != 0;
    UrgSimParams P;
    urg_sim_fn fn;
    int warps, ctas;
    std::lock_guard<std::mutex> lk(g_launch_mu);
    st = prepare_launch(w, p, b, wide, false, P, fn, warps, ctas);
    if (st != URG_OK) return st;
    CUDA_TRY(cudaMemsetAsync(w->d_work, 0, 8, s), "cudaMemsetAsync(work counter)");
    fn<<<ctas, warps * 32, P.smem_bytes, s>>>(w->d_blob, P, o->records, (unsigned long long *)o->agg, w->d_work,
                                              w->d_err);
    CUDA_TRY(cudaGetLastError(), "launching urg_sim_kernel");
    return URG_OK;
}

// ---- TH_urgent calibration (Q5) ----
static int64_t cal_end(const urg_batch *b, int64_t window_ns) { return b->horizon_ns < window_ns ? b->horizon_ns : window_ns; }
static uint64_t cal_cap(const urg_batch *b, int64_t window_ns) { return (uint64_t)(cal_end(b, window_ns) / 1000000) + 2; }

extern "C" uint64_t urg_calibration_words(const urg_workload *w, const urg_batch *b, int64_t window_ns)
{
    if (!w || !b || window_ns < 0) return 0;
    return b->scenario_count + b->scenario_count * cal_cap(b, window_ns) + 260;
}

extern "C" urg_status urg_calibrate(const urg_workload *w, const urg_policy *p, const urg_batch *b, int64_t window_ns,
                                    int64_t *scratch, uint64_t scratch_words, int64_t *result, void *cuda_stream)
{
    g_err.clear();
    urg_status st = validate_call(w, p, b);
    if (st != URG_OK) return st;
    if (p->kind != URG_URGENGO) return fail(URG_EINVAL, "policy.kind must be URG_URGENGO (the AKB is UrgenGo's)");
    if (window_ns < 0) return fail(URG_EINVAL, "window_ns must be >= 0");
    if (!scratch || !result) return fail(URG_EINVAL, "scratch and result must not be NULL");
    if (b->scenario_count == 0) return fail(URG_EINVAL, "batch.scenario_count must be >= 1");
    const uint64_t need = urg_calibration_words(w, b, window_ns);
    if (scratch_words < need) return fail(URG_ERANGE, "scratch has %llu words, calibration needs %llu",
                                          (unsigned long long)scratch_words, (unsigned long long)need);
    cudaStream_t s = (cudaStream_t)cuda_stream;
    urg_policy pc = *p;
    pc.lax_threshold_ns = -1;                                   // nothing is truly urgent while sampling
    UrgSimParams P;
    urg_sim_fn fn;
    int warps, ctas;
    std::lock_guard<std::mutex> lk(g_launch_mu);
    st = prepare_launch(w, &pc, b, false, true, P, fn, warps, ctas);
    if (st != URG_OK) return st;
    P.cal_end = cal_end(b, window_ns);
    P.cal_cap = cal_cap(b, window_ns);
    P.cal_buf = scratch;
    long long *ws = (long long *)(scratch + b->scenario_count + b->scenario_count * P.cal_cap);
    CUDA_TRY(cudaMemsetAsync(ws, 0, 260 * 8, s), "cudaMemsetAsync(select workspace)");
    CUDA_TRY(cudaMemsetAsync(w->d_work, 0, 8, s), "cudaMemsetAsync(work counter)");
    fn<<<ctas, warps * 32, P.smem_bytes, s>>>(w->d_blob, P, nullptr, nullptr, w->d_work, w->d_err);
    CUDA_TRY(cudaGetLastError(), "launching the calibration simulation");
    int grid = (int)(b->scenario_count < (uint64_t)w->num_sms * 4 ? b->scenario_count : (uint64_t)w->num_sms * 4);
    for (int pass = 7; pass >= 0; --pass) {
        urg_cal_hist_kernel<<<grid, 256, 0, s>>>(scratch, b->scenario_count, P.cal_cap, ws, pass);
        urg_cal_pick_kernel<<<1, 32, 0, s>>>(ws, pass, 95, (long long *)result);
    }
    CUDA_TRY(cudaGetLastError(), "launching the nearest-rank selection");
    return URG_OK;
}

extern "C" urg_status urg_check(const urg_workload *w, void *cuda_stream, int64_t *scenario_out);

extern "C" urg_status urg_simulate_batch_host(const urg_workload *w, const urg_policy *p, const urg_batch *b,
                                              const urg_outputs *host_o, void *cuda_stream)
{
    g_err.clear();
    urg_status st = validate_call(w, p, b);
    if (st != URG_OK) return st;
    if (!host_o || !host_o->agg) return fail(URG_EINVAL, "outputs.agg must not be NULL");
    cudaStream_t s = (cudaStream_t)cuda_stream;
    const uint64_t nagg = urg_agg_words(w);
    const uint64_t nrec = host_o->records ? b->scenario_count * w->num_chains * 8 : 0;
    urg_outputs d = {nullptr, nullptr};
    std::vector<int64_t> tmp(nagg);
    CUDA_TRY(cudaMallocAsync((void **)&d.agg, nagg * 8, s), "cudaMallocAsync(agg)");
    if (nrec) CUDA_TRY(cudaMallocAsync((void **)&d.records, nrec * 4, s), "cudaMallocAsync(records)");
    CUDA_TRY(cudaMemsetAsync(d.agg, 0, nagg * 8, s), "cudaMemsetAsync(agg)");
    st = urg_simulate_batch(w, p, b, &d, cuda_stream);
    if (st == URG_OK) {
        cudaError_t e = cudaMemcpyAsync(tmp.data(), d.agg, nagg * 8, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && nrec)
            e = cudaMemcpyAsync(host_o->records, d.records, nrec * 4, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) st = cuda_fail(e, "copying results to the host");
    }
    cudaFreeAsync(d.agg, s);
    if (d.records) cudaFreeAsync(d.records, s);
    if (st != URG_OK) return st;
    // a synchronous call reports a device invariant trip itself (and clears the word)
    st = urg_check(w, cuda_stream, nullptr);
    if (st != URG_OK) return st;
    for (uint64_t i = 0; i < nagg; ++i) host_o->agg[i] += tmp[i];
    return URG_OK;
}

extern "C" urg_status urg_check(const urg_workload *w, void *cuda_stream, int64_t *scenario_out)
{
    g_err.clear();
    if (!w) return fail(URG_EINVAL, "workload must not be NULL");
    long long e2[2] = {0, 0};
    cudaStream_t s = (cudaStream_t)cuda_stream;
    CUDA_TRY(cudaMemcpyAsync(e2, w->d_err, sizeof e2, cudaMemcpyDeviceToHost, s), "reading the error word");
    CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    if (scenario_out) *scenario_out = e2[1];
    if (e2[0] != 0) {
        // reported once: cleared so a later trip on this workload is recorded and reported too
        CUDA_TRY(cudaMemsetAsync(w->d_err, 0, sizeof e2, s), "clearing the error word");
        CUDA_TRY(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        return fail(URG_EINTERNAL, "device invariant %lld tripped in scenario %lld (%s)", e2[0], e2[1],
                    e2[0] == 1 ? "time did not advance" : e2[0] == 2 ? "step iteration guard"
                               : e2[0] == 17 ? "debug: kernel started before it was ready"
                               : e2[0] == 18 ? "debug: GPU capacity exceeded"
                               : e2[0] == 19 ? "debug: kernel retired at a time other than its end"
                               : e2[0] == 20 ? "debug: instance completed with kernels not launched or not done"
                               : e2[0] == 21 ? "debug: record counts inconsistent"
                               : e2[0] == 22 ? "debug: event scheduled in the past"
                               : e2[0] == 23 ? "debug: stream level out of range or urgent task not at level 0"
                                             : "unknown");
    }
    return URG_OK;
}

extern "C" urg_status urg_miss_ratios(const urg_workload *w, const int64_t *agg_host, double *per_chain_out,
                                      double *overall_out)
{
    g_err.clear();
    if (!w || !agg_host) return fail(URG_EINVAL, "workload and agg_host must not be NULL");
    const uint64_t stride = 5 + w->rt_bins + 101;
    double sum = 0.0;
    uint32_t used = 0;
    for (uint32_t c = 0; c < w->num_chains; ++c) {
        const int64_t total = agg_host[c * stride + 0], miss = agg_host[c * stride + 1];
        const double r = total ? (double)miss / (double)total : 0.0;
        if (per_chain_out) per_chain_out[c] = r;
        if (total) { sum += r; ++used; }
    }
    if (overall_out) *overall_out = used ? sum / used : 0.0;
    return URG_OK;
}

// profiling hook (liburg_stats.so, -DURG_STATS): event-loop counters of the launches since the
// last call -- [single-chain steps, multi-chain steps, Phase C dispatches, 64-bit rebases]
extern "C" urg_status urg_debug_stats(const urg_workload *w, uint64_t *out4)
{
    if (!w || !out4) return fail(URG_EINVAL, "workload and out must not be NULL");
    CUDA_TRY(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    CUDA_TRY(cudaMemcpy(out4, w->d_work + 4, 32, cudaMemcpyDeviceToHost), "reading stats");
    CUDA_TRY(cudaMemset(w->d_work + 4, 0, 32), "clearing stats");
    return URG_OK;
}

// debug hook: record the event trace of global scenario `scenario` into dev_buf (DEVICE int64:
// [0] row counter, then cap_rows rows of 6) during the following simulate calls of this process;
// dev_buf = NULL turns it off.  Only the debug build (liburg_debug.so, -DURG_DEBUG) writes rows.
extern "C" urg_status urg_debug_set_trace(int64_t *dev_buf, uint64_t cap_rows, uint64_t scenario)
{
    std::lock_guard<std::mutex> lk(g_launch_mu);
    g_trace.buf = dev_buf; g_trace.cap = dev_buf ? cap_rows : 0; g_trace.scenario = scenario;
    return URG_OK;
}

// 1 if this library is the debug build (device invariant asserts, event trace), else 0
extern "C" int urg_debug_build(void)
{
#ifdef URG_DEBUG
    return 1;
#else
    return 0;
#endif
}

// test hook: device Philox on n (ctr, key) pairs in device memory (Philox KAT / oracle cross-check)
extern "C" urg_status urg_debug_philox(const void *d_ctr, const void *d_key, void *d_out, int n, void *cuda_stream)
{
    if (n <= 0) return URG_OK;
    urg_philox_kat_kernel<<<(n + 255) / 256, 256, 0, (cudaStream_t)cuda_stream>>>((const uint4 *)d_ctr,
                                                                                   (const uint2 *)d_key,
                                                                                   (uint4 *)d_out, n);
    CUDA_TRY(cudaGetLastError(), "launching urg_philox_kat_kernel");
    return URG_OK;
}
