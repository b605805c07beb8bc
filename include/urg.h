/*
 * include/urg.h -- C ABI of the B200 batched UrgenGo launch-policy simulator.
 *
 * Implemented by liburg.so (paper_2509_12207_b200/csrc/, CUDA for sm_100a).
 * All integers; times are int64 nanoseconds; utilisation is per-mille of the GPU.
 * The rules being simulated are DESIGN.md "Model M0" (R0-R23), our reading of
 * arXiv 2509.12207 (UrgenGo); every function below cites the passage that
 * defines what it computes.
 *
 * Ownership: the caller owns every descriptor and output buffer.  The library
 * allocates only inside urg_create_workload (a device copy of the template and
 * two small device scratch words) and frees them in urg_destroy_workload.
 * Errors: every call returns a urg_status; urg_last_error() gives a
 * thread-local message naming the offending field, e.g.
 * "chains[3].tasks[1].kernels[7].nominal_ns must be > 0".
 */
#ifndef URG_H
#define URG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    URG_OK = 0,
    URG_EINVAL = -1,     /* malformed descriptor or argument */
    URG_ERANGE = -2,     /* valid but outside what the device path supports (C > 32, template > smem) */
    URG_ENOMEM = -3,     /* device allocation failed */
    URG_ECUDA = -4,      /* a CUDA runtime call failed */
    URG_EINTERNAL = -5   /* the kernel tripped an internal invariant (see urg_check) */
} urg_status;

/* One GPU operation of a task: a kernel's lookup-table record (Table 1)
 * or a memcpy (flags bit 0).
 * nominal_ns: execution time before per-scenario factors (> 0);
 * estimate_ns: ~E^gpu_k used in Eq. 2; util_permille: U_k in [0, 1000]. */
typedef struct {
    uint32_t nominal_ns;
    uint32_t estimate_ns;
    uint16_t util_permille;
    uint16_t flags;            /* bit 0 (URG_OP_MEMCPY): runs on the copy engine, one at a time, no
                                  stream priority, no compute capacity (Table 3, PAPER.md:374;
                                  DESIGN.md R31); other bits must be 0 */
} urg_kernel_desc;
enum { URG_OP_MEMCPY = 1 };

/* One task: a CPU segment, then num_kernels (>= 1) kernels launched in order on
 * one stream, then a final stream synchronisation. */
typedef struct {
    uint32_t cpu_nominal_ns;   /* CPU segment time before the per-instance factor */
    uint32_t cpu_estimate_ns;  /* ~E^cpu_j used in Eq. 2 */
    uint32_t num_kernels;
    const urg_kernel_desc *kernels;
    uint32_t flags;            /* bit 0 (URG_TASK_FREE): the task ends with cudaFree, a device-wide
                                  barrier (R28); other bits must be 0 */
} urg_task_desc;
enum { URG_TASK_FREE = 1 };

/* A periodic task chain with an end-to-end deadline (Table 2). */
typedef struct {
    int64_t period_ns;         /* > 0 */
    int64_t deadline_ns;       /* > 0 */
    int64_t offset_ns;         /* >= 0, first arrival before jitter */
    uint32_t num_tasks;        /* >= 1 */
    const urg_task_desc *tasks;
    uint32_t cpu_sigma_ppm;    /* per-instance CPU spread, ppm of the mean (Table 2 "+-") */
    uint32_t gpu_sigma_ppm;    /* per-instance GPU spread */
} urg_chain_desc;

/* A workload template shared by every scenario of a batch. */
typedef struct {
    uint32_t num_chains;                  /* 1..32 (one warp lane per chain) */
    const urg_chain_desc *chains;
    uint32_t num_prio;                    /* NUM_PRI stream priorities, 1..8 (6) */
    int64_t launch_ns;                    /* lambda, CPU cost of a launch */
    int64_t launch_akb_ns;                /* extra UrgenGo cost per launch: AKB update */
    int64_t sync_lo_ns, sync_hi_ns;       /* sigma range per sync call; 0 <= lo <= hi < 2^32 - 1 */
    int64_t jitter_ns;                    /* arrival jitter J; must be < every P' */
    const int32_t *inst_quantiles_q16;    /* host, 4096 truncated-normal z quantiles (Q16.16) or NULL */
    const uint32_t *kern_quantiles_q16;   /* host, 4096 per-kernel factor quantiles (Q16.16) or NULL */
    int64_t rt_bin_ns;                    /* response-time histogram bin width (> 0) */
    uint32_t rt_bins;                     /* number of bins B (>= 1; last bin is open-ended) */
    int64_t free_ns;                      /* cudaFree cost on an idle device (Table 5: 188 us);
                                             must be > 0 when any task ends with cudaFree */
    uint32_t cpu_cores;                   /* CPU cores shared by the chains' threads with the policy's
                                             SCHED_FIFO priorities (8; DESIGN.md
                                             R29); 0 = one core per thread, <= 32 */
    uint32_t contention_permille;         /* alpha: a kernel started while U per-mille of the GPU runs
                                             takes d + floor(d * alpha * U / 10^6) (
                                             DESIGN.md R30); 0 = no slow-down */
    uint32_t executors;                   /* URG_EXEC_CHAIN: one thread per chain runs its tasks in turn
                                             (R6).  URG_EXEC_TASK: one executor thread per task
                                             ("each task is executed by a dedicated thread"):
                                             task j+1 of instance i starts when task j publishes it, tasks
                                             of successive instances overlap, and each subscription keeps
                                             the latest message only (depth 1; R32).  Needs
                                             sum(num_tasks) <= 32 (URG_ERANGE) and no CPU predictor
                                             (urg_policy.cpu_ma_window = 0, else URG_EINVAL at simulate) */
    uint32_t num_variants;                /* template variants V >= 1 (0 reads as 1; <= 65536): scenario s
                                             runs on kernel-record set s mod V (SURVEY.md §8(d) cfg 2
                                             "64 templates"; R33).  Set 0 is the chains' own
                                             kernels; the records of every set are read from HBM/L2 */
    const urg_kernel_desc *variant_kernels; /* host, sets 1..V-1: (V-1) x sum(num_kernels) records,
                                             chain-major like the chains' kernels; flags must equal the
                                             chains' kernel flags (URG_EINVAL, locus variant_kernels[v][k]) */
} urg_workload_desc;
enum { URG_EXEC_CHAIN = 0, URG_EXEC_TASK = 1 };

typedef struct urg_workload urg_workload; /* opaque; immutable after create; owns its device copy */

/* Validate d and build the device template (on the current CUDA device).
 * All descriptor pointers are host pointers and are not retained. */
urg_status urg_create_workload(const urg_workload_desc *d, urg_workload **out);
void urg_destroy_workload(urg_workload *w);

/* Policies (§4.4; baselines P:614-615; classical policies of the policy study
 * EDF, SJF, HRRN, lowest chain utilisation first, R27). */
enum { URG_FIFO = 0, URG_STATIC = 1, URG_URGENGO = 2, URG_EDF = 3, URG_SJF = 4, URG_HRRN = 5, URG_LCUF = 6 };
/* UrgenGo mechanisms: stream binding, delayed launching, early exit;
 * URG_F_COLLISIONS counts kernel collisions of urgent kernels (R24) into the
 * aggregate's collision histogram -- a metric only, the schedule is unchanged. */
enum { URG_F_BIND = 1, URG_F_DELAY = 2, URG_F_EARLY_EXIT = 4, URG_F_COLLISIONS = 8 };
/* Launch synchronisation (Fig. fig:launch (a)-(d)). */
enum { URG_SYNC_ASYNC = 0, URG_SYNC_EACH = 1, URG_SYNC_BATCHED = 2, URG_SYNC_OVERLAP = 3 };

typedef struct {
    uint32_t kind;                 /* URG_FIFO / URG_STATIC / URG_URGENGO */
    uint32_t flags;                /* URG_F_* (UrgenGo only) */
    uint32_t sync_mode;            /* URG_SYNC_* */
    int64_t delta_eval_ns;         /* Delta_eval (0.5 ms), > 0 */
    int64_t lax_threshold_ns;      /* L_th = 1/TH_urgent; < 0 disables urgency */
    int64_t sleep_ns;              /* delay-loop sleep (1 ms), > 0 */
    uint32_t util_exempt_permille; /* kernels below this are never delayed (100) */
    uint32_t noise_permille;       /* urgency-estimation noise eps <= 1000, uniform per task instance
                                      (R25); 0 = exact estimates */
    uint32_t cpu_ma_window;        /* CPU-segment moving-average window W <= 64 (R26);
                                      0 = profiled estimates; needs max_tasks*(W+2)*4 B of shared
                                      memory per warp lane (URG_ERANGE if it does not fit) */
} urg_policy;

typedef struct {
    uint64_t seed;                 /* Philox key */
    uint64_t scenario_begin;       /* global index of the first scenario (randomness is keyed by it) */
    uint64_t scenario_count;       /* scenario_begin + scenario_count <= 2^32 */
    int64_t horizon_ns;            /* H: instances arriving before H are admitted (R7) */
    uint32_t fa_num, fa_den;       /* arrival-rate factor f_a = fa_num/fa_den */
    uint32_t fd_num, fd_den;       /* deadline factor f_d */
    uint32_t ftight_permille;      /* f_tight: fraction of chains with halved deadlines */
    uint32_t tight_explicit;       /* 1: use tight_mask instead of the per-scenario draw */
    uint32_t tight_mask;
} urg_batch;

/* Outputs (DEVICE pointers for urg_simulate_batch, HOST for urg_simulate_batch_host).
 * records: [scenario_count][num_chains][8] uint32 per DESIGN.md R22 (total, miss, early,
 *          unfinished, launches, rt_hash, sum_rt_lo, sum_rt_hi), or NULL;
 * agg:     urg_agg_words(w) int64, R23 layout; the kernel ADDS into it (zero it first). */
typedef struct {
    uint32_t *records;
    int64_t *agg;
} urg_outputs;

/* Number of int64 words of the aggregate buffer:
 * num_chains * (5 + rt_bins + 101) + 33 (collision histogram, index = number of colliding
 * tasks, R24) + 2 (launch events, loop steps). */
uint64_t urg_agg_words(const urg_workload *w);

/* Bytes of the packed template urg_create_workload copied host -> device
 * (chains, tasks, kernel records, quantile tables; urg_layout.h). */
uint64_t urg_template_bytes(const urg_workload *w);

/* Simulate scenarios [scenario_begin, scenario_begin + scenario_count) of the
 * workload under policy p (DESIGN.md Model M0) and add their results to o.
 * Asynchronous: enqueued on cuda_stream (a cudaStream_t, NULL = legacy default);
 * calls using the same workload must be ordered on one stream. */
urg_status urg_simulate_batch(const urg_workload *w, const urg_policy *p, const urg_batch *b,
                              const urg_outputs *o, void *cuda_stream);

/* Same with HOST output buffers: allocates device outputs, simulates, copies
 * records and agg back (agg is ADDED into the host buffer).  Synchronous; a device
 * invariant trip of this call is returned as URG_EINTERNAL (as urg_check would). */
urg_status urg_simulate_batch_host(const urg_workload *w, const urg_policy *p, const urg_batch *b,
                                   const urg_outputs *host_o, void *cuda_stream);

/* Synchronise cuda_stream and report a device-side invariant trip recorded by an
 * earlier urg_simulate_batch (URG_EINTERNAL, *scenario_out = offending scenario).
 * The first trip since the last report is kept; reporting clears the device error
 * word, so a later trip on the same workload is reported by a later call.
 * Thread safety: calls on one workload must be ordered (one stream); launches of
 * different workloads from several host threads are safe (the per-kernel attribute
 * set and the launch are serialised inside the library). */
urg_status urg_check(const urg_workload *w, void *cuda_stream, int64_t *scenario_out);

/* TH_urgent calibration ("periodically recording the highest urgency
 * value among all active kernels in AKB ... the 95th percentile"; Q5).
 * Every scenario of b is simulated under p (UrgenGo) with the threshold disabled; every
 * 1 ms of the first min(H, window_ns) the laxity of the most urgent AKB entry is
 * sampled (none when the AKB is empty or that laxity is negative); the samples of all
 * scenarios are pooled and the laxity of their nearest-rank 95th-percentile urgency
 * (rank floor(0.95 m) + 1 in ascending urgency) is L_th = 1/TH_urgent.
 * scratch: DEVICE int64[urg_calibration_words(w, b, window_ns)]; after the call it holds
 *          [count] per-scenario sample counts, then [count][cap] samples in time order.
 * result:  DEVICE int64[2] = {L_th (or -1 with no sample), number of samples m}.
 * Asynchronous on cuda_stream; URG_ERANGE if scratch is too small. */
uint64_t urg_calibration_words(const urg_workload *w, const urg_batch *b, int64_t window_ns);
urg_status urg_calibrate(const urg_workload *w, const urg_policy *p, const urg_batch *b, int64_t window_ns,
                         int64_t *scratch, uint64_t scratch_words, int64_t *result, void *cuda_stream);

/* Eq. 3 from a HOST aggregate buffer: per_chain_out[c] =
 * M_miss/M_total (0 when M_total = 0); overall = mean over chains with M_total > 0. */
urg_status urg_miss_ratios(const urg_workload *w, const int64_t *agg_host, double *per_chain_out,
                           double *overall_out);

/* Thread-local description of the last error (empty string if none). */
const char *urg_last_error(void);

/* ---- debug and test hooks (not part of the simulation path) ---- */

/* Record the event trace of global scenario `scenario` during the following simulate calls of
 * this process into dev_buf (DEVICE int64: [0] = number of rows written, then cap_rows rows of
 * (t, kind, lane, instance, a, b) -- the CPU oracle's trace schema and kind codes
 * "time_ns, seq, kind, chain, instance, detail" with seq = row order per lane).  dev_buf = NULL
 * turns it off.  Only the debug build (liburg_debug.so, compiled with -DURG_DEBUG) writes rows;
 * it also checks the invariants of SPEC.md:171-174 on device (a kernel never starts before it is
 * ready, capacity <= 1000 permille, a kernel retires exactly at its end, every kernel of a
 * finished instance launched and completed once, record counts consistent, no event scheduled
 * in the past, urgent tasks at level 0) and reports a violation through urg_check
 * (URG_EINTERNAL, codes 17-23). */
urg_status urg_debug_set_trace(int64_t *dev_buf, uint64_t cap_rows, uint64_t scenario);

/* 1 in the debug build, 0 in the product build. */
int urg_debug_build(void);

/* Device Philox4x32-10 of n (ctr, key) pairs (DEVICE uint32 [n][4], [n][2], out [n][4]) --
 * the known-answer test of the device RNG copy. */
urg_status urg_debug_philox(const void *d_ctr, const void *d_key, void *d_out, int n, void *cuda_stream);

/* Event-loop counters of the profiling build (liburg_stats.so, -DURG_STATS) since the last call:
 * [single-chain steps, multi-chain steps, Phase C dispatches, 64-bit rebases]; zeros otherwise. */
urg_status urg_debug_stats(const urg_workload *w, uint64_t *out4);

#ifdef __cplusplus
}
#endif

#endif /* URG_H */
