/*
 * oracle/urg_oracle.c -- CPU ORACLE for the batched UrgenGo launch-policy
 * simulation.  TEST INFRASTRUCTURE ONLY: loaded by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * legs -- never by the product path (paper_2509_12207_b200/).
 *
 * Plain, slow, single-threaded C.  It shares no code, header or table with the
 * CUDA path; the only common things are the seeded input records
 * (workloads/) and the written model.  Where the paper
 * defines an operation the code follows it literally and in its order:
 *
 *   - Eq. 2 urgency (§4.2) is evaluated as the literal sums
 *     over the remaining kernels / CPU segments (no suffix-sum caches);
 *   - the Active Kernel Buffer (§4.4.2) is an explicit list
 *     of entries (K, U_K, S_K, C, T_K, UL_C(T_K)) per chain, an entry deleted
 *     once its kernel completed and a covering synchronisation returned;
 *   - each chain's stream (§2, §4.4.3) is an
 *     explicit FIFO queue of launched kernels;
 *   - stream binding ranks the AKB chains with qsort;
 *   - delayed launching scans the other chains' AKB entries;
 *   - batched / overlapped synchronisation follows PAPER.md:496-509 (§4.4.5);
 *   - early chain exit follows PAPER.md:401 (§4.3);
 *   - GPU dispatch sorts the waiting stream heads.
 *
 * Everything the paper leaves open is a DESIGN.md "Model M0" reading (R0-R23);
 * comments name the rule.  All time is int64 nanoseconds, no floating point.
 *
 * Parity pins for every exported function and every scenario draw: tests/test_oracle_*.py
 * (the draws R3-R5 -- factors, tight subset, arrivals, per-instance / per-kernel factors, sync
 * costs -- in test_oracle_draws.py; R15's levels at NUM_PRI > 2 in the W11 fixture and an exact
 * trace replay; R21's same-t continuation in the W10 fixture).
 * Unpinned: the Table 2 C2/C7 rank tie (Q7) -- "parity unpinned".
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_INF INT64_MAX
/* The oracle's own size limit: the rank / dispatch / CPU-job scratch arrays hold 64 entries.  It is
 * not the GPU path's limit (one warp lane per chain: 32, rejected there with URG_ERANGE). */
#define ORC_MAX_CHAINS 64

/* ------------------------------------------------------------------ */
/* Input records (mirrors workloads/spec.py; oracle-private definition) */
/* ------------------------------------------------------------------ */
typedef struct {
    /* workload */
    uint32_t num_chains;
    const int64_t *ch_period, *ch_deadline, *ch_offset;
    const uint32_t *ch_ntasks, *ch_cpu_sigma, *ch_gpu_sigma;
    const uint32_t *t_cpu_nom, *t_cpu_est, *t_nk;   /* all tasks, chain-major */
    const uint32_t *t_flags;                        /* bit 0: the task ends with cudaFree (R28) */
    const uint32_t *k_nom, *k_est;                  /* all kernels, chain-major; num_variants sets */
    const uint16_t *k_util;
    const uint16_t *k_flags;        /* bit 0: the operation is a memcpy on the copy engine (R31) */
    uint32_t num_prio;
    int64_t launch_ns, launch_akb_ns, sync_lo_ns, sync_hi_ns, jitter_ns;
    const int32_t *inst_q16;    /* 4096 z quantiles or NULL */
    const uint32_t *kern_q16;   /* 4096 factor quantiles or NULL */
    int64_t rt_bin_ns;
    uint32_t rt_bins;
    int64_t free_ns;            /* cudaFree cost once the device is idle (Table 5) */
    uint32_t cpu_cores;         /* CPU cores shared by the chains' threads, 0 = one per thread (R29) */
    uint32_t contention_permille; /* alpha: kernel slow-down per unit of co-running utilisation (R30) */
    uint32_t task_exec;         /* 1: one executor thread per task, hand-over by message (R32) */
    uint32_t num_variants;      /* kernel-record sets; scenario s uses set s mod num_variants (R33) */
    /* policy */
    uint32_t kind, flags, sync_mode;
    int64_t delta_eval_ns, lax_threshold_ns, sleep_ns;
    uint32_t util_exempt_permille;
    uint32_t noise_permille;    /* urgency-estimation noise epsilon, per task instance (R25) */
    uint32_t cpu_ma_window;     /* CPU-segment moving-average window W, 0 = profiled estimate (R26) */
    /* batch */
    uint64_t seed, scenario_begin, scenario_count;
    int64_t horizon_ns;
    uint32_t fa_num, fa_den, fd_num, fd_den, ftight_permille, tight_explicit, tight_mask;
} orc_input;

enum { ORC_FIFO = 0, ORC_STATIC = 1, ORC_URGENGO = 2, ORC_EDF = 3, ORC_SJF = 4, ORC_HRRN = 5, ORC_LCUF = 6 };
enum { ORC_BIND = 1, ORC_DELAY = 2, ORC_EARLY_EXIT = 4, ORC_COLLISIONS = 8 };
enum { ORC_ASYNC = 0, ORC_EACH = 1, ORC_BATCHED = 2, ORC_OVERLAP = 3 };
enum { TAG_ARR = 1, TAG_TIGHT = 2, TAG_INST = 3, TAG_KERN = 4, TAG_SYNC = 5, TAG_NOISE = 6 };

/* trace kinds */
enum { TR_STEP = 1, TR_INST_START, TR_TASK_START, TR_EVAL, TR_DELAY, TR_BIND, TR_ENQUEUE,
       TR_DISPATCH, TR_RETIRE, TR_SYNC_CALL, TR_SYNC_RET, TR_FREE_CLOSE, TR_INST_DONE,
       TR_EARLY_EXIT, TR_COLLISION, TR_FREE_CALL, TR_FREE_START, TR_FREE_RET, TR_CPU_RUN, TR_CPU_STOP,
       TR_PUBLISH, TR_TAKE };

#define REC_WORDS 8
#define AGG_COUNTERS 5
#define RATIO_BINS 101
#define COLL_BINS 33      /* kernel-collision histogram by number of colliding tasks (R24) */

/* ------------------------------------------------------------------ */
/* Philox4x32-10 counter-based RNG (Salmon, Moraes, Dror, Shaw, SC'11). */
/* Oracle-private copy; pinned by known-answer vectors in the tests.    */
/* ------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* One 32-bit random word of scenario s (R3-R5):
 * ctr = (s, tag<<24 | c<<16, i, k>>2), key = (seed_lo, seed_hi), word k&3. */
static uint32_t orc_word(uint64_t seed, uint64_t s, uint32_t tag, uint32_t c, uint32_t i, uint32_t k)
{
    uint32_t ctr[4] = {(uint32_t)s, (tag << 24) | (c << 16), i, k >> 2};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t out[4];
    orc_philox4x32_10(ctr, key, out);
    return out[k & 3];
}

/* ------------------------------------------------------------------ */
/* Urgency (Eq. 2), its order key and the "truly urgent" predicate      */
/* ------------------------------------------------------------------ */

/* Eq. 2 denominator, the laxity
 *   L = t_arr + D - sum_{k=n}^{N-1} ~E^gpu_k - sum_{j=m}^{M-1} ~E^cpu_j - t,
 * with n = I~gpu (the launch counter) and m = I~cpu
 * (PAPER.md:335).  UL_C(t) = 1/L is never formed (R9). */
int64_t orc_eq2_laxity(int64_t t_arr, int64_t D, const uint32_t *est_gpu, uint32_t N, uint32_t n,
                       const uint32_t *est_cpu, uint32_t M, uint32_t m, int64_t t)
{
    int64_t rem_gpu = 0, rem_cpu = 0;
    for (uint32_t k = n; k < N; ++k) rem_gpu += est_gpu[k];
    for (uint32_t j = m; j < M; ++j) rem_cpu += est_cpu[j];
    return t_arr + D - rem_gpu - rem_cpu - t;
}

/* An int64 whose order is the order of UL = 1/L (R9):
 * L = 0 -> +max (saturation), L > 0 -> 2^62 - L, L < 0 -> -2^62 - L. */
int64_t orc_urgency_key(int64_t L)
{
    if (L == 0) return INT64_MAX;
    if (L > 0) return ((int64_t)1 << 62) - L;
    return -((int64_t)1 << 62) - L;
}

/* UL >= TH_urgent  <=>  0 <= L <= L_th  (R10) */
int orc_is_urgent(int64_t L, int64_t L_th) { return L >= 0 && L <= L_th; }

/* ------------------------------------------------------------------ */
/* Ranking and stream-level normalisation     */
/* ------------------------------------------------------------------ */
typedef struct { int64_t key; uint32_t chain; } orc_rank_item;

static int orc_rank_cmp(const void *a, const void *b)
{
    const orc_rank_item *x = a, *y = b;
    if (x->key != y->key) return x->key > y->key ? -1 : 1;   /* more urgent first */
    return x->chain < y->chain ? -1 : (x->chain > y->chain);  /* ties: smaller chain id */
}

/* rank_out[i] = 1-based rank of item i when sorted by urgency key descending. */
void orc_rank(const int64_t *keys, const uint32_t *chains, uint32_t n, uint32_t *rank_out)
{
    orc_rank_item *it = malloc(sizeof(orc_rank_item) * (n ? n : 1));
    for (uint32_t i = 0; i < n; ++i) { it[i].key = keys[i]; it[i].chain = chains[i]; }
    qsort(it, n, sizeof(orc_rank_item), orc_rank_cmp);
    for (uint32_t i = 0; i < n; ++i)
        for (uint32_t r = 0; r < n; ++r)
            if (it[r].chain == chains[i] && it[r].key == keys[i]) { rank_out[i] = r + 1; break; }
    free(it);
}

/* Rank r of n_r normalised onto stream levels 1..NUM_PRI-1 (PAPER.md:466,
 * "normalize these rankings to the range (1, NUM_PRI-1)"); level 0 is reserved
 * for truly urgent tasks.  Floor linear map, middle level for a single
 * member (R15; SPEC.md:402-404 examples). */
uint32_t orc_normalise_level(uint32_t r, uint32_t n_r, uint32_t num_prio)
{
    if (num_prio <= 2) return num_prio - 1;
    if (n_r <= 1) return 1 + (num_prio - 2) / 2;
    return 1 + (uint32_t)(((uint64_t)(r - 1) * (num_prio - 2)) / (n_r - 1));
}

/* Batch closing rule of batched launching: kernels join the
 * batch while the running sum of their estimates stays below Delta_eval; the
 * kernel whose estimate brings the sum to >= Delta_eval is the last member
 * (R17 / Q9).  Returns 1 when the batch closes after this kernel. */
int orc_batch_add(int64_t *acc, uint32_t est, int64_t delta_eval)
{
    *acc += est;
    if (*acc >= delta_eval) { *acc = 0; return 1; }
    return 0;
}

void orc_plan_batches(const uint32_t *est, uint32_t n, int64_t delta_eval, uint8_t *close_after)
{
    int64_t acc = 0;
    for (uint32_t k = 0; k < n; ++k) close_after[k] = (uint8_t)orc_batch_add(&acc, est[k], delta_eval);
}

/* Eq. 3: mean over chains of M_miss/M_total; chains with
 * M_total = 0 are left out (R22). */
double orc_overall_miss_ratio(const uint64_t *miss, const uint64_t *total, uint32_t n)
{
    double s = 0.0;
    uint32_t used = 0;
    for (uint32_t i = 0; i < n; ++i)
        if (total[i]) { s += (double)miss[i] / (double)total[i]; ++used; }
    return used ? s / used : 0.0;
}

/* ------------------------------------------------------------------ */
/* Simulation state                                                    */
/* ------------------------------------------------------------------ */
typedef struct {            /* one AKB entry */
    uint32_t K;             /* kernel index within the chain instance */
    uint32_t U;             /* profiled utilisation (per-mille) */
    uint32_t S;             /* stream = priority level bound */
    uint32_t C;             /* chain id */
    int64_t T;              /* last evaluation time T_K */
    int64_t L;              /* last-evaluated laxity (UL_C(T_K) = 1/L) */
} orc_akb_entry;

typedef struct { uint32_t K; int64_t t_enq; } orc_stream_entry;

enum { PC_ARRIVE = 0, PC_CPU_DONE, PC_ATTEMPT, PC_ENQUEUE, PC_SYNC_WAIT, PC_SYNC_RET, PC_FREE_WAIT, PC_FREE_RET,
       PC_WAIT_MSG, PC_DONE };

typedef struct {
    /* static per scenario */
    uint32_t chain;                 /* the chain this thread serves (randomness, records) */
    uint32_t stage, stage_end;      /* tasks [stage, stage_end) of every instance it runs: the whole
                                       chain (R6), or one task under per-task executors (R32) */
    uint32_t k0;                    /* kernels of the chain's tasks before `stage` */
    int64_t Pp, Dp;                 /* P', D' (R3) */
    uint32_t static_level;
    uint32_t N, M;                  /* kernels and tasks (= CPU segments) per instance */
    uint32_t kbase, tbase;          /* offsets into the flattened kernel / task arrays */
    /* CPU thread of the chain (R6) */
    int pc;
    int64_t cpu_next;
    uint32_t inst;                  /* current (or next) instance index */
    int64_t t_arr;
    uint32_t Fg, Fc;                /* per-instance factors, Q16.16 */
    uint32_t task;                  /* current task tau */
    uint32_t launched;              /* I~gpu: kernels launched in this instance */
    uint32_t cpu_idx;               /* I~cpu */
    uint32_t done;                  /* kernels of this instance completed on the GPU */
    uint32_t level;                 /* stream level of the current task */
    int64_t acc;                    /* estimated time of the open batch */
    uint32_t batch_start;           /* first kernel of the open batch */
    uint32_t sync_target, sync_ord;
    int64_t sync_cost;
    /* CPU-segment predictor (R26): measured durations per task, newest last */
    uint32_t *cpu_hist;             /* [M][W] ring of measurements */
    uint32_t *cpu_hist_n;           /* [M] measurements recorded so far */
    uint32_t *cpu_pred;             /* [M] ~E^cpu_j used by the current instance */
    /* AKB instance of the chain */
    orc_akb_entry *akb;
    uint32_t akb_n;
    int64_t T_last, L_last;
    /* stream */
    orc_stream_entry *q;
    uint32_t q_head, q_tail;        /* entries [q_head, q_tail) */
    int head_running;
    int64_t head_ready, head_end;
    int64_t free_req;               /* time of this chain's pending cudaFree request (R28) */
    /* CPU job of the chain's thread under a limited core count (R29) */
    int job, job_run;               /* a job exists / it holds a core */
    int64_t job_rem, job_ready, run_start;
    int64_t cpu_prio;               /* SCHED_FIFO priority key: higher runs first */
    /* per-task executors (R32): the subscription's latest undelivered / delivered message
     * (instance index + 1, 0 = none) and, on the chain's last stage, the next instance to record */
    uint32_t msg_pend, msg;
    uint32_t expect;
    /* results */
    uint32_t total, miss, early, unfin, launches, hash;
    uint64_t sum_rt;
} orc_lane;

typedef struct {
    const orc_input *in;
    uint64_t s;
    uint32_t C;                     /* chains (records, aggregates) */
    uint32_t nL;                    /* threads: C, or one per task under per-task executors (R32) */
    orc_lane *lane;
    uint32_t gpu_used;              /* sum of running utilisations, <= 1000 */
    int64_t H, H_stop;
    int64_t *snap_L;                /* AKB read view at the start of Phase B */
    uint32_t *snap_n;
    uint32_t *snap_level;           /* stream level of each chain's current task, same snapshot */
    uint8_t *snap_busy;             /* the chain's stream holds a kernel (waiting or running) */
    int64_t *snap_tarr;             /* arrival time of the chain's current instance, same snapshot */
    int64_t *snap_R;                /* its remaining estimated work (kernels + CPU segments, Eq. 2 sums) */
    int64_t *akb_L_view;            /* scratch */
    int64_t *trace; int64_t trace_cap; int64_t trace_len;
    int64_t *agg;
    int64_t steps, launches, t_prev;
    int cpu_dirty, rerank;          /* R29: the runnable set / the priorities changed in this step */
    int copy_busy;                  /* R31: the copy engine runs a memcpy */
    /* calibration sampling */
    int64_t cal_next, cal_end;
    int64_t *cal_L; int64_t cal_n, cal_cap;
} orc_sim;

static void tr(orc_sim *S, int64_t t, int64_t kind, int64_t c, int64_t i, int64_t a, int64_t b)
{
    if (!S->trace || S->trace_len >= S->trace_cap) return;
    int64_t *r = S->trace + 6 * S->trace_len++;
    r[0] = t; r[1] = kind; r[2] = c; r[3] = i; r[4] = a; r[5] = b;
}

static uint32_t hash_fold(uint32_t h, uint32_t x) { return (h ^ x) * 16777619u; }

/* ---- scenario randomness (R3-R5) ---- */
static int64_t arrival(const orc_sim *S, uint32_t c, uint32_t i)
{
    const orc_input *in = S->in;
    const uint32_t ch = S->lane[c].chain;
    int64_t jit = 0;
    if (in->jitter_ns > 0)
        jit = (int64_t)(orc_word(in->seed, S->s, TAG_ARR, ch, i, 0) % (uint64_t)(in->jitter_ns + 1));
    return in->ch_offset[ch] + (int64_t)i * S->lane[c].Pp + jit;
}

static uint32_t inst_factor(const orc_sim *S, uint32_t ch, uint32_t i, uint32_t which, uint32_t sigma_ppm)
{
    const orc_input *in = S->in;
    if (!in->inst_q16) return 65536u;
    int64_t z = in->inst_q16[orc_word(in->seed, S->s, TAG_INST, ch, i, which) >> 20];
    int64_t F = 65536 + (z * (int64_t)sigma_ppm) / 1000000;   /* C division truncates toward 0 */
    if (F < 6554) F = 6554;                                    /* factor floor 0.1 (R4) */
    return (uint32_t)F;
}

static int64_t kernel_duration(const orc_sim *S, uint32_t c, uint32_t i, uint32_t k)
{
    const orc_input *in = S->in;
    const orc_lane *L = &S->lane[c];
    uint64_t G = 65536u;
    if (in->kern_q16) G = in->kern_q16[orc_word(in->seed, S->s, TAG_KERN, L->chain, i, k) >> 20];
    uint64_t d = (((uint64_t)in->k_nom[L->kbase + k] * L->Fg) >> 16) * G >> 16;
    if (d < 1) d = 1;
    if (d > 0xFFFFFFFFull) d = 0xFFFFFFFFull;
    return (int64_t)d;
}

static int64_t cpu_duration(const orc_sim *S, uint32_t c)
{
    const orc_lane *L = &S->lane[c];
    return (int64_t)(((uint64_t)S->in->t_cpu_nom[L->tbase + L->task] * L->Fc) >> 16);
}

static int64_t sync_cost(const orc_sim *S, uint32_t c, uint32_t i, uint32_t ord)
{
    const orc_input *in = S->in;
    if (in->sync_hi_ns <= in->sync_lo_ns) return in->sync_lo_ns;
    uint64_t span = (uint64_t)(in->sync_hi_ns - in->sync_lo_ns + 1);
    return in->sync_lo_ns + (int64_t)(orc_word(in->seed, S->s, TAG_SYNC, S->lane[c].chain, i, ord) % span);
}

/* ---- urgency evaluation trigger (R8): Eq. 2 + AKB refresh ---- */
/* Urgency-estimation noise ("noise to the estimated execution times
 * used to calculate task urgency ... uniformly sampled for each task instance";
 * DESIGN.md R25): the remaining estimated work of Eq. 2 during task tau of instance i
 * is scaled by (1000 + n)/1000, n uniform in [-eps, eps] per-mille, floor division. */
static int64_t noisy_laxity(const orc_sim *S, uint32_t c, int64_t t_arr, int64_t D, int64_t t, int64_t lax)
{
    const orc_input *in = S->in;
    const orc_lane *L = &S->lane[c];
    if (in->noise_permille == 0) return lax;
    uint32_t w = orc_word(in->seed, S->s, TAG_NOISE, L->chain, L->inst, L->task);
    int64_t n = (int64_t)(w % (2 * in->noise_permille + 1)) - (int64_t)in->noise_permille;
    int64_t remaining = t_arr + D - t - lax;           /* sum of the remaining estimates (>= 0) */
    return t_arr + D - (remaining * (1000 + n)) / 1000 - t;
}

static int64_t evaluate(orc_sim *S, uint32_t c, int64_t t)
{
    orc_lane *L = &S->lane[c];
    const orc_input *in = S->in;
    int64_t lax = orc_eq2_laxity(L->t_arr, L->Dp, in->k_est + L->kbase, L->N, L->launched,
                                 L->cpu_pred, L->M, L->cpu_idx, t);
    lax = noisy_laxity(S, c, L->t_arr, L->Dp, t, lax);
    L->T_last = t; L->L_last = lax;
    for (uint32_t e = 0; e < L->akb_n; ++e) { L->akb[e].T = t; L->akb[e].L = lax; }
    tr(S, t, TR_EVAL, c, L->inst, lax, L->launched);
    return lax;
}

static int urgengo(const orc_sim *S) { return S->in->kind == ORC_URGENGO; }
/* classical policies of the paper's policy study (R27) */
static int classical(const orc_sim *S) { return S->in->kind >= ORC_EDF; }

/* Remaining estimated work of chain c's current instance: the two sums of Eq. 2. */
static int64_t remaining_work(const orc_sim *S, uint32_t c)
{
    const orc_lane *L = &S->lane[c];
    int64_t r = 0;
    for (uint32_t k = L->launched; k < L->N; ++k) r += S->in->k_est[L->kbase + k];
    for (uint32_t j = L->cpu_idx; j < L->M; ++j) r += L->cpu_pred[j];
    return r;
}

/* "a ranks before b" under the classical policy (R27), ties by smaller chain id:
 * EDF absolute deadline t_arr + D' ascending; SJF remaining work R ascending; HRRN response
 * ratio (t - t_arr + R) / R descending (R = 0: infinite); LCUF chain utilisation
 * sum(~E^gpu) / P' ascending.  Ratios compare by exact 128-bit cross-multiplication. */
typedef struct { uint32_t chain; int64_t tarr, D, R, G, Pp; } orc_cl_item;

static int orc_cl_before(const orc_sim *S, const orc_cl_item *a, const orc_cl_item *b, int64_t t)
{
    switch (S->in->kind) {
    case ORC_EDF:
        if (a->tarr + a->D != b->tarr + b->D) return a->tarr + a->D < b->tarr + b->D;
        break;
    case ORC_SJF:
        if (a->R != b->R) return a->R < b->R;
        break;
    case ORC_HRRN: {
        if (a->R == 0 || b->R == 0) {
            if (a->R == 0 && b->R != 0) return 1;
            if (b->R == 0 && a->R != 0) return 0;
            break;
        }
        __int128 x = (__int128)(t - a->tarr + a->R) * b->R, y = (__int128)(t - b->tarr + b->R) * a->R;
        if (x != y) return x > y;
        break;
    }
    case ORC_LCUF: {
        __int128 x = (__int128)a->G * b->Pp, y = (__int128)b->G * a->Pp;
        if (x != y) return x < y;
        break;
    }
    }
    return a->chain < b->chain;
}
static int flag(const orc_sim *S, uint32_t f) { return urgengo(S) && (S->in->flags & f); }

/* Delayed launching (R14): delay kernel K iff its
 * utilisation is not exempt, the launching chain itself is not truly urgent,
 * and some other chain's active kernel has a truly urgent last evaluation. */
static int should_delay(const orc_sim *S, uint32_t c, uint32_t util, int64_t own_L)
{
    const orc_input *in = S->in;
    if (util < in->util_exempt_permille) return 0;
    if (orc_is_urgent(own_L, in->lax_threshold_ns)) return 0;
    for (uint32_t o = 0; o < S->nL; ++o) {
        if (o == c) continue;
        for (uint32_t e = 0; e < S->snap_n[o]; ++e)   /* every active kernel of chain o */
            if (orc_is_urgent(S->snap_L[o], in->lax_threshold_ns)) return 1;
    }
    return 0;
}

/* Task-level stream binding with reservation (R15). */
/* Rank (1-based) of item `self` among n items under classical policy `kind` at time t
 * (test export of orc_cl_before: the pure ordering of DESIGN.md R27). */
uint32_t orc_classical_rank(uint32_t kind, const int64_t *tarr, const int64_t *D, const int64_t *R, const int64_t *G,
                            const int64_t *Pp, uint32_t n, uint32_t self, int64_t t)
{
    orc_input in;
    memset(&in, 0, sizeof in);
    in.kind = kind;
    orc_sim S;
    memset(&S, 0, sizeof S);
    S.in = &in;
    orc_cl_item it[ORC_MAX_CHAINS];
    if (n > ORC_MAX_CHAINS) n = ORC_MAX_CHAINS;
    if (self >= n) return 0;
    for (uint32_t i = 0; i < n; ++i) {
        it[i].chain = i; it[i].tarr = tarr[i]; it[i].D = D[i]; it[i].R = R[i]; it[i].G = G[i]; it[i].Pp = Pp[i];
    }
    uint32_t r = 1;
    for (uint32_t i = 0; i < n; ++i)
        if (i != self && orc_cl_before(&S, &it[i], &it[self], t)) ++r;
    return r;
}

static uint32_t bind_level(orc_sim *S, uint32_t c, int64_t own_L, int64_t t)
{
    const orc_input *in = S->in;
    if (in->kind == ORC_FIFO) return in->num_prio - 1;
    if (in->kind == ORC_STATIC) return S->lane[c].static_level;
    if (classical(S)) {
        /* rank among the chain itself and every other chain with active kernels (read view),
         * normalised like UrgenGo's non-urgent ranks (R15) */
        orc_cl_item it[ORC_MAX_CHAINS];
        uint32_t n = 0;
        for (uint32_t o = 0; o < S->nL; ++o) {
            if (o != c && S->snap_n[o] == 0) continue;
            orc_cl_item *x = &it[n++];
            const orc_lane *L = &S->lane[o];
            x->chain = o; x->D = L->Dp; x->Pp = L->Pp;
            x->G = 0;
            for (uint32_t k = 0; k < L->N; ++k) x->G += in->k_est[L->kbase + k];
            if (o == c) { x->tarr = L->t_arr; x->R = remaining_work(S, c); }   /* own, current */
            else { x->tarr = S->snap_tarr[o]; x->R = S->snap_R[o]; }
        }
        uint32_t r = 1;
        const orc_cl_item *self = 0;
        for (uint32_t i = 0; i < n; ++i) if (it[i].chain == c) self = &it[i];
        for (uint32_t i = 0; i < n; ++i)
            if (it[i].chain != c && orc_cl_before(S, &it[i], self, t)) ++r;
        return orc_normalise_level(r, n, in->num_prio);
    }
    if (!(in->flags & ORC_BIND)) return in->num_prio - 1;
    if (orc_is_urgent(own_L, in->lax_threshold_ns)) return 0;
    int64_t keys[ORC_MAX_CHAINS]; uint32_t chains[ORC_MAX_CHAINS], ranks[ORC_MAX_CHAINS], n = 0;
    keys[n] = orc_urgency_key(own_L); chains[n] = c; ++n;
    for (uint32_t o = 0; o < S->nL; ++o)
        if (o != c && S->snap_n[o] > 0) { keys[n] = orc_urgency_key(S->snap_L[o]); chains[n] = o; ++n; }
    orc_rank(keys, chains, n, ranks);
    return orc_normalise_level(ranks[0], n, in->num_prio);
}

static void record_outcome(orc_sim *S, uint32_t c, int64_t t, int early)
{
    orc_lane *L = &S->lane[c];
    const orc_input *in = S->in;
    if (early) {
        L->early++; L->miss++;
        L->hash = hash_fold(hash_fold(L->hash, 0xFFFFFFFFu), 0xFFFFFFFFu);
        tr(S, t, TR_EARLY_EXIT, c, L->inst, 0, 0);
        return;
    }
    int64_t rt = t - L->t_arr;                  /* response time (R18) */
    int late = rt > L->Dp;
    if (late) L->miss++;
    L->sum_rt += (uint64_t)rt;
    L->hash = hash_fold(hash_fold(L->hash, (uint32_t)rt), (uint32_t)((uint64_t)rt >> 32));
    int64_t bin = rt / in->rt_bin_ns;
    if (bin > (int64_t)in->rt_bins - 1) bin = in->rt_bins - 1;
    S->agg[(int64_t)L->chain * (AGG_COUNTERS + in->rt_bins + RATIO_BINS) + AGG_COUNTERS + bin] += 1;
    tr(S, t, TR_INST_DONE, c, L->inst, rt, late);
}

/* Per-task executors (R32; "each task is executed by a dedicated
 * thread"): the thread of stage j > 0 takes the message naming instance i.  On the chain's
 * last stage, instances the message sequence skipped -- exited early at an earlier stage, or
 * overwritten in a full subscription queue of depth 1 -- are recorded now, in order, as
 * misses (the early-exit marker in the hash). */
static void take_message(orc_sim *S, uint32_t c, int64_t t)
{
    orc_lane *L = &S->lane[c];
    uint32_t i = L->msg - 1;
    L->msg = 0;
    if (L->stage_end == L->M)
        for (; L->expect < i; ++L->expect) {
            L->miss++;
            L->hash = hash_fold(hash_fold(L->hash, 0xFFFFFFFFu), 0xFFFFFFFFu);
        }
    L->inst = i;
    L->t_arr = arrival(S, c, i);
    L->pc = PC_ARRIVE; L->cpu_next = t;
    tr(S, t, TR_TAKE, c, i, 0, 0);
}

/* Start of the instance L->inst at time t (frame arrival, or the end of the
 * previous instance when the chain ran late -- DESIGN.md R6). */
static void start_instance(orc_sim *S, uint32_t c, int64_t t)
{
    orc_lane *L = &S->lane[c];
    if (!S->in->task_exec) L->total++;
    L->Fg = inst_factor(S, L->chain, L->inst, 0, S->in->ch_gpu_sigma[L->chain]);
    L->Fc = inst_factor(S, L->chain, L->inst, 1, S->in->ch_cpu_sigma[L->chain]);
    /* the thread's first task of the instance; I~gpu / I~cpu count over the whole instance */
    L->task = L->stage; L->launched = L->k0; L->cpu_idx = L->stage; L->done = L->k0;
    L->sync_ord = L->stage << 16;               /* per-task executors: sync draws keyed per task (R32) */
    L->q_head = L->q_tail = 0;
    /* ~E^cpu_j for this instance ("moving averages across recent instances";
     * DESIGN.md R26): mean of the last min(W, h_j) measured durations of task j, floor;
     * the profiled estimate while task j has no measurement or W = 0 */
    const orc_input *in = S->in;
    for (uint32_t j = 0; j < L->M; ++j) {
        uint32_t W = in->cpu_ma_window, h = L->cpu_hist_n[j];
        if (W == 0 || h == 0) { L->cpu_pred[j] = in->t_cpu_est[L->tbase + j]; continue; }
        uint32_t k = h < W ? h : W;
        uint64_t sum = 0;
        for (uint32_t q = 0; q < k; ++q) sum += L->cpu_hist[j * W + (h - 1 - q) % W];
        L->cpu_pred[j] = (uint32_t)(sum / k);
    }
    tr(S, t, TR_INST_START, c, L->inst, L->t_arr, 0);
}

/* the chain moves on to instance inst+1 at time t; returns 1 if it starts now.  A per-task
 * executor of stage j > 0 takes the delivered message instead, or waits for one (R32). */
static int next_instance(orc_sim *S, uint32_t c, int64_t t)
{
    orc_lane *L = &S->lane[c];
    if (L->stage > 0) {
        if (L->msg) { take_message(S, c, t); return 1; }
        L->pc = PC_WAIT_MSG; L->cpu_next = ORC_INF;
        return 0;
    }
    L->inst++;
    L->t_arr = arrival(S, c, L->inst);
    if (L->t_arr >= S->H) { L->pc = PC_DONE; L->cpu_next = ORC_INF; return 0; }   /* not admitted (R7) */
    if (L->t_arr > t) { L->pc = PC_ARRIVE; L->cpu_next = L->t_arr; return 0; }
    L->pc = PC_ARRIVE; L->cpu_next = t;
    return 1;
}

static void cpu_busy(orc_sim *S, uint32_t c, int64_t t, int64_t d);

static void issue_sync(orc_sim *S, uint32_t c, int64_t t, uint32_t target)
{
    orc_lane *L = &S->lane[c];
    L->sync_target = target;
    L->sync_cost = sync_cost(S, c, L->inst, L->sync_ord++);
    tr(S, t, TR_SYNC_CALL, c, L->inst, target, L->sync_cost);
    if (L->done >= target) { L->pc = PC_SYNC_RET; cpu_busy(S, c, t, L->sync_cost); }
    else { L->pc = PC_SYNC_WAIT; L->cpu_next = ORC_INF; }
}

static uint32_t task_first_kernel(const orc_sim *S, uint32_t c)
{
    const orc_lane *L = &S->lane[c];
    uint32_t k = 0;
    for (uint32_t j = 0; j < L->task; ++j) k += S->in->t_nk[L->tbase + j];
    return k;
}

/* Kernel collisions of an urgent kernel ("priority collision" /
 * "inverted binding", "kernel collisions for urgent kernels";
 * DESIGN.md R24): when chain c enqueues a kernel while its last evaluation is
 * truly urgent, every other chain whose stream holds a kernel and whose task is
 * bound to the same or a higher priority (level <= c's) while being less urgent
 * collides with it.  One event per such enqueue, counted in the histogram bin
 * of the number of colliding tasks (c and its colliders). */
static void count_collision(orc_sim *S, uint32_t c, int64_t t)
{
    orc_lane *L = &S->lane[c];
    const orc_input *in = S->in;
    if (!orc_is_urgent(L->L_last, in->lax_threshold_ns)) return;
    int64_t own = orc_urgency_key(L->L_last);
    uint32_t k = 0;
    for (uint32_t o = 0; o < S->nL; ++o) {
        if (o == c || !S->snap_busy[o]) continue;
        if (S->snap_level[o] <= L->level && orc_urgency_key(S->snap_L[o]) < own) ++k;
    }
    if (k == 0) return;
    uint32_t card = k + 1;
    if (card > COLL_BINS - 1) card = COLL_BINS - 1;
    S->agg[(int64_t)S->C * (AGG_COUNTERS + in->rt_bins + RATIO_BINS) + card] += 1;
    tr(S, t, TR_COLLISION, c, L->inst, card, L->level);
}

/* The chain's thread is busy for d ns from t -- a CPU segment, a launch call or a sync
 * call's cost.  With one core per thread (cpu_cores = 0) it simply runs; with cpu_cores
 * cores it becomes a CPU job that runs when the scheduler gives it a core (R29). */
static void cpu_busy(orc_sim *S, uint32_t c, int64_t t, int64_t d)
{
    orc_lane *L = &S->lane[c];
    if (S->in->cpu_cores == 0 || d == 0) { L->cpu_next = t + d; return; }
    L->job = 1; L->job_run = 0; L->job_rem = d; L->job_ready = t; L->cpu_next = ORC_INF;
    S->cpu_dirty = 1;
}

/* Chain c's urgency laxity at t without refreshing its AKB (the CPU re-rank of R29). */
static int64_t current_laxity(const orc_sim *S, uint32_t c, int64_t t)
{
    const orc_lane *L = &S->lane[c];
    int64_t lax = orc_eq2_laxity(L->t_arr, L->Dp, S->in->k_est + L->kbase, L->N, L->launched,
                                 L->cpu_pred, L->M, L->cpu_idx, t);
    return noisy_laxity(S, c, L->t_arr, L->Dp, t, lax);
}

/* One CPU step of chain c at time t (R21 Phase B): the thread runs
 * its program until it must wait for time to pass or for the GPU. */
static void lane_step(orc_sim *S, uint32_t c, int64_t t)
{
    orc_lane *L = &S->lane[c];
    const orc_input *in = S->in;
    for (;;) {
        switch (L->pc) {
        case PC_ARRIVE: {
            start_instance(S, c, t);
            goto task_start;
        }
        task_start: {
            /* a new CPU segment starts: evaluate, early exit */
            tr(S, t, TR_TASK_START, c, L->inst, L->task, 0);
            if (urgengo(S)) {
                int64_t lax = evaluate(S, c, t);
                if (flag(S, ORC_EARLY_EXIT) && lax < 0) {
                    L->akb_n = 0;                          /* purge the chain's AKB entries */
                    if (L->stage_end == L->M) { record_outcome(S, c, t, 1); L->expect = L->inst + 1; }
                    else { L->early++; tr(S, t, TR_EARLY_EXIT, c, L->inst, 0, 0); }   /* no message (R32) */
                    if (next_instance(S, c, t)) continue;
                    return;
                }
            }
            int64_t e = cpu_duration(S, c);
            if (in->cpu_ma_window) {                     /* measured segment time (clock_gettime) */
                uint32_t W = in->cpu_ma_window;
                L->cpu_hist[L->task * W + L->cpu_hist_n[L->task] % W] = (uint32_t)e;
                L->cpu_hist_n[L->task]++;
            }
            if (urgengo(S)) S->rerank = 1;                  /* a CPU segment starts: re-rank */
            L->pc = PC_CPU_DONE; cpu_busy(S, c, t, e);
            if (e > 0) return;
            continue;
        }
        case PC_CPU_DONE:
        case PC_ATTEMPT: {
            /* launch attempt for kernel n = L->launched */
            uint32_t n = L->launched;
            int64_t lax = 0;
            if (urgengo(S)) lax = evaluate(S, c, t);
            if (flag(S, ORC_DELAY) && should_delay(S, c, in->k_util[L->kbase + n], lax)) {
                tr(S, t, TR_DELAY, c, L->inst, n, 0);
                L->pc = PC_ATTEMPT; L->cpu_next = t + in->sleep_ns;
                return;
            }
            if (n == task_first_kernel(S, c)) {          /* first kernel of the task: bind */
                L->level = bind_level(S, c, lax, t);
                tr(S, t, TR_BIND, c, L->inst, L->level, n);
            }
            int64_t busy = in->launch_ns + (urgengo(S) ? in->launch_akb_ns : 0);
            L->pc = PC_ENQUEUE; cpu_busy(S, c, t, busy);
            if (busy > 0) return;
            continue;
        }
        case PC_ENQUEUE: {
            uint32_t n = L->launched;
            uint32_t first = task_first_kernel(S, c);
            uint32_t end = first + in->t_nk[L->tbase + L->task];
            /* the kernel reaches its stream (R16) */
            if (L->q_head == L->q_tail) { L->head_running = 0; L->head_ready = t; }
            L->q[L->q_tail].K = n; L->q[L->q_tail].t_enq = t; L->q_tail++;
            L->launched++; L->launches++; S->launches++;
            if (urgengo(S) || classical(S)) {            /* updateAKB: a new active kernel */
                orc_akb_entry *a = &L->akb[L->akb_n++];
                a->K = n; a->U = in->k_util[L->kbase + n]; a->S = L->level; a->C = c;
                a->T = L->T_last; a->L = L->L_last;
            }
            tr(S, t, TR_ENQUEUE, c, L->inst, n, L->level);
            if (flag(S, ORC_COLLISIONS)) count_collision(S, c, t);
            int last = (L->launched == end);
            if (last) L->cpu_idx++;
            uint32_t est = in->k_est[L->kbase + n];
            if (n == first) { L->acc = 0; L->batch_start = first; }
            int sync = 0;
            uint32_t target = 0;
            switch (in->sync_mode) {
            case ORC_ASYNC:
                if (last) { sync = 1; target = L->launched; }
                break;
            case ORC_EACH:
                sync = 1; target = L->launched;
                break;
            case ORC_BATCHED: {
                int closes = orc_batch_add(&L->acc, est, in->delta_eval_ns);
                if (closes || last) { L->acc = 0; sync = 1; target = L->launched; }
                break;
            }
            case ORC_OVERLAP: {
                int closes = orc_batch_add(&L->acc, est, in->delta_eval_ns);
                if (last) { L->acc = 0; sync = 1; target = L->launched; }
                else if (closes) {
                    uint32_t prev_batch_end = L->batch_start;   /* wait for the previous batch */
                    L->batch_start = L->launched;
                    if (prev_batch_end == first) {             /* the task's first close: no sync */
                        tr(S, t, TR_FREE_CLOSE, c, L->inst, L->launched, 0);
                        if (urgengo(S)) evaluate(S, c, t);
                    } else { sync = 1; target = prev_batch_end; }
                }
                break;
            }
            }
            if (sync) {
                issue_sync(S, c, t, target);
                /* a wait already satisfied that costs 0 returns at this same t: the step goes on (R21) */
                if (L->pc == PC_SYNC_RET && L->cpu_next == t) continue;
                return;
            }
            L->pc = PC_ATTEMPT;                          /* next kernel, same time */
            continue;
        }
        case PC_SYNC_RET: {
            /* the synchronisation returned: covered kernels leave the AKB */
            uint32_t keep = 0;
            for (uint32_t e = 0; e < L->akb_n; ++e)
                if (L->akb[e].K >= L->sync_target) L->akb[keep++] = L->akb[e];
            L->akb_n = keep;
            tr(S, t, TR_SYNC_RET, c, L->inst, L->sync_target, 0);
            if (urgengo(S)) evaluate(S, c, t);            /* periodic evaluation */
            uint32_t end = task_first_kernel(S, c) + in->t_nk[L->tbase + L->task];
            if (L->launched < end) { L->pc = PC_ATTEMPT; continue; }
            if (in->t_flags && (in->t_flags[L->tbase + L->task] & 1u)) {
                /* the task ends with cudaFree: a device-wide barrier request (R28) */
                L->pc = PC_FREE_WAIT; L->cpu_next = ORC_INF; L->free_req = t;
                tr(S, t, TR_FREE_CALL, c, L->inst, L->task, 0);
                return;
            }
            goto task_done;
        }
        case PC_FREE_RET: {
            tr(S, t, TR_FREE_RET, c, L->inst, L->task, 0);
            goto task_done;
        }
        case PC_WAIT_MSG: {                              /* a message was delivered (R32) */
            take_message(S, c, t);
            continue;
        }
        task_done: {
            L->task++;
            if (L->task < L->stage_end) goto task_start;
            if (L->stage_end < L->M) {
                /* per-task executors: publish to the next task's subscription, depth 1 -- an
                 * undelivered older message is replaced (R32) */
                S->lane[c + 1].msg_pend = L->inst + 1;
                tr(S, t, TR_PUBLISH, c, L->inst, 0, 0);
            } else {
                record_outcome(S, c, t, 0);              /* instance complete (R18) */
                L->expect = L->inst + 1;
            }
            if (next_instance(S, c, t)) continue;
            return;
        }
        default:
            return;
        }
    }
}

/* Phase C: GPU dispatch of waiting stream heads (R20). */
typedef struct { uint32_t level; int64_t ready; uint32_t chain; } orc_cand;

static int orc_cand_cmp(const void *a, const void *b)
{
    const orc_cand *x = a, *y = b;
    if (x->level != y->level) return x->level < y->level ? -1 : 1;
    if (x->ready != y->ready) return x->ready < y->ready ? -1 : 1;
    return x->chain < y->chain ? -1 : (x->chain > y->chain);
}

/* cudaFree device barriers ("cudaFree calls introduce global
 * synchronization"; R28): requests queue in (request time,
 * chain) order; while any is queued or being served the GPU starts no kernel; the queue
 * head is served once no kernel runs, costing free_ns, after which its chain resumes.
 * Returns 1 if a barrier is queued or in service (no dispatch at t). */
static int barrier(orc_sim *S, int64_t t)
{
    int queued = 0, serving = 0, running = 0;
    int32_t head = -1;
    for (uint32_t c = 0; c < S->nL; ++c) {
        const orc_lane *L = &S->lane[c];
        if (L->pc == PC_FREE_RET) serving = 1;
        if (L->pc == PC_FREE_WAIT) {
            queued = 1;
            if (head < 0 || L->free_req < S->lane[head].free_req) head = (int32_t)c;   /* ties: smaller id */
        }
        if (L->q_head < L->q_tail && L->head_running) running = 1;
    }
    if (!queued && !serving) return 0;
    if (!serving && !running) {                      /* the device is idle: serve the head */
        orc_lane *L = &S->lane[head];
        L->pc = PC_FREE_RET; L->cpu_next = t + S->in->free_ns;
        tr(S, t, TR_FREE_START, head, L->inst, L->cpu_next, 0);
    }
    return 1;
}

static int is_copy(const orc_sim *S, uint32_t c, uint32_t K)
{
    return S->in->k_flags && (S->in->k_flags[S->lane[c].kbase + K] & 1u);
}

static void dispatch(orc_sim *S, int64_t t)
{
    orc_cand cand[ORC_MAX_CHAINS];
    uint32_t n = 0;
    if (barrier(S, t)) return;
    /* the copy engine (Table 3 "cuMemCpy: no stream priority"; SPEC.md:271;
     * DESIGN.md R31): one memcpy at a time, the waiting memcpy heads in (ready time, chain)
     * order, independent of the compute capacity */
    if (!S->copy_busy) {
        int32_t best = -1;
        for (uint32_t c = 0; c < S->nL; ++c) {
            const orc_lane *L = &S->lane[c];
            if (!(L->q_head < L->q_tail && !L->head_running && is_copy(S, c, L->q[L->q_head].K))) continue;
            if (best < 0 || L->head_ready < S->lane[best].head_ready) best = (int32_t)c;
        }
        if (best >= 0) {
            orc_lane *L = &S->lane[best];
            uint32_t K = L->q[L->q_head].K;
            S->copy_busy = 1;
            L->head_running = 1;
            L->head_end = t + kernel_duration(S, (uint32_t)best, L->inst, K);
            tr(S, t, TR_DISPATCH, best, L->inst, K, L->head_end);
        }
    }
    for (uint32_t c = 0; c < S->nL; ++c) {
        orc_lane *L = &S->lane[c];
        if (L->q_head < L->q_tail && !L->head_running && !is_copy(S, c, L->q[L->q_head].K)) {
            cand[n].level = L->level; cand[n].ready = L->head_ready; cand[n].chain = c; ++n;
        }
    }
    qsort(cand, n, sizeof(orc_cand), orc_cand_cmp);
    for (uint32_t j = 0; j < n; ++j) {
        orc_lane *L = &S->lane[cand[j].chain];
        uint32_t K = L->q[L->q_head].K;
        uint32_t u = S->in->k_util[L->kbase + K];
        if (S->gpu_used + u > 1000) continue;            /* does not fit: skip (greedy) */
        /* contention (R30): a kernel started while
         * U_run per-mille of the GPU is busy runs d + floor(d * alpha * U_run / 10^6) */
        int64_t d = kernel_duration(S, cand[j].chain, L->inst, K);
        d += d * (int64_t)S->in->contention_permille * (int64_t)S->gpu_used / 1000000;
        S->gpu_used += u;
        L->head_running = 1;
        L->head_end = t + d;
        tr(S, t, TR_DISPATCH, cand[j].chain, L->inst, K, L->head_end);
    }
}

/* Phase A: retire every kernel ending at t (R21). */
static void retire(orc_sim *S, int64_t t)
{
    for (uint32_t c = 0; c < S->nL; ++c) {
        orc_lane *L = &S->lane[c];
        if (!(L->q_head < L->q_tail && L->head_running && L->head_end == t)) continue;
        uint32_t K = L->q[L->q_head].K;
        if (is_copy(S, c, K)) S->copy_busy = 0;          /* R31 */
        else S->gpu_used -= S->in->k_util[L->kbase + K];
        L->q_head++; L->done++; L->head_running = 0;
        if (L->q_head < L->q_tail) L->head_ready = t;    /* next kernel becomes head */
        tr(S, t, TR_RETIRE, c, L->inst, K, 0);
        if (L->pc == PC_SYNC_WAIT && L->done >= L->sync_target) {
            L->pc = PC_SYNC_RET; cpu_busy(S, c, t, L->sync_cost);
        }
    }
}

/* CPU scheduling of the chains' threads on cpu_cores cores ("we
 * calculate UL_C(t0) and then map the urgency level to the corresponding CPU priority
 * PRI_C for all active chains ... sched_setscheduler(SCHED_FIFO)"; SPEC.md:130-134;
 * DESIGN.md R29).  UrgenGo re-ranks every active chain by its urgency at t whenever a
 * chain starts a CPU segment; STATIC uses its static levels; the other policies give every
 * thread the same priority.  The runnable jobs are ordered by (priority descending, time
 * they became runnable, chain id) and the first cpu_cores of them hold a core; a job that
 * loses its core keeps its remaining work. */
typedef struct { int64_t prio, ready; uint32_t chain; } orc_job;

static int orc_job_cmp(const void *a, const void *b)
{
    const orc_job *x = a, *y = b;
    if (x->prio != y->prio) return x->prio > y->prio ? -1 : 1;
    if (x->ready != y->ready) return x->ready < y->ready ? -1 : 1;
    return x->chain < y->chain ? -1 : (x->chain > y->chain);
}

static void cpu_schedule(orc_sim *S, int64_t t)
{
    const orc_input *in = S->in;
    if (in->cpu_cores == 0) return;
    if (S->rerank) {
        S->rerank = 0;
        for (uint32_t c = 0; c < S->nL; ++c) {
            orc_lane *L = &S->lane[c];
            if (L->pc == PC_ARRIVE || L->pc == PC_WAIT_MSG || L->pc == PC_DONE) continue;   /* not active */
            L->cpu_prio = orc_urgency_key(current_laxity(S, c, t));
        }
        S->cpu_dirty = 1;
    }
    if (!S->cpu_dirty) return;
    S->cpu_dirty = 0;
    orc_job jobs[ORC_MAX_CHAINS];
    uint32_t n = 0;
    for (uint32_t c = 0; c < S->nL; ++c) {
        const orc_lane *L = &S->lane[c];
        if (!L->job) continue;
        jobs[n].prio = in->kind == ORC_STATIC ? -(int64_t)L->static_level : in->kind == ORC_URGENGO ? L->cpu_prio : 0;
        jobs[n].ready = L->job_ready; jobs[n].chain = c; ++n;
    }
    qsort(jobs, n, sizeof(orc_job), orc_job_cmp);
    for (uint32_t i = 0; i < n; ++i) {
        orc_lane *L = &S->lane[jobs[i].chain];
        if (i < in->cpu_cores && !L->job_run) {
            L->job_run = 1; L->run_start = t; L->cpu_next = t + L->job_rem;
            tr(S, t, TR_CPU_RUN, jobs[i].chain, L->inst, L->job_rem, 0);
        } else if (i >= in->cpu_cores && L->job_run) {
            L->job_run = 0; L->job_rem -= t - L->run_start; L->cpu_next = ORC_INF;
            tr(S, t, TR_CPU_STOP, jobs[i].chain, L->inst, L->job_rem, 0);
        }
    }
}

static void cal_sample(orc_sim *S)
{
    /* highest urgency among all active kernels of the AKB */
    int have = 0; int64_t best = 0, bestL = 0;
    for (uint32_t c = 0; c < S->nL; ++c) {
        orc_lane *L = &S->lane[c];
        for (uint32_t e = 0; e < L->akb_n; ++e) {
            int64_t k = orc_urgency_key(L->akb[e].L);
            if (!have || k > best) { best = k; bestL = L->akb[e].L; have = 1; }
        }
    }
    if (!have || bestL < 0) return;                      /* skip empty / negative (Q5) */
    if (S->cal_n < S->cal_cap) S->cal_L[S->cal_n++] = bestL;
}

/* Simulate scenario s.  Returns 0 on success. */
static int sim_scenario(const orc_input *in_all, uint64_t s, uint32_t *rec, int64_t *agg,
                        int64_t *trace, int64_t trace_cap, int64_t *trace_len,
                        int64_t *cal_L, int64_t cal_cap, int64_t *cal_n, int64_t cal_end)
{
    /* template variants (R33): scenario s runs on kernel-record set s mod V */
    orc_input in_v = *in_all;
    const orc_input *in = &in_v;
    if (in_all->num_variants > 1) {
        uint64_t nk = 0, nt = 0;
        for (uint32_t c = 0; c < in_all->num_chains; ++c) nt += in_all->ch_ntasks[c];
        for (uint64_t j = 0; j < nt; ++j) nk += in_all->t_nk[j];
        uint64_t off = (s % in_all->num_variants) * nk;
        in_v.k_nom += off; in_v.k_est += off; in_v.k_util += off;
        if (in_v.k_flags) in_v.k_flags += off;
    }
    orc_sim S;
    memset(&S, 0, sizeof S);
    S.in = in; S.s = s; S.C = in->num_chains; S.agg = agg;
    S.trace = trace; S.trace_cap = trace_cap; S.trace_len = trace_len ? *trace_len : 0;
    S.cal_L = cal_L; S.cal_cap = cal_cap; S.cal_n = 0; S.cal_end = cal_end; S.cal_next = 0;
    S.t_prev = -1;
    int rc = 0;
    /* threads: one per chain (R6), or one per task, chain-major (per-task executors, R32) */
    S.nL = S.C;
    if (in->task_exec) { S.nL = 0; for (uint32_t c = 0; c < S.C; ++c) S.nL += in->ch_ntasks[c]; }
    S.lane = calloc(S.nL, sizeof(orc_lane));
    S.snap_L = calloc(S.nL, sizeof(int64_t));
    S.snap_n = calloc(S.nL, sizeof(uint32_t));
    S.snap_level = calloc(S.nL, sizeof(uint32_t));
    S.snap_busy = calloc(S.nL, sizeof(uint8_t));
    S.snap_tarr = calloc(S.nL, sizeof(int64_t));
    S.snap_R = calloc(S.nL, sizeof(int64_t));
    uint32_t kb = 0, tb = 0, nl = 0;
    for (uint32_t ch = 0; ch < S.C; ++ch) {
        uint32_t M = in->ch_ntasks[ch], N = 0, k0 = 0;
        for (uint32_t j = 0; j < M; ++j) N += in->t_nk[tb + j];
        for (uint32_t j = 0; j < (in->task_exec ? M : 1); ++j) {
            orc_lane *L = &S.lane[nl++];
            L->chain = ch; L->tbase = tb; L->kbase = kb; L->M = M; L->N = N;
            L->stage = in->task_exec ? j : 0; L->stage_end = in->task_exec ? j + 1 : M; L->k0 = k0;
            k0 += in->t_nk[tb + j];
            L->akb = calloc(L->N, sizeof(orc_akb_entry));
            L->cpu_hist = calloc((size_t)L->M * (in->cpu_ma_window ? in->cpu_ma_window : 1), sizeof(uint32_t));
            L->cpu_hist_n = calloc(L->M, sizeof(uint32_t));
            L->cpu_pred = calloc(L->M, sizeof(uint32_t));
            for (uint32_t q = 0; q < L->M; ++q) L->cpu_pred[q] = in->t_cpu_est[L->tbase + q];
            L->q = calloc(L->N, sizeof(orc_stream_entry));
            L->hash = 2166136261u;
        }
        tb += M; kb += N;
    }
    /* scenario factors (R3): P' = P / f_a, D' = D * f_d, tight set halved */
    uint64_t tight = 0;
    if (in->tight_explicit) tight = in->tight_mask;   /* an explicit mask names chains 0..31 */
    else if (in->ftight_permille) {
        uint32_t n_tight = (in->ftight_permille * S.C + 999) / 1000;
        for (uint32_t c = 0; c < S.C; ++c) {
            uint32_t wc = orc_word(in->seed, s, TAG_TIGHT, c, 0, 0), rank = 0;
            for (uint32_t o = 0; o < S.C; ++o) {
                uint32_t wo = orc_word(in->seed, s, TAG_TIGHT, o, 0, 0);
                if (wo < wc || (wo == wc && o < c)) ++rank;
            }
            if (rank < n_tight) tight |= 1ull << c;
        }
    }
    int64_t maxD = 0;
    int64_t *chD = calloc(S.C, sizeof(int64_t));
    for (uint32_t c = 0; c < S.nL; ++c) {
        orc_lane *L = &S.lane[c];
        L->Pp = in->ch_period[L->chain] * (int64_t)in->fa_den / (int64_t)in->fa_num;
        L->Dp = in->ch_deadline[L->chain] * (int64_t)in->fd_num / (int64_t)in->fd_den;
        if (tight & (1ull << L->chain)) L->Dp /= 2;
        if (L->Dp > maxD) maxD = L->Dp;
        chD[L->chain] = L->Dp;
    }
    /* STATIC (PAAM-like) levels: rank the chains by D' ascending, ties by chain id (R15) */
    for (uint32_t c = 0; c < S.nL; ++c) {
        uint32_t r = 1, ch = S.lane[c].chain;
        for (uint32_t o = 0; o < S.C; ++o)
            if (chD[o] < chD[ch] || (chD[o] == chD[ch] && o < ch)) ++r;
        S.lane[c].static_level = (S.C <= 1 || in->num_prio <= 1) ? 0
            : (uint32_t)(((uint64_t)(r - 1) * (in->num_prio - 1)) / (S.C - 1));
    }
    free(chD);
    S.H = in->horizon_ns;
    S.H_stop = S.H + maxD;                               /* R7 */
    for (uint32_t c = 0; c < S.nL; ++c) {
        orc_lane *L = &S.lane[c];
        L->inst = 0;
        L->t_arr = arrival(&S, c, 0);
        if (L->stage > 0) { L->pc = PC_WAIT_MSG; L->cpu_next = ORC_INF; }   /* R32: waits for a message */
        else if (L->t_arr < S.H) { L->pc = PC_ARRIVE; L->cpu_next = L->t_arr; }
        else { L->pc = PC_DONE; L->cpu_next = ORC_INF; }
    }
    /* main loop (R21) */
    for (;;) {
        int64_t t = ORC_INF;
        for (uint32_t c = 0; c < S.nL; ++c) {
            orc_lane *L = &S.lane[c];
            if (L->cpu_next < t) t = L->cpu_next;
            if (L->q_head < L->q_tail && L->head_running && L->head_end < t) t = L->head_end;
        }
        if (S.cal_L) {
            while (S.cal_next < S.cal_end && S.cal_next < t) { cal_sample(&S); S.cal_next += 1000000; }
        }
        if (t > S.H_stop) break;
        if (t <= S.t_prev) { rc = -3; break; }            /* every loop step advances time (R21) */
        S.t_prev = t;
        S.steps++;
        tr(&S, t, TR_STEP, -1, -1, 0, 0);
        retire(&S, t);                                                   /* Phase A */
        for (uint32_t c = 0; c < S.nL; ++c) {
            S.snap_L[c] = S.lane[c].L_last; S.snap_n[c] = S.lane[c].akb_n;
            S.snap_level[c] = S.lane[c].level; S.snap_busy[c] = S.lane[c].q_head < S.lane[c].q_tail;
            if (classical(&S)) { S.snap_tarr[c] = S.lane[c].t_arr; S.snap_R[c] = remaining_work(&S, c); }
        }
        for (uint32_t c = 0; c < S.nL; ++c)                              /* Phase B */
            if (S.lane[c].cpu_next == t) {
                if (S.lane[c].job) { S.lane[c].job = 0; S.lane[c].job_run = 0; S.cpu_dirty = 1; }   /* job done */
                lane_step(&S, c, t);
            }
        /* per-task executors (R32): messages published in a round are delivered at its end;
         * a thread waiting for one runs in the next round, at the same t, against the same
         * read view; a delivered message replaces an untaken one (queue depth 1) */
        while (in->task_exec) {
            int woke = 0;
            for (uint32_t c = 0; c < S.nL; ++c) {
                orc_lane *L = &S.lane[c];
                if (L->msg_pend) { L->msg = L->msg_pend; L->msg_pend = 0; }
                if (L->pc == PC_WAIT_MSG && L->msg) { L->cpu_next = t; woke = 1; }
            }
            if (!woke) break;
            for (uint32_t c = 0; c < S.nL; ++c)
                if (S.lane[c].pc == PC_WAIT_MSG && S.lane[c].cpu_next == t) lane_step(&S, c, t);
        }
        cpu_schedule(&S, t);                                             /* CPU cores (R29) */
        dispatch(&S, t);                                                 /* Phase C */
    }
    /* end of horizon (R7): admitted, unfinished instances are misses */
    const uint32_t stride = AGG_COUNTERS + in->rt_bins + RATIO_BINS;
    for (uint32_t c = 0, l0 = 0; c < S.C; l0 += in->task_exec ? in->ch_ntasks[c] : 1, ++c) {
        orc_lane *L;
        if (!in->task_exec) {
            L = &S.lane[c];
            uint32_t first_unstarted = L->inst;
            if (L->pc != PC_ARRIVE && L->pc != PC_DONE) { L->unfin++; first_unstarted = L->inst + 1; }
            if (L->pc != PC_DONE)
                for (uint32_t i = first_unstarted; arrival(&S, c, i) < S.H; ++i) { L->unfin++; L->total++; }
        } else {
            /* R32: the chain's last stage has recorded instances [0, expect); every later admitted
             * instance is unfinished; early exits and launches are summed over the stages */
            L = &S.lane[l0 + in->ch_ntasks[c] - 1];
            for (uint32_t i = L->expect; arrival(&S, l0, i) < S.H; ++i) L->unfin++;
            L->total = L->expect + L->unfin;
            uint32_t early = 0, launches = 0;
            for (uint32_t j = 0; j < in->ch_ntasks[c]; ++j) {
                early += S.lane[l0 + j].early; launches += S.lane[l0 + j].launches;
            }
            L->early = early; L->launches = launches;
        }
        L->miss += L->unfin;
        uint32_t *r = rec + (uint64_t)c * REC_WORDS;
        r[0] = L->total; r[1] = L->miss; r[2] = L->early; r[3] = L->unfin;
        r[4] = L->launches; r[5] = L->hash;
        r[6] = (uint32_t)L->sum_rt; r[7] = (uint32_t)(L->sum_rt >> 32);
        int64_t *a = agg + (int64_t)c * stride;
        a[0] += L->total; a[1] += L->miss; a[2] += L->early; a[3] += L->unfin; a[4] += (int64_t)L->sum_rt;
        if (L->total) a[AGG_COUNTERS + in->rt_bins + (uint64_t)100 * L->miss / L->total] += 1;
    }
    for (uint32_t c = 0; c < S.nL; ++c) {
        orc_lane *L = &S.lane[c];
        free(L->akb); free(L->q); free(L->cpu_hist); free(L->cpu_hist_n); free(L->cpu_pred);
    }
    agg[(int64_t)S.C * stride + COLL_BINS + 0] += S.launches;
    agg[(int64_t)S.C * stride + COLL_BINS + 1] += S.steps;
    if (trace_len) *trace_len = S.trace_len;
    if (cal_n) *cal_n = S.cal_n;
    free(S.lane); free(S.snap_L); free(S.snap_n); free(S.snap_level); free(S.snap_busy); free(S.snap_tarr);
    free(S.snap_R);
    return rc;
}

/* Simulate scenarios [scenario_begin, scenario_begin + scenario_count).
 * records: [count][C][8] u32; agg: int64 words (accumulated, caller zeroes);
 * trace (optional): [cap][6] int64 (t, kind, chain, instance, a, b). */
int orc_run(const orc_input *in, uint32_t *records, int64_t *agg,
            int64_t *trace, int64_t trace_cap, int64_t *trace_len)
{
    if (!in || in->num_chains == 0 || in->num_chains > ORC_MAX_CHAINS) return -1;
    if (in->fa_num == 0 || in->fa_den == 0 || in->fd_den == 0 || in->rt_bins == 0 || in->rt_bin_ns <= 0) return -1;
    if (in->t_flags) {                                /* a served cudaFree takes time (R28) */
        uint32_t nt = 0;
        for (uint32_t c = 0; c < in->num_chains; ++c) nt += in->ch_ntasks[c];
        for (uint32_t j = 0; j < nt; ++j) if ((in->t_flags[j] & 1u) && in->free_ns <= 0) return -1;
    }
    for (uint32_t c = 0; c < in->num_chains; ++c)     /* arrivals strictly increasing: P' > J (R3) */
        if (in->ch_period[c] * (int64_t)in->fa_den / (int64_t)in->fa_num <= in->jitter_ns) return -2;
    if (in->task_exec) {                              /* R32: at most ORC_MAX_CHAINS threads; no R26 predictor */
        uint32_t nt = 0;
        for (uint32_t c = 0; c < in->num_chains; ++c) nt += in->ch_ntasks[c];
        if (nt > ORC_MAX_CHAINS) return -2;
        if (in->cpu_ma_window) return -1;
    }
    if (trace_len) *trace_len = 0;
    for (uint64_t j = 0; j < in->scenario_count; ++j) {
        uint32_t *rec = records + j * (uint64_t)in->num_chains * REC_WORDS;
        int rc = sim_scenario(in, in->scenario_begin + j, rec, agg, trace, trace_cap, trace_len, 0, 0, 0, 0);
        if (rc) return rc;
    }
    return 0;
}

/* TH_urgent from recorded maximum urgencies: the
 * nearest-rank pct-th percentile of UL = 1/L over the samples, returned as its
 * laxity L_th (UL >= TH <=> 0 <= L <= L_th).  Samples with L < 0 are skipped
 * (SPEC.md:328-330).  Sorts L[] in place by ascending urgency.  -1 if empty.
 * DESIGN.md Q5 states the rank reading. */
int64_t orc_nearest_rank_lth(int64_t *L, int64_t n, int64_t pct)
{
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i) if (L[i] >= 0) L[m++] = L[i];
    if (m == 0) return -1;
    for (int64_t i = 1; i < m; ++i) {                 /* insertion sort by urgency key, plain */
        int64_t ll = L[i], kk = orc_urgency_key(ll), j = i - 1;
        while (j >= 0 && orc_urgency_key(L[j]) > kk) { L[j + 1] = L[j]; --j; }
        L[j + 1] = ll;
    }
    /* rank floor(pct/100 * m) + 1 in ascending urgency: the smallest sample with
     * more than pct % of the samples below it, so that UL >= TH holds for the top
     * (100 - pct) % only (SPEC.md:328 example: {0.01 x95, 0.05 x5} -> 0.05). */
    int64_t k = (pct * m) / 100 + 1;
    if (k > m) k = m;
    return L[k - 1];
}

/* Calibration samples ("periodically recording the highest urgency
 * value among all active kernels in AKB"; Q5): each scenario of the batch
 * is simulated with the threshold disabled (L_th = -1, nothing is truly urgent) and,
 * every 1 ms of the first min(H, window), the laxity of the most urgent AKB entry is
 * recorded (no sample when the AKB is empty or that laxity is negative).  Scenario j's
 * samples go to L_out[j * cap ...], their number to n_out[j]. */
int orc_calibration_samples(const orc_input *in_, int64_t window_ns, int64_t *L_out, int64_t cap, int64_t *n_out)
{
    orc_input in = *in_;
    in.lax_threshold_ns = -1;
    int64_t end = in.horizon_ns < window_ns ? in.horizon_ns : window_ns;
    uint32_t *rec = calloc((size_t)in.num_chains * REC_WORDS, sizeof(uint32_t));
    int64_t *agg = calloc((size_t)in.num_chains * (AGG_COUNTERS + in.rt_bins + RATIO_BINS) + COLL_BINS + 2,
                          sizeof(int64_t));
    int rc = 0;
    for (uint64_t j = 0; j < in.scenario_count && rc == 0; ++j)
        rc = sim_scenario(&in, in.scenario_begin + j, rec, agg, 0, 0, 0, L_out + (int64_t)j * cap, cap,
                          &n_out[j], end);
    free(rec); free(agg);
    return rc;
}

/* TH_urgent calibration (Q5): the samples of every
 * scenario of the batch pooled, and the laxity of their nearest-rank 95th percentile
 * urgency returned.  *n_samples receives the number of samples; -1 if none. */
int64_t orc_calibrate(const orc_input *in, int64_t window_ns, int64_t *n_samples)
{
    int64_t end = in->horizon_ns < window_ns ? in->horizon_ns : window_ns;
    int64_t cap = end / 1000000 + 2;
    uint64_t cnt = in->scenario_count ? in->scenario_count : 1;
    orc_input one = *in;
    one.scenario_count = cnt;
    int64_t *L = calloc((size_t)(cap * (int64_t)cnt), sizeof(int64_t));
    int64_t *n = calloc(cnt, sizeof(int64_t));
    orc_calibration_samples(&one, window_ns, L, cap, n);
    int64_t m = 0;                                     /* pool: concatenate the scenarios' samples */
    for (uint64_t j = 0; j < cnt; ++j)
        for (int64_t i = 0; i < n[j]; ++i) L[m++] = L[(int64_t)j * cap + i];
    int64_t out = orc_nearest_rank_lth(L, m, 95);
    if (n_samples) *n_samples = m;
    free(L); free(n);
    return out;
}
