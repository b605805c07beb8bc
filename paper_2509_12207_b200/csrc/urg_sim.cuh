// urg_sim.cuh -- the B200 (sm_100a) batched UrgenGo launch-policy simulation kernel.
// Included by the urg_sim_part*.cu translation units, each instantiating a slice of
// the (policy kind, UrgenGo flags, factor table, build) table so nvcc runs them in
// parallel; urg_sim.cu holds the dispatch table.
//
// One warp simulates one scenario; lane c is task chain c (C <= 32).  Per-chain
// state lives in registers; the workload template lives in shared memory
// (staged once per CTA with cp.async.bulk + mbarrier); cross-chain reads use
// warp votes, REDUX min/add reductions and a per-warp shared-memory snapshot.
// The rules are DESIGN.md "Model M0" (R0-R23); comments name the rule and the
// paper passage.  Nothing here is shared with the CPU oracle (oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "urg_layout.h"

#define FULL 0xFFFFFFFFu
#define INF64 0x7FFFFFFFFFFFFFFFLL
// 32-bit distances of a lane's next CPU event and kernel end from the last step time (see
// the event loop): D_INF = none, D_FAR = at least 2^31 ns away (a lower bound), and every
// value drifts down by less than D_SLOW between two exact refreshes
#define D_INF 0xFFFFFFFFu
#define D_FAR 0x80000000u
#define D_SLOW 0x40000000u
#ifdef URG_NO_DIST
#define URG_DIST_OFF true
#else
#define URG_DIST_OFF false
#endif

enum { K_FIFO = 0, K_STATIC = 1, K_URGENGO = 2, K_EDF = 3, K_SJF = 4, K_HRRN = 5, K_LCUF = 6 };
enum { F_BIND = 1, F_DELAY = 2, F_EARLY = 4, F_COLL = 8 };
enum { S_ASYNC = 0, S_EACH = 1, S_BATCHED = 2, S_OVERLAP = 3 };
// lane program counter; the per-launch states come first so one range test skips the
// per-task / per-instance states on the common path
enum { PC_ENQUEUE = 0, PC_ATTEMPT, PC_CPU_DONE, PC_SYNC_RET, PC_FREE_RET, PC_ARRIVE, PC_TASK_START, PC_SYNC_WAIT,
       PC_FREE_WAIT, PC_WAIT_MSG, PC_DONE };
enum { ERR_TIME = 1, ERR_GUARD = 2, ERR_DEBUG = 16 };   // debug build: 16 + invariant id
// debug-build event kinds (the oracle's trace codes, oracle/oracle.py TRACE_KINDS)
enum { TR_STEP = 1, TR_INST_START, TR_TASK_START, TR_EVAL, TR_DELAY, TR_BIND, TR_ENQUEUE, TR_DISPATCH, TR_RETIRE,
       TR_SYNC_CALL, TR_SYNC_RET, TR_FREE_CLOSE, TR_INST_DONE, TR_EARLY_EXIT, TR_COLLISION };
// debug-build invariants (SPEC.md:171-174 and DESIGN.md R16-R21), checked on device
enum { INV_START_BEFORE_READY = 1, INV_CAPACITY, INV_RETIRE_TIME, INV_CONSERVATION, INV_COUNTS, INV_PAST_EVENT,
       INV_LEVEL };
#ifdef URG_DEBUG
#define URG_TR(t, kind, a, b) trace_row((t), (kind), (a), (b))
#define URG_DASSERT(cond, id)                                                                                    \
    do {                                                                                                         \
        if (!(cond) && atomicCAS((unsigned long long *)err, 0ull, (unsigned long long)(ERR_DEBUG + (id))) == 0ull) \
            err[1] = s;                                                                                          \
    } while (0)
#else
#define URG_TR(t, kind, a, b) ((void)0)
#define URG_DASSERT(cond, id) ((void)0)
#endif

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11) -- device copy, KAT-tested (tests/test_gpu_*.py)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// word(tag, c, i, k) of scenario s (R3-R5).  Not inlined: the draws are
// rare (per arrival, instance, sync call), and an inlined copy lets the compiler
// hoist ~80 speculative instructions into the per-step path.
static __device__ __noinline__ uint32_t rng_word(uint64_t seed, uint32_t s, uint32_t tag, uint32_t c, uint32_t i,
                                             uint32_t k)
{
    const uint4 o = philox4x32_10(make_uint4(s, (tag << 24) | (c << 16), i, k >> 2),
                                  make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
    const uint32_t q = k & 3u;
    return q == 0 ? o.x : q == 1 ? o.y : q == 2 ? o.z : o.w;
}


// All four words of the block holding word (tag, c, i, k): words k & ~3 .. k | 3 share one
// Philox call (R4; the per-kernel draws are cached four at a time).
static __device__ __noinline__ uint4 rng_block(uint64_t seed, uint32_t s, uint32_t tag, uint32_t c, uint32_t i,
                                               uint32_t k)
{
    return philox4x32_10(make_uint4(s, (tag << 24) | (c << 16), i, k >> 2),
                         make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

// ---------------------------------------------------------------------------
// small warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t lane_id()
{
    uint32_t r;
    asm("mov.u32 %0, %%laneid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t lane_bit()   // 1 << lane_id()
{
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_eq;" : "=r"(r));
    return r;
}
__device__ __forceinline__ int64_t warp_min_nonneg(int64_t v)    // v >= 0 for every lane
{
    const uint32_t hi = (uint32_t)((uint64_t)v >> 32), lo = (uint32_t)v;
    const uint32_t mh = __reduce_min_sync(FULL, hi);
    const uint32_t ml = __reduce_min_sync(FULL, hi == mh ? lo : 0xFFFFFFFFu);
    return (int64_t)(((uint64_t)mh << 32) | ml);
}

__device__ __forceinline__ int64_t shfl64(int64_t v, int src)
{
    return (int64_t)__shfl_sync(FULL, (unsigned long long)v, src);
}

// urgency key: orders as 1/L, L = 0 saturating (R9)
__device__ __forceinline__ int64_t urgency_key(int64_t L)
{
    return L == 0 ? INF64 : (L > 0 ? (((int64_t)1 << 62) - L) : (-((int64_t)1 << 62) - L));
}

// ---------------------------------------------------------------------------
// shared-memory staging helpers (cp.async.bulk + mbarrier)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void stage_blob(uint8_t *dst, const uint8_t *src, uint32_t bytes, uint64_t *mbar)
{
    const uint32_t bar = smem_addr(mbar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        for (uint32_t off = 0; off < bytes; off += 32768u) {
            const uint32_t n = bytes - off < 32768u ? bytes - off : 32768u;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(dst + off)),
                "l"(src + off), "r"(n), "r"(bar)
                : "memory");
        }
    }
    __syncthreads();   // barrier initialised before anyone waits on it
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "URG_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra URG_WAIT_%=;\n}" ::"r"(bar)
        : "memory");
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
struct Tmpl {   // shared-memory views of the staged template
    const UrgChainRec *ch;
    const UrgTaskRec *task;
    const int32_t *inst_q;
    const uint32_t *kern_q;
};

// One kernel record from HBM/L2 (read-only path, one 16-byte load).  The records of all
// template variants live in global memory (R33); a CTA's warps work on scenarios of the
// same variant at the same time (grouped work order), so the record lines stay in L1.
__device__ __forceinline__ UrgKernRec kern_rec(const UrgKernRec *k)
{
    const uint4 q = __ldg(reinterpret_cast<const uint4 *>(k));
    UrgKernRec r;
    r.nominal_ns = q.x; r.estimate_ns = q.y; r.util_permille = q.z; r.flags = q.w;
    return r;
}

// Work index -> scenario offset, grouping the scenarios of one template variant (offsets o with
// (begin + o) mod V fixed) into consecutive work indices (R33).  Identity when V = 1.
__device__ __forceinline__ uint64_t work_offset(uint64_t j, uint64_t S, uint32_t V)
{
    if (V <= 1) return j;
    const uint64_t q = S / V, m = S % V;
    uint64_t g, r;
    if (j < m * (q + 1)) { g = j / (q + 1); r = j % (q + 1); }
    else { const uint64_t jj = j - m * (q + 1); g = m + jj / q; r = jj % q; }
    return g + r * V;
}

// One instantiation per (policy kind, UrgenGo flags, per-kernel factor table present):
// the policy is uniform over a launch, so its branches are resolved at compile time
// and code a policy never runs (e.g. the per-kernel Philox draw) is not in its loop.
//
// WIDE: the throughput build (1024 threads per CTA, so <= 64 registers and 32 warps per
// SM) for batches that fill the GPU; otherwise the latency build (512 threads, ~100
// registers), faster per scenario when there are fewer scenarios than warp slots.
//
// CAL: the TH_urgent calibration build (Q5): every 1 ms of
// simulated time before P.cal_end the laxity of the most urgent AKB entry is appended
// to the scenario's sample row; no records or aggregates are written.
//
// EXT: the extended-model build (estimation noise R25, CPU predictor R26, cudaFree
// barriers R28 resolved at run time); the core build has none of their branches (the
// policies of the benchmarks use none of them and run ~9 % faster without).
//
// PK: two scenarios per warp (lanes 0-15 and 16-31, at most 16 chains), throughput core
// build only: the halves step in lockstep, every warp collective is segmented per half,
// so the step's overhead is shared by two scenarios.
//
// SMALL: the latency core build for batches of at most 8 warps per SM: 256-thread CTAs, so
// ptxas may use up to 255 registers (it takes ~134; measured 2.3 % faster on configs[1]
// than the 128-register cap of the 512-thread build).
template <int KIND, int FLAGS, bool KQ, bool WIDE, bool CAL = false, bool EXT = true, bool PK = false,
          bool SMALL = false>
// packed-build CTA size per policy: the packed loop's throughput grows with resident warps (22 -> 26
// warps per SM: 2.36 -> 2.53 G launch events/s on a configs[3] slice), so UrgenGo takes the largest
// CTA, 1024 threads (64 registers, a few spilled values: 2.55 -> 2.63 G/s against 832 / 72), and the
// ASYNC policies 896 (72 registers: configs[2] FIFO 4.91 -> 5.04, STATIC 4.69 -> 4.85 G/s against
// 768 / 80) -- profiles/r02_ab_m_dp_pre2_cta.txt
#ifndef URG_PK_THREADS
#define URG_PK_THREADS 1024
#endif
#ifndef URG_PK_THREADS_ASYNC
#define URG_PK_THREADS_ASYNC 896
#endif
#ifndef URG_LAT_THREADS
#define URG_LAT_THREADS 512
#endif
__global__ void __launch_bounds__(WIDE ? (PK ? (KIND == K_URGENGO ? URG_PK_THREADS : URG_PK_THREADS_ASYNC) : 1024) : (SMALL ? 256 : URG_LAT_THREADS), 1)
urg_sim_kernel(const uint8_t *__restrict__ blob, const UrgSimParams P, uint32_t *__restrict__ records,
               unsigned long long *__restrict__ agg, unsigned long long *__restrict__ work,
               long long *__restrict__ err)
{
    extern __shared__ __align__(128) uint8_t sm[];
    // packed UrgenGo build: lane index and lane bit from the special registers (one S2R each when the
    // compiler rematerialises them at 64 registers, instead of S2R TID + logic): configs[3] slice
    // 2.630 -> 2.730 G/s, configs[4] 3.290 -> 3.398; the other builds measured 0.6-0.8 % slower with it
    // (profiles/r02_ab_p_laneid.txt)
    constexpr bool sreg_lane = PK && KIND == K_URGENGO;
    const int lane = sreg_lane ? (int)lane_id() : (int)(threadIdx.x & 31);
    // packed UrgenGo build: the warp index through a shuffle from lane 0, warp-uniform by construction,
    // so the compiler keeps the warp's slot base in a uniform register instead of rematerialising it
    // (S2R TID + the shared-window base + multiply) at every use: configs[3] slice 2.868 -> 2.965 G/s,
    // configs[4] 3.516 -> 3.544; FIFO measured 3 % slower with it (profiles/r02_ab_w_uniform_warp.txt)
#ifndef URG_UW_ALL
#define URG_UW_ALL 0
#endif
    constexpr bool uw_on = URG_UW_ALL || sreg_lane;
    const int warp = uw_on ? __shfl_sync(FULL, (int)(threadIdx.x >> 5), 0) : (int)(threadIdx.x >> 5);

    // ---- A0: template staging (once per CTA) ----
    stage_blob(sm, blob, P.blob_bytes, (uint64_t *)(sm + P.mbar_offset));
    const UrgBlobHeader *hdr = (const UrgBlobHeader *)sm;
    UrgChainRec *chs = (UrgChainRec *)(sm + hdr->off_chains);
    Tmpl T;
    T.ch = chs;
    T.task = (const UrgTaskRec *)(sm + hdr->off_tasks);
    T.inst_q = hdr->off_inst_q ? (const int32_t *)(sm + hdr->off_inst_q) : nullptr;
    T.kern_q = hdr->off_kern_q ? (const uint32_t *)(sm + hdr->off_kern_q) : nullptr;
    const uint32_t C = P.num_lanes;    // threads: chains, or tasks under per-task executors (R32)
    const uint32_t NC = P.num_chains;  // chains: records and aggregates

    // per-warp Phase B snapshot (R21): last laxity of each lane, then its stream level
    // per-warp Phase B snapshot (R21), 1 KB: last laxity, two policy keys, stream level
    int64_t *snapL = (int64_t *)(sm + P.snap_offset) + warp * (URG_SNAP_BYTES_PER_LANE * 32 / 8);
    int64_t *snapA = snapL + 32, *snapB = snapL + 64;
    uint32_t *snapLev = (uint32_t *)(snapL + 96);
    uint32_t *mbox = (uint32_t *)(snapL + 112);   // R32: message published to each lane this round
    UrgVarRec *myvar = (UrgVarRec *)(snapL + 128);  // R33: each lane's variant estimate totals
    uint4 *kqw = (uint4 *)(snapL + 192);            // R4: the lane's current block of four KERN words
    uint4 *syw = (uint4 *)(snapL + 256);            // R5: the lane's current block of four SYNC words
    // cold per-lane scalars kept in shared memory (read once per instance / on the rare path), so the
    // packed build's registers hold the per-step state: P' and the half's H_stop
    volatile int64_t *cold_Pp = snapL + 320, *cold_Hs = snapL + 352;
    // ... the throughput UrgenGo build's t_arr and D' (read per instance), and every build's per-scenario
    // record counters of R22 (updated once per instance)
    volatile int64_t *cold_Ta = snapL + 384, *cold_Dp = snapL + 416;
    // (launches: the kernels launched by the lane's finished instances; the current instance's are
    // launched - k_first, so the per-launch path keeps no launch counter)
    struct UrgAcc { uint32_t total, miss, early, unfin, hash, launches; unsigned long long sum_rt; };   // 32 B
    volatile UrgAcc *rac = (volatile UrgAcc *)(snapL + 448) + lane;
    constexpr bool urg = KIND == K_URGENGO;
    constexpr bool cls = KIND >= K_EDF;        // classical policies (R27): AKB-tracking, no urgency
    constexpr bool akb_on = urg || cls;
    constexpr bool f_bind = urg && (FLAGS & F_BIND), f_delay = urg && (FLAGS & F_DELAY),
                   f_early = urg && (FLAGS & F_EARLY);
    constexpr bool coll = urg && (FLAGS & F_COLL);   // collision metric (R24): not in the schedule
    // Core build: Phase C's fit ballot runs at every step and is itself the test, so no "new
    // stream head" vote sits between Phase B and Phase C (a head that did not fit at an earlier
    // Phase C still does not: `used` only falls at a retirement).
    // Measured: +1-2 % on UrgenGo packed in round 1, +8 % on the round-2 build (configs[3] slice 2.772 ->
    // 2.993 G/s, profiles/r02_ab_ac_newhead_vote_rejected.txt); the latency build ran 3x slower; the
    // ASYNC policies (FIFO / STATIC) lost 13 % with it (configs[2]) and keep the new-head vote.
#ifdef URG_OLD_CALWAYS
    constexpr bool c_always = PK && !EXT && !CAL;
    constexpr bool r17_sel = true;
#else
    constexpr bool c_always = PK && !EXT && !CAL && urg;
    constexpr bool r17_sel = urg;   // R17 with selects for UrgenGo, branches for the others
#endif
    const bool noise = EXT && urg && P.noise_pm > 0;       // R25
    const bool ma = EXT && akb_on && P.ma_w > 0;           // R26 (every policy that estimates remaining work)
    const bool has_free = EXT && P.has_free != 0;          // R28: some task ends with cudaFree
    const bool cores_on = EXT && P.cpu_cores > 0;          // R29: the chains' threads share P.cpu_cores cores
    const bool contend = EXT && P.alpha_pm > 0;            // R30: co-running kernels slow a starting one down
    const bool has_copy = EXT && P.has_copy != 0;          // R31: memcpy operations on the copy engine
    const bool te = EXT && P.task_exec != 0;               // R32: one executor thread per task
    // R26 predictor state of this lane's chain in shared memory: [max_tasks][W] ring of
    // measured CPU durations, [max_tasks] counts, [max_tasks] this instance's estimates
    uint32_t *ma_ring = (uint32_t *)(sm + P.ma_offset) + (size_t)threadIdx.x * P.ma_slot;
    uint32_t *ma_cnt = ma_ring + P.ma_max_tasks * P.ma_w;
    uint32_t *ma_pred = ma_cnt + P.ma_max_tasks;
    // lambda (+ lambda_akb for UrgenGo), host-derived.  The packed builds of the other policies read it
    // from the parameter bank at each use (a constant operand) instead of holding it in registers:
    // configs[2] FIFO 5.07 -> 5.22 G/s; the packed UrgenGo build was 1 % slower that way and keeps the
    // register (profiles/r02_ab_aa_lambda_param.txt).  busy_launch_d32 != 0 <=> busy_launch_ns > 0.
    constexpr bool bl_param = PK && !urg;
    const int64_t busy_launch_r = P.busy_launch_ns;
#define busy_launch (bl_param ? P.busy_launch_ns : busy_launch_r)
    const uint32_t stride = P.agg_stride;
    // lane -> (half, chain); masks and snapshot slots stay indexed by lane
    const int half = PK ? (lane >> 4) : 0;
    const uint32_t hmask = PK ? (0xFFFFu << (lane & 16)) : FULL;
    auto lbit = [&]() -> uint32_t { return sreg_lane ? lane_bit() : (1u << lane); };
    const int hbase = PK ? (lane & 16) : 0;
    const uint32_t c = PK ? (uint32_t)(lane & 15) : (uint32_t)lane;
    const bool valid_c = c < C;
    // per-half warp collectives (the whole warp when !PK)
    auto hmin = [&](uint32_t v) -> uint32_t {
        if (!PK) return __reduce_min_sync(FULL, v);
        const uint32_t a = __reduce_min_sync(FULL, half ? 0xFFFFFFFFu : v);
        const uint32_t b = __reduce_min_sync(FULL, half ? v : 0xFFFFFFFFu);
        return half ? b : a;
    };
    auto hsum = [&](uint32_t v) -> uint32_t {
        if (!PK) return __reduce_add_sync(FULL, v);
        const uint32_t a = __reduce_add_sync(FULL, half ? 0u : v);
        const uint32_t b = __reduce_add_sync(FULL, half ? v : 0u);
        return half ? b : a;
    };
    auto hany = [&](bool pred) -> bool { return (__ballot_sync(FULL, pred) & hmask) != 0u; };
    auto hmin64 = [&](int64_t v) -> int64_t {   // v >= 0 in every lane
        const uint32_t hi = (uint32_t)((uint64_t)v >> 32), lo = (uint32_t)v;
        const uint32_t mh = hmin(hi);
        const uint32_t ml = hmin(hi == mh ? lo : 0xFFFFFFFFu);
        return (int64_t)(((uint64_t)mh << 32) | ml);
    };
    unsigned long long my_steps = 0;
#ifdef URG_STATS
    unsigned long long st_single = 0, st_multi = 0, st_dispatch = 0, st_rebase = 0;   // profiling build only
#endif

    // static per-chain template data
    UrgChainRec cr = {};
    if (valid_c) cr = chs[c];
    // the chain record: a register copy in the latency build; re-read from shared memory in
    // the throughput build (64-register budget), except the two bases the per-launch path uses
    const volatile UrgChainRec *crv = &chs[valid_c ? c : 0];
    const uint32_t kbase = cr.kern_base, tbase = cr.task_base;
#define CRF(f) (WIDE ? crv->f : cr.f)
    // R32: the chain this thread serves (randomness keys, records) and the tasks it runs
    const uint32_t cid = EXT ? cr.chain_id : c;
    const uint32_t stage = EXT ? cr.stage : 0u, k_first = EXT ? cr.k_first : 0u;
    const bool last_stage = !EXT || cr.stage_end == cr.num_tasks;

    bool first_fetch = true;
    for (;;) {
        // work fetch: the first scenario of every warp is static (consecutive within a CTA, so a
        // CTA's warps share template variants, R33), later ones come from one atomic counter
        unsigned long long jw = 0;
        const unsigned long long per_fetch = PK ? 2ull : 1ull;
        if (lane == 0)
            jw = first_fetch ? ((unsigned long long)blockIdx.x * (blockDim.x >> 5) + warp) * per_fetch
                             : (unsigned long long)gridDim.x * (blockDim.x >> 5) * per_fetch + atomicAdd(work, per_fetch);
        first_fetch = false;
        jw = __shfl_sync(FULL, jw, 0);
        if (jw >= P.scenario_count) break;
        jw += (unsigned long long)half;                        // PK: the upper half takes the next one
        const bool valid = valid_c && jw < P.scenario_count;
        if (jw < P.scenario_count) jw = work_offset(jw, P.scenario_count, P.num_variants);
        const uint32_t s = (uint32_t)(P.scenario_begin + jw);
        // R33: this scenario's template variant -- its kernel records and estimate totals
        const uint32_t vidx = P.num_variants > 1 ? s % P.num_variants : 0u;
        const UrgKernRec *KR = P.kern + (size_t)vidx * P.nk_total + kbase;
        if (valid_c) myvar[lane] = P.var[(size_t)vidx * C + c];   // the variant's estimate totals, per lane

        // ---- A1: scenario init (R3, R15 STATIC) ----
        int64_t Pp = 0, Dp = 0;
        if (valid) {
            Pp = CRF(period_ns) * (int64_t)P.fa_den / (int64_t)P.fa_num;
            Dp = CRF(deadline_ns) * (int64_t)P.fd_num / (int64_t)P.fd_den;
        }
        bool tight = false;
        // chain-level draws: with per-task executors only each chain's first thread counts (R32)
        const bool first_of_chain = stage == 0u;
        if (P.tight_explicit) tight = valid && ((P.tight_mask >> cid) & 1u);
        else if (P.ftight_permille) {
            const uint32_t n_tight = (P.ftight_permille * NC + 999u) / 1000u;
            const uint32_t w = valid ? rng_word(P.seed, s, URG_TAG_TIGHT, cid, 0, 0) : 0xFFFFFFFFu;
            uint32_t rank = 0;
            for (uint32_t o = 0; o < C; ++o) {
                const uint32_t wo = __shfl_sync(FULL, w, hbase + (int)o);
                const uint32_t co = EXT ? __shfl_sync(FULL, cid, hbase + (int)o) : o;
                const bool fo = !EXT || __shfl_sync(FULL, first_of_chain, hbase + (int)o);
                rank += (fo && (wo < w || (wo == w && co < cid))) ? 1u : 0u;
            }
            tight = valid && rank < n_tight;
        }
        if (tight) Dp /= 2;
        int64_t maxD = Dp;
#pragma unroll
        for (int o = PK ? 8 : 16; o > 0; o >>= 1) {
            const int64_t x = (int64_t)__shfl_xor_sync(FULL, (unsigned long long)maxD, o);
            maxD = x > maxD ? x : maxD;
        }
        const int64_t H = P.horizon_ns, H_stop = H + maxD;
        cold_Pp[lane] = Pp;
        cold_Hs[lane] = H_stop;
        uint32_t static_level = 0;
        {
            uint32_t r = 1;
            for (uint32_t o = 0; o < C; ++o) {
                const int64_t Do = shfl64(Dp, hbase + (int)o);
                const uint32_t co = EXT ? __shfl_sync(FULL, cid, hbase + (int)o) : o;
                const bool fo = !EXT || __shfl_sync(FULL, first_of_chain, hbase + (int)o);
                r += (fo && (Do < Dp || (Do == Dp && co < cid))) ? 1u : 0u;
            }
            if (NC > 1 && P.num_prio > 1) static_level = (uint32_t)(((uint64_t)(r - 1) * (P.num_prio - 1)) / (NC - 1));
        }

        // ---- per-lane dynamic state ----
        if (te) { mbox[lane] = 0u; __syncwarp(); }   // R32: no message published yet
        if (ma)
            for (uint32_t j = 0; j < P.ma_max_tasks; ++j) ma_cnt[j] = 0;
        int pc = PC_DONE;
        int64_t cpu_next = INF64;
        uint32_t dc = D_INF, dh = D_INF;       // distances of cpu_next and head_end from the last step time
        auto dsat = [](int64_t d) -> uint32_t { return d >= (int64_t)D_FAR ? D_FAR : (uint32_t)d; };
        uint32_t inst = 0;
        int64_t t_arr = 0;
        uint32_t Fg = 65536u, Fc = 65536u;
        uint32_t task = 0, launched = k_first, done = k_first, level = 0;
        uint32_t task_first = 0, task_end = 0;
        int64_t rem_g = 0, rem_c = 0;          // sum of estimates of kernels / CPU segments not yet passed
        // core UrgenGo build: Eq. 2 without its t, lb = t_arr + D' - rem_g - rem_c, kept instead of the two sums
        constexpr bool lb_on = urg && !EXT && WIDE;   // measured: +2.6 % / +4.7 % packed, -2 % latency build
        int64_t lb = 0;
        int32_t nz = 0;                        // R25: estimation noise of the current task instance, per-mille
        int64_t free_req = 0;                  // R28: time of this chain's pending cudaFree request
        bool job = false, job_run = false;     // R29: a CPU job exists / it holds a core
        bool cpu_chg = false, rerank_req = false;
        int64_t job_rem = 0, job_ready = 0, run_start = 0, cpu_prio = 0;
        int64_t acc = 0;
        uint32_t batch_start = 0, sync_target = 0, sync_ord = 0;
        uint32_t sync_cost = 0;                // sigma of the pending sync call (host: < 2^32 - 1 ns)
        uint32_t akb = 0;
        int64_t L_last = 0;
        int64_t head_end = INF64;              // end of the running kernel, INF64 when the stream runs nothing
        int64_t head_ready = 0;                // time the waiting head became head (R20 key)
        uint32_t head_util = 0;                // util of the running kernel
        uint32_t head_u = 0xFFFFu;             // util of the waiting head; 0xFFFF while none waits (no head,
                                               // the head runs, or the half's scenario ended), so the
                                               // Phase C fit test alone excludes such a lane
        uint32_t head_dur = 0;                 // its actual duration (R4), drawn when it becomes head
        UrgKernRec nxt = {};                   // latency build: record of the next kernel to launch (kernel
                                               // `launched`), loaded one launch ahead (off the critical path;
                                               // the throughput builds reload it: registers)
        bool head_copy = false;                // R31: the head is a memcpy (copy engine)
        rac->total = 0; rac->miss = 0; rac->early = 0; rac->unfin = 0; rac->hash = 2166136261u; rac->sum_rt = 0ull;
        rac->launches = 0;
        uint32_t msg = 0;                      // R32: delivered, untaken message (instance + 1), 0 = none
        uint32_t expect = 0;                   // R32, last stage: next instance to record
#ifdef URG_DEBUG
        // one scenario's event trace, rows (t, kind, lane, instance, a, b) as the oracle writes them
        auto trace_row = [&](int64_t t, int kind, int64_t a, int64_t b) {
            if (!P.trace_buf || !valid || (uint64_t)s != P.trace_scn) return;
            const unsigned long long i = atomicAdd((unsigned long long *)P.trace_buf, 1ull);
            if (i >= P.trace_cap) return;
            int64_t *r = P.trace_buf + 1 + 6 * i;
            r[0] = t; r[1] = kind; r[2] = kind == TR_STEP ? -1 : (int64_t)c; r[3] = kind == TR_STEP ? -1 : (int64_t)inst;
            r[4] = a; r[5] = b;
        };
#endif

        auto arrival = [&](uint32_t i) -> int64_t {
            int64_t jit = 0;
            if (P.jitter_ns > 0)
                jit = (int64_t)(rng_word(P.seed, s, URG_TAG_ARR, cid, i, 0) % (uint32_t)(P.jitter_ns + 1));
            return CRF(offset_ns) + (int64_t)i * (WIDE ? cold_Pp[lane] : Pp) + jit;
        };
        auto inst_factor = [&](uint32_t w, uint32_t sigma) -> uint32_t {
            if (!T.inst_q) return 65536u;
            const int64_t z = T.inst_q[w >> 20];
            int64_t F = 65536 + (z * (int64_t)sigma) / 1000000;
            return (uint32_t)(F < 6554 ? 6554 : F);
        };
        // Eq. 2 laxity (R9), with the remaining estimated work scaled by the task
        // instance's noise (R25; floor division, identity when noise is off)
        auto laxity = [&](int64_t t) -> int64_t {
            if (lb_on) return lb - t;
            int64_t rem = rem_g + rem_c;
            if (noise) rem = rem * (1000 + nz) / 1000;
            return t_arr + Dp - rem - t;
        };
        // R29: the thread is busy for d ns from t; with shared cores that is a CPU job
        auto cpu_busy = [&](int64_t t, int64_t d) {
            if (!cores_on || d == 0) { cpu_next = t + d; dc = dsat(d); return; }
            job = true; job_run = false; job_rem = d; job_ready = t; cpu_next = INF64; dc = D_INF; cpu_chg = true;
        };
        // R27 policy keys of this chain: EDF (t_arr + D', -), SJF (-, R), HRRN (t_arr, R),
        // LCUF (P', sum of kernel estimates); R = the remaining estimated work of Eq. 2
        auto cls_key_a = [&]() -> int64_t {
            return KIND == K_EDF ? t_arr + Dp : KIND == K_HRRN ? t_arr : KIND == K_LCUF ? Pp : 0;
        };
        auto cls_key_b = [&]() -> int64_t { return KIND == K_LCUF ? myvar[lane].gpu_est_chain : rem_g + rem_c; };
        // "chain o ranks before chain s" (ties by smaller chain id; exact 128-bit ratios)
        auto cls_before = [&](int64_t oA, int64_t oB, int o, int64_t sA, int64_t sB, int sl, int64_t t) -> bool {
            if (KIND == K_EDF || KIND == K_SJF) {
                const int64_t ko = KIND == K_EDF ? oA : oB, ks = KIND == K_EDF ? sA : sB;
                if (ko != ks) return ko < ks;
            } else if (KIND == K_HRRN) {
                if (oB == 0 || sB == 0) {
                    if (oB == 0 && sB != 0) return true;
                    if (sB == 0 && oB != 0) return false;
                } else {
                    const __int128 x = (__int128)(t - oA + oB) * sB, y = (__int128)(t - sA + sB) * oB;
                    if (x != y) return x > y;
                }
            } else if (KIND == K_LCUF) {
                const __int128 x = (__int128)oB * sA, y = (__int128)sB * oA;
                if (x != y) return x < y;
            }
            return o < sl;
        };

        if (lb_on) cold_Dp[lane] = Dp;
        if (valid) {
            t_arr = arrival(0);
            if (lb_on) cold_Ta[lane] = t_arr;
            if (te && stage > 0) pc = PC_WAIT_MSG;   // R32: waits for the previous task's message
            else if (t_arr < H) { pc = PC_ARRIVE; cpu_next = t_arr; dc = dsat(t_arr + 1); }   // t_prev = -1
        }
        // R32: take the delivered message (instance msg - 1); on the chain's last stage, record
        // the instances the message sequence skipped as misses, in order
        auto take_msg = [&]() {
            const uint32_t i = msg - 1u;
            msg = 0;
            if (last_stage)
                for (; expect < i; ++expect) {
                    rac->miss = rac->miss + 1u;
                    rac->hash = (((rac->hash ^ 0xFFFFFFFFu) * 16777619u) ^ 0xFFFFFFFFu) * 16777619u;
                }
            inst = i;
            t_arr = arrival(i);
            pc = PC_ARRIVE;
        };

        // ---- lane-local pieces of a loop step (R21); used by the warp-wide
        //      step and by the single-lane ("solo") steps below ----
        // R4: the actual duration of kernel k (the stream head) from its nominal duration -- drawn when
        // the kernel becomes head (kernels become head in stream order), kept until it starts.  (Drawing
        // the kernel behind the head ahead, so a retirement issues no load, measured 6 % slower on
        // configs[1]: profiles/r02_ab_m_dp_pre2_cta.txt)
        auto head_duration = [&](uint32_t nom, uint32_t k) -> uint32_t {
            uint64_t G = 65536u;
#ifdef URG_NO_KQCACHE
            if (KQ) G = T.kern_q[rng_word(P.seed, s, URG_TAG_KERN, cid, inst, k) >> 20];
#else
            if (KQ) {
                // kernel k follows k - 1 of the same instance, so the four words of a Philox block
                // are drawn once and kept in the lane's shared-memory slot; a new block (or the
                // instance's first kernel) refills it
                if ((k & 3u) == 0u || k == k_first) kqw[lane] = rng_block(P.seed, s, URG_TAG_KERN, cid, inst, k);
                G = T.kern_q[((const uint32_t *)&kqw[lane])[k & 3u] >> 20];
            }
#endif
            const uint64_t d = ((((uint64_t)nom * Fg) >> 16) * G) >> 16;
            // clamp to [1, 2^32 - 1] on the two 32-bit halves (one test of the high word, one max)
            const uint32_t lo = (uint32_t)d, lo1 = lo > 1u ? lo : 1u;
            return (uint32_t)(d >> 32) ? 0xFFFFFFFFu : lo1;
        };
        // Phase A for a lane whose running kernel ends at t (R19)
        auto retire = [&](int64_t t) {
            URG_DASSERT(head_end == t, INV_RETIRE_TIME);
            URG_TR(t, TR_RETIRE, done, 0);
            ++done;
            head_end = INF64;
            dh = D_INF;
            head_u = 0xFFFFu;
            if (launched > done) {
                head_ready = t;
                const UrgKernRec kr = kern_rec(KR + done);
                head_u = kr.util_permille; head_dur = head_duration(kr.nominal_ns, done);
                if (has_copy) head_copy = kr.flags & 1u;
            }
            if (pc == PC_SYNC_WAIT && done >= sync_target) { pc = PC_SYNC_RET; cpu_busy(t, sync_cost); }
        };
        // Phase C start of this lane's waiting head: non-preemptive, exact duration (R4, R19, R20)
        auto start_head = [&](int64_t t, uint32_t u_run) {
            uint64_t d = head_dur;
            if (contend && !head_copy) d += d * (uint64_t)P.alpha_pm * u_run / 1000000ull;   // R30
            head_util = head_copy ? 0u : head_u;   // a memcpy uses the copy engine, not the SMs (R31)
            head_u = 0xFFFFu;                       // no waiting head now
            head_end = t + (int64_t)d;
            dh = contend ? dsat((int64_t)d) : ((uint32_t)d < D_FAR ? (uint32_t)d : D_FAR);   // d < 2^32 without R30
            URG_DASSERT(t >= head_ready && launched > done, INV_START_BEFORE_READY);
            URG_TR(t, TR_DISPATCH, done, head_end);
        };
        // Phase B: this lane's CPU program at t, until it has to wait for time to pass.
        // urgent_m / active_m / snapL are the round snapshot of the other chains (R14, R15).
        // Returns true if the lane's stream got a new head (Phase C must run).
        auto phase_b = [&](int64_t t, uint32_t urgent_m, uint32_t active_m, uint32_t busy_m) -> bool {
            bool newhead = false;
            if (cores_on && job) { job = false; job_run = false; cpu_chg = true; }   // R29: the job completed
            if (te && pc == PC_WAIT_MSG) take_msg();   // woken by a delivered message (R32)
            for (uint32_t guard = 0;; ++guard) {
                if (guard > (1u << 24)) {
                    if (atomicCAS((unsigned long long *)err, 0ull, (unsigned long long)ERR_GUARD) == 0ull) err[1] = s;
                    cpu_next = INF64; dc = D_INF;
                    break;
                }
                if ((uint32_t)(pc - PC_SYNC_RET) <= (uint32_t)(PC_TASK_START - PC_SYNC_RET)) {
                bool next_inst = false;
                bool task_done = false;
                if (pc == PC_SYNC_RET) {   // sync returned: covered kernels leave the AKB
                    URG_TR(t, TR_SYNC_RET, sync_target, 0);
                    if (urg) URG_TR(t, TR_EVAL, laxity(t), launched);   // P:496 (the next attempt re-evaluates)
                    if (akb_on) akb = launched - sync_target;
                    if (launched < task_end) pc = PC_ATTEMPT;
                    else if (has_free && (T.task[tbase + task].flags & 1u)) {
                        // R28: the task ends with cudaFree -- request the device barrier and block
                        pc = PC_FREE_WAIT;
                        free_req = t;
                        cpu_next = INF64; dc = D_INF;
                        break;
                    } else task_done = true;
                }
                if (pc == PC_FREE_RET) task_done = true;   // R28: the barrier was served
                if (task_done) {
                    if (++task < (EXT ? CRF(stage_end) : CRF(num_tasks))) {
                        task_first = task_end;
                        task_end += T.task[tbase + task].num_kernels;
                        pc = PC_TASK_START;
                    } else if (!last_stage) {   // R32: publish instance inst to the next task's thread
                        mbox[lane + 1] = inst + 1u;
                        next_inst = true;
                    } else {   // instance complete (R18, R22)
                        expect = inst + 1u;
                        const int64_t rt = t - (lb_on ? cold_Ta[lane] : t_arr);
                        const int64_t Dpc = lb_on ? cold_Dp[lane] : Dp;
                        URG_DASSERT(te || (done == launched && launched == CRF(num_kernels)), INV_CONSERVATION);
                        URG_TR(t, TR_INST_DONE, rt, rt > Dpc ? 1 : 0);
                        if (rt > Dpc) rac->miss = rac->miss + 1u;
                        rac->sum_rt = rac->sum_rt + (uint64_t)rt;
                        rac->hash = (((rac->hash ^ (uint32_t)rt) * 16777619u) ^ (uint32_t)((uint64_t)rt >> 32)) * 16777619u;
                        int64_t bin = rt / P.rt_bin_ns;
                        if (bin > (int64_t)P.rt_bins - 1) bin = P.rt_bins - 1;
                        if (!CAL) atomicAdd(&agg[(uint64_t)cid * stride + 5 + bin], 1ull);
                        next_inst = true;
                    }
                }
                if (pc == PC_ARRIVE) {   // frame arrival / instance start (R6; R32: the thread's task)
                    URG_TR(t, TR_INST_START, lb_on ? cold_Ta[lane] : t_arr, 0);
                    if (!te) rac->total = rac->total + 1u;
                    if (T.inst_q) {   // words 0 (GPU) and 1 (CPU) of one Philox block (R4)
                        const uint4 w = rng_block(P.seed, s, URG_TAG_INST, cid, inst, 0);
                        Fg = inst_factor(w.x, CRF(gpu_sigma_ppm));
                        Fc = inst_factor(w.y, CRF(cpu_sigma_ppm));
                    }
                    rac->launches = rac->launches + (launched - k_first);   // the previous instance's launches
                    task = stage; launched = k_first; done = k_first; sync_ord = stage << 16;
                    if (!WIDE) nxt = kern_rec(KR + k_first);
                    rem_g = myvar[lane].gpu_est_total; rem_c = CRF(cpu_est_total);
                    if (lb_on) lb = cold_Ta[lane] + cold_Dp[lane] - rem_g - rem_c;
                    if (ma) {   // R26: this instance's ~E^cpu_j, floor mean of the last min(W, h_j) measurements
                        rem_c = 0;
                        for (uint32_t j = 0; j < CRF(num_tasks); ++j) {
                            const uint32_t h = ma_cnt[j];
                            uint32_t pred = T.task[tbase + j].cpu_estimate_ns;
                            if (h) {
                                const uint32_t k = h < P.ma_w ? h : P.ma_w;
                                uint64_t sum = 0;
                                for (uint32_t q = 0; q < k; ++q) sum += ma_ring[j * P.ma_w + (h - 1 - q) % P.ma_w];
                                pred = (uint32_t)(sum / k);
                            }
                            ma_pred[j] = pred;
                            rem_c += pred;
                        }
                    }
                    task_first = k_first; task_end = k_first + T.task[tbase + stage].num_kernels;
                    pc = PC_TASK_START;
                }
                if (pc == PC_TASK_START) {   // new CPU segment: evaluate, early exit
                    bool exited = false;
                    URG_TR(t, TR_TASK_START, task, 0);
                    if (urg) {
                        if (noise)
                            nz = (int32_t)(rng_word(P.seed, s, URG_TAG_NOISE, cid, inst, task) %
                                           (2u * P.noise_pm + 1u)) - (int32_t)P.noise_pm;
                        const int64_t lax = laxity(t);   // Eq. 2 (R9)
                        L_last = lax;
                        URG_TR(t, TR_EVAL, lax, launched);
                        if (f_early && lax < 0) {
                            URG_TR(t, TR_EARLY_EXIT, 0, 0);
                            akb = 0;
                            rac->early = rac->early + 1u;
                            if (last_stage) {   // R32: an earlier task's exit is a gap the last task records
                                rac->miss = rac->miss + 1u;
                                rac->hash = (((rac->hash ^ 0xFFFFFFFFu) * 16777619u) ^ 0xFFFFFFFFu) * 16777619u;
                                expect = inst + 1u;
                            }
                            pc = PC_DONE;
                            next_inst = exited = true;
                        }
                    }
                    if (!exited) {
                        const int64_t e = (int64_t)(((uint64_t)T.task[tbase + task].cpu_nominal_ns * Fc) >> 16);
                        if (ma) { ma_ring[task * P.ma_w + ma_cnt[task] % P.ma_w] = (uint32_t)e; ++ma_cnt[task]; }
                        if (cores_on && urg) rerank_req = true;   // R29: a CPU segment starts
                        pc = PC_CPU_DONE;
                        cpu_busy(t, e);
                        if (e > 0) break;
                    }
                }
                if (next_inst) {   // advance to the next instance of this chain (R6, R7)
                    if (te && stage > 0) {   // R32: the next message, or wait for one
                        if (msg) { take_msg(); continue; }
                        pc = PC_WAIT_MSG;
                        cpu_next = INF64; dc = D_INF;
                        break;
                    }
                    ++inst;
                    const int64_t ta = arrival(inst);
                    if (lb_on) cold_Ta[lane] = ta; else t_arr = ta;
                    if (ta >= H) { pc = PC_DONE; cpu_next = INF64; dc = D_INF; break; }   // not admitted
                    pc = PC_ARRIVE;
                    cpu_next = ta;
                    if (ta > t) { dc = dsat(ta - t); break; }
                    continue;
                }
                }
                if (pc == PC_ENQUEUE) {   // the kernel reaches its stream (R16) + sync decision (R17)
                    const uint32_t n = launched;
                    const UrgKernRec kr = WIDE ? kern_rec(KR + n) : nxt;
                    const int64_t est = kr.estimate_ns;
                    if (launched == done) {   // stream was empty: head now
                        head_ready = t; head_u = kr.util_permille; head_dur = head_duration(kr.nominal_ns, n); newhead = true;
                        if (has_copy) head_copy = kr.flags & 1u;
                    }
                    URG_TR(t, TR_ENQUEUE, n, level);
                    ++launched;
                    if (!WIDE && launched < CRF(num_kernels)) nxt = kern_rec(KR + launched);
                    rem_g -= est;
                    if (lb_on) lb += est;
                    if (akb_on) ++akb;
                    if (coll && (uint64_t)L_last < P.lth_excl) {
                        // R24: less urgent chains with a busy stream at the same or a higher priority
                        const int64_t own = urgency_key(L_last);
                        uint32_t mm = busy_m & ~lbit(), k = 0;
                        while (mm) {
                            const int o = __ffs(mm) - 1;
                            mm &= mm - 1;
                            k += (snapLev[o] <= level && urgency_key(snapL[o]) < own) ? 1u : 0u;
                        }
                        if (k && !CAL) atomicAdd(&agg[(uint64_t)NC * stride + (k + 1 > 32 ? 32 : k + 1)], 1ull);
                        if (k) URG_TR(t, TR_COLLISION, k + 1 > 32 ? 32 : k + 1, level);
                    }
                    const bool last = launched == task_end;
                    if (last) {
                        const uint32_t ce = ma ? ma_pred[task] : T.task[tbase + task].cpu_estimate_ns;
                        rem_c -= ce;
                        if (lb_on) lb += ce;
                    }
                    const uint32_t sm = P.sync_mode;
                    int32_t target = -1;
                    if (r17_sel) {
                        // R17 with selects (one rare branch): the estimate sum only matters in the
                        // batched modes; a batch closes when it reaches Delta_eval, crossing kernel included
                        if (n == task_first) batch_start = task_first;
                        const int64_t acc2 = (n == task_first ? 0 : acc) + est;
                        const bool closes = sm >= S_BATCHED && acc2 >= P.delta_eval_ns;
                        acc = (closes || last) ? 0 : acc2;
                        target = (last || sm == S_EACH || (closes && sm == S_BATCHED)) ? (int32_t)launched : -1;
                        if (closes && !last && sm == S_OVERLAP) {   // OVERLAP: wait for the previous batch
                            const uint32_t prev = batch_start;
                            batch_start = launched;
                            if (prev != task_first) target = (int32_t)prev;   // first close: not issued
#ifdef URG_DEBUG
                            else { URG_TR(t, TR_FREE_CLOSE, launched, 0); if (urg) URG_TR(t, TR_EVAL, laxity(t), launched); }
#endif
                        }
                    } else if (sm == S_ASYNC) {   // the other policies' benchmarks sync once per task
                        if (last) target = (int32_t)launched;
                    } else if (sm == S_EACH) {
                        target = (int32_t)launched;
                    } else {
                        if (n == task_first) { acc = 0; batch_start = task_first; }
                        acc += est;
                        const bool closes = acc >= P.delta_eval_ns;
                        if (closes || last) acc = 0;
                        if (last || (closes && sm == S_BATCHED)) target = (int32_t)launched;
                        else if (closes) {   // OVERLAP: wait for the previous batch
                            const uint32_t prev = batch_start;
                            batch_start = launched;
                            if (prev != task_first) target = (int32_t)prev;   // first close: not issued
#ifdef URG_DEBUG
                            else { URG_TR(t, TR_FREE_CLOSE, launched, 0); if (urg) URG_TR(t, TR_EVAL, laxity(t), launched); }
#endif
                        }
                    }
                    if (target >= 0) {
                        sync_target = (uint32_t)target;
                        sync_cost = (uint32_t)P.sync_lo_ns;
                        if (P.sync_hi_ns > P.sync_lo_ns) {
                            // the sync ordinals of an instance are drawn in order from (stage << 16), a
                            // multiple of 4: one Philox block serves four consecutive sync calls
                            if ((sync_ord & 3u) == 0u) syw[lane] = rng_block(P.seed, s, URG_TAG_SYNC, cid, inst, sync_ord);
                            sync_cost += (((const uint32_t *)&syw[lane])[sync_ord & 3u] %
                                                   (uint32_t)(P.sync_hi_ns - P.sync_lo_ns + 1));
                        }
                        ++sync_ord;
                        URG_TR(t, TR_SYNC_CALL, sync_target, sync_cost);
                        if (done >= sync_target) {
                            pc = PC_SYNC_RET;
                            cpu_busy(t, sync_cost);
                            if (sync_cost > 0) break;
                            continue;
                        }
                        pc = PC_SYNC_WAIT;
                        cpu_next = INF64; dc = D_INF;
                        break;
                    }
                    pc = PC_ATTEMPT;
                }
                if (pc == PC_CPU_DONE || pc == PC_ATTEMPT) {   // launch attempt for kernel n = launched (R14-R16)
                    int64_t lax = 0;
                    if (urg) { lax = laxity(t); L_last = lax; URG_TR(t, TR_EVAL, lax, launched); }
                    const bool own_urgent = (uint64_t)lax < P.lth_excl;   // R10: 0 <= L <= L_th
                    if (f_delay && !own_urgent && (urgent_m & ~lbit()) &&
                        (WIDE ? kern_rec(KR + launched) : nxt).util_permille >= P.util_exempt) {
                        URG_TR(t, TR_DELAY, launched, 0);
                        pc = PC_ATTEMPT;
                        cpu_next = t + P.sleep_ns;
                        dc = P.sleep_d32;
                        break;
                    }
                    if (launched == task_first) {   // task-level stream binding
                        if (KIND == K_STATIC) level = static_level;
                        else if (cls) {   // R27: rank among itself and the AKB-active chains
                            uint32_t mm = active_m & ~lbit();
                            const uint32_t n_r = 1 + __popc(mm);
                            const int64_t ownA = cls_key_a(), ownB = cls_key_b();
                            uint32_t r = 1;
                            while (mm) {
                                const int o = __ffs(mm) - 1;
                                mm &= mm - 1;
                                r += cls_before(snapA[o], snapB[o], o, ownA, ownB, lane, t) ? 1u : 0u;
                            }
                            level = P.num_prio <= 2 ? P.num_prio - 1
                                    : n_r <= 1      ? 1 + (P.num_prio - 2) / 2
                                                    : 1 + (uint32_t)(((uint64_t)(r - 1) * (P.num_prio - 2)) / (n_r - 1));
                        }
                        else if (!f_bind) level = P.num_prio - 1;
                        else if (own_urgent) level = 0;
                        else {
                            const int64_t own = urgency_key(lax);
                            uint32_t mm = active_m & ~lbit();
                            const uint32_t n_r = 1 + __popc(mm);
                            uint32_t r = 1;
                            while (mm) {
                                const int o = __ffs(mm) - 1;
                                mm &= mm - 1;
                                const int64_t k = urgency_key(snapL[o]);
                                r += (k > own || (k == own && o < lane)) ? 1u : 0u;
                            }
                            level = P.num_prio <= 2 ? P.num_prio - 1
                                    : n_r <= 1      ? 1 + (P.num_prio - 2) / 2
                                                    : 1 + (uint32_t)(((uint64_t)(r - 1) * (P.num_prio - 2)) / (n_r - 1));
                        }
                        URG_DASSERT(level < P.num_prio && (!f_bind || !own_urgent || level == 0), INV_LEVEL);
                        URG_TR(t, TR_BIND, level, launched);
                    }
                    pc = PC_ENQUEUE;
                    if (!cores_on || busy_launch == 0) { cpu_next = t + busy_launch; dc = P.busy_launch_d32; }
                    else cpu_busy(t, busy_launch);
                    if (bl_param ? P.busy_launch_d32 != 0u : busy_launch > 0) break;
                    continue;
                }
                break;   // PC_SYNC_WAIT / PC_DONE: nothing to do at t
            }
            return newhead;
        };
        // Round snapshot of the chains' (AKB non-empty, last laxity) for Phase B (R14, R15, R21).
        // `may_bind`: this lane can reach a task's first launch in this phase (else the
        // binding snapshot is not needed).
        auto snapshot = [&](bool may_bind, uint32_t &urgent_m, uint32_t &active_m, uint32_t &busy_m) {
            urgent_m = 0; active_m = 0; busy_m = 0;
            if (f_delay) urgent_m = __ballot_sync(FULL, akb > 0 && (uint64_t)L_last < P.lth_excl) & hmask;
            if (coll) {
                busy_m = __ballot_sync(FULL, launched > done) & hmask;
                active_m = __ballot_sync(FULL, akb > 0) & hmask;
                __syncwarp();   // the previous phase's reads of the snapshot are done
                snapL[lane] = L_last;
                snapLev[lane] = level;
                __syncwarp();
            } else if (f_bind && __any_sync(FULL, may_bind)) {
                active_m = __ballot_sync(FULL, akb > 0) & hmask;
                __syncwarp();
                snapL[lane] = L_last;
                __syncwarp();
            } else if (cls && __any_sync(FULL, may_bind)) {
                active_m = __ballot_sync(FULL, akb > 0) & hmask;
                __syncwarp();
                snapA[lane] = cls_key_a();
                snapB[lane] = cls_key_b();
                __syncwarp();
            }
        };
        // a due lane can bind in this phase unless it is mid-task and the launch cost
        // makes it yield before reaching the next task's first kernel
        auto can_bind = [&]() -> bool {
            return !((bl_param ? P.busy_launch_d32 != 0u : busy_launch > 0) && ((pc == PC_ENQUEUE && launched + 1 < task_end) ||
                                         (pc == PC_ATTEMPT && launched != task_first)));
        };

        // ---- A2-A10: the event loop (R21) ----
        // Warp-uniform: t_prev (time of the previous loop step) and `used`, the util
        // per-mille of the running kernels (kept incrementally).
        int64_t t_prev = -1;
        // fast-step budget: a step of m ns stays on the fast path iff 0 < m < budget, where budget =
        // min(2^30 - advance since the last exact refresh, H_stop - t_prev + 1) -- one compare covers
        // "time did not advance", "a distance may be inexact" and "past the end of the horizon"
        // kept as its end point lim = low 32 bits of (t_prev + budget), fixed between rare-path steps
        // (budget <= 2^30, so budget = lim - low 32 bits of t_prev): nothing to update on a fast step
        uint32_t lim = (uint32_t)-1 + (H_stop + 2 >= (int64_t)D_SLOW ? D_SLOW : (uint32_t)(H_stop + 2));   // t_prev = -1
        uint32_t used = 0;
        bool bar_prev = false;                  // R28: a barrier was pending at the previous step
        int64_t cal_next = 0;                   // CAL: next sampling time
        uint32_t cal_n = 0;                     // CAL: samples of this scenario
        bool fin = false;                       // PK: this half's scenario has ended
        uint32_t nsteps = 0;                    // PK: loop steps since the last rare-path step
        // Core UrgenGo build: the Phase B snapshot (R21) is taken where it changes -- at the
        // end of the previous Phase B, beside that phase's new-head vote -- instead of on the
        // next phase's critical path (Phase A and Phase C touch neither the AKB nor L_last).
        // At scenario start no lane has an AKB entry.
        constexpr bool snap_late = urg && !coll && !EXT;
        uint32_t urgent_nx = 0, active_nx = 0;
        for (;;) {
            // A2: next event time.  Each lane keeps 32-bit distances dc / dh of its next CPU event
            // and kernel end from t_prev (exact below 2^31, lower bounds above), so the step is one
            // REDUX of min(dc, dh) and a subtraction.  A distance of 0 (time did not advance), one
            // of 2^30 or more (a far lane may be nearer than it says), a drift of 2^30 since the
            // last refresh, or the end of the horizon take the rare path: the exact 64-bit
            // minimum, with every distance recomputed from it.
            int64_t t;
            bool bad = false;   // time did not advance (invariant)
            if constexpr (!URG_DIST_OFF) {   // (the 64-bit head below is kept for A/B: -DURG_NO_DIST)
                const uint32_t m = hmin(fin ? D_INF : (dc < dh ? dc : dh));
                t = (int64_t)((uint64_t)t_prev + m);   // (an ended half's t_prev may be INF64: wraps, unused)
                const bool slow = !fin && (m - 1u) >= (lim - (uint32_t)t_prev) - 1u;
                if (PK ? __any_sync(FULL, slow) : slow) {
                    t = hmin64(fin ? INF64 : (head_end < cpu_next ? head_end : cpu_next));
                    bad = !fin && t <= t_prev;
                    if (!fin && t != INF64) {
                        dc = cpu_next == INF64 ? D_INF : dsat(cpu_next - t);
                        dh = head_end == INF64 ? D_INF : dsat(head_end - t);
                    }
                    {
                        const int64_t hs = WIDE ? cold_Hs[lane] : H_stop;
                        const int64_t hb = hs - t + 1;
                        lim = (uint32_t)t + (hb >= (int64_t)D_SLOW ? D_SLOW : (hb < 1 ? 1u : (uint32_t)hb));
                    }
                    if (!PK && !CAL) {
                        if (t > H_stop) break;
                        if (bad) {   // report and stop this scenario
                            if (lane == 0 && atomicCAS((unsigned long long *)err, 0ull, (unsigned long long)ERR_TIME) == 0ull)
                                err[1] = s;
                            break;
                        }
                    }
                    if (PK) {   // each half ends on its own (only here: a fast step cannot end one)
                        if (!fin && lane == hbase) my_steps += nsteps;   // this half's steps so far
                        nsteps = 0;
                        if (bad && lane == hbase &&
                            atomicCAS((unsigned long long *)err, 0ull, (unsigned long long)ERR_TIME) == 0ull)
                            err[1] = s;
                        fin = fin || t > cold_Hs[lane] || bad;
                        if (fin) head_u = 0xFFFFu;   // an ended half dispatches nothing
                        if (__all_sync(FULL, fin)) break;
                    }
                } else {
                    dc -= m;
                    dh -= m;
                }
            } else {   // 64-bit next-event times; 32-bit distances from t_prev, saturated
                const int64_t mine = fin ? INF64 : (head_end < cpu_next ? head_end : cpu_next);
                const uint64_t dl = (uint64_t)mine - (uint64_t)t_prev;   // exact when mine > t_prev
                const uint32_t d32 = mine <= t_prev ? 0u : (dl >= 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)dl);
                const uint32_t m = hmin(d32);
                if (__any_sync(FULL, m == 0xFFFFFFFFu && !fin)) {
                    const int64_t tt = hmin64(mine);
                    t = m == 0xFFFFFFFFu ? tt : t_prev + m;
                } else t = t_prev + m;
                bad = !fin && m == 0u;
            }
            if (CAL && cal_next < P.cal_end && cal_next < t) {
                // the state between two steps is constant: one warp max of the AKB urgency
                // keys (order-preserving unsigned), then one sample per elapsed 1 ms tick
                const bool act = valid && akb > 0;
                const uint64_t u = act ? ((uint64_t)urgency_key(L_last) ^ 0x8000000000000000ull) : 0ull;
                const uint32_t mh = __reduce_max_sync(FULL, (uint32_t)(u >> 32));
                const uint32_t ml = __reduce_max_sync(FULL, (uint32_t)(u >> 32) == mh ? (uint32_t)u : 0u);
                const int64_t key = (int64_t)((((uint64_t)mh << 32) | ml) ^ 0x8000000000000000ull);
                const bool have = __any_sync(FULL, act);
                const bool keep = have && key >= 0;                   // skip none / negative laxity
                const int64_t bestL = key == INF64 ? 0 : ((int64_t)1 << 62) - key;
                for (; cal_next < P.cal_end && cal_next < t; cal_next += 1000000) {
                    if (keep) {
                        if (lane == 0 && cal_n < P.cal_cap) P.cal_buf[P.scenario_count + jw * P.cal_cap + cal_n] = bestL;
                        ++cal_n;
                    }
                }
            }
            if (CAL && cal_next >= P.cal_end) break;   // no sample left to take
            if (PK && URG_DIST_OFF) {   // each half ends on its own; the warp goes on while one half runs
                if (bad && lane == hbase &&
                    atomicCAS((unsigned long long *)err, 0ull, (unsigned long long)ERR_TIME) == 0ull)
                    err[1] = s;
                fin = fin || t > H_stop || bad;
                if (fin) head_u = 0xFFFFu;
                if (__all_sync(FULL, fin)) break;
            } else if (CAL) {
                if (t > H_stop) break;
                if (bad) {   // time must advance (invariant); report and stop this scenario
                    if (lane == 0 && atomicCAS((unsigned long long *)err, 0ull, (unsigned long long)ERR_TIME) == 0ull)
                        err[1] = s;
                    break;
                }
            }
            if (PK && !URG_DIST_OFF) {
                // every lane counts its half's loop steps in 32 bits; the count is moved into the
                // 64-bit total on the rare path (at most 2^30 ns of simulated time, hence fewer than
                // 2^30 steps, apart) while the half runs.  An ended half's t_prev is never read.
                t_prev = t;
                ++nsteps;
#ifdef URG_DEBUG
                if (!fin && lane == hbase) trace_row(t, TR_STEP, 0, 0);
#endif
            } else if (!fin) {
                t_prev = t;
                if (lane == hbase) ++my_steps;   // one loop step of this half's scenario
#ifdef URG_DEBUG
                if (lane == hbase) trace_row(t, TR_STEP, 0, 0);
#endif
            }

            // Phase A: retire (R21, R19)
            const bool ret = !fin && (URG_DIST_OFF ? head_end == t : dh == 0u);
            // The retire and due votes are issued together: a retirement makes its own lane due
            // at t only through a sync return of zero cost (retire(): cpu_busy(t, 0) sets cpu_next = t).
            // (bitwise operators: no short-circuit branches around the vote; measured +1.1 % configs[3],
            // +2.3 % configs[4], +0.8 % configs[1])
            const bool due_pre = !fin & ((URG_DIST_OFF ? cpu_next == t : dc == 0u) |
                                         (ret & (pc == PC_SYNC_WAIT) & (done + 1u >= sync_target) & (sync_cost == 0)));
            const uint32_t retm = __ballot_sync(FULL, ret), duem = __ballot_sync(FULL, due_pre);
            bool dirty = (retm & hmask) != 0u;   // GPU state changed: Phase C must run
            if (retm) {
                used -= hsum(ret ? head_util : 0u);
                if (ret) retire(t);
            }
            const bool due = !fin && (URG_DIST_OFF ? cpu_next == t : dc == 0u);   // == due_pre
            const bool any_due = duem != 0u;

            // Phase B: CPU steps of every chain due at t, against the round snapshot (R21)
            if (any_due) {
#ifdef URG_STATS
                ++st_multi;
#endif
                uint32_t urgent_m = urgent_nx, active_m = active_nx, busy_m = 0;
                if (!snap_late && (urg || cls)) snapshot(te || (due && can_bind()), urgent_m, active_m, busy_m);
                bool nh = false;
                if (due) nh = phase_b(t, urgent_m, active_m, busy_m);
                URG_DASSERT(!due || cpu_next > t, INV_PAST_EVENT);
                if (snap_late) {   // the next phase's snapshot: this lane's L_last and the two masks
                    if (f_bind) {
                        __syncwarp();   // this phase's reads of the snapshot are done
                        if (due) snapL[lane] = L_last;
                        __syncwarp();
                    }
                    const uint32_t nhm = c_always ? 0u : __ballot_sync(FULL, nh);
                    if (f_delay)
                        urgent_nx = __ballot_sync(FULL, akb > 0 && (uint64_t)L_last < P.lth_excl) & hmask;
                    if (f_bind) active_nx = __ballot_sync(FULL, akb > 0) & hmask;
                    dirty |= (nhm & hmask) != 0u;
                } else if (!c_always)
                    dirty |= PK ? hany(nh) : __any_sync(FULL, nh);
                // R32: messages published in a round are delivered at its end (a newer one replaces
                // an untaken one); threads waiting for one run in the next round, same t and read view
                while (te) {
                    __syncwarp();
                    const uint32_t pub = mbox[lane];
                    if (pub) { msg = pub; mbox[lane] = 0u; }
                    __syncwarp();
                    const bool wake = !fin && pc == PC_WAIT_MSG && msg != 0u;
                    if (!__any_sync(FULL, wake)) break;
                    bool nh2 = false;
                    if (wake) nh2 = phase_b(t, urgent_m, active_m, busy_m);
                    dirty |= __any_sync(FULL, nh2);
                }
            }


            // R29: CPU cores -- re-rank UrgenGo's priorities when a CPU segment started, then
            // give the cores to the first K runnable jobs by (priority, runnable since, chain)
            if (cores_on) {
                const bool rr = __any_sync(FULL, rerank_req);
                rerank_req = false;
                if (rr && urg && valid && pc != PC_ARRIVE && pc != PC_WAIT_MSG && pc != PC_DONE)
                    cpu_prio = urgency_key(laxity(t));
                if (rr || __any_sync(FULL, cpu_chg)) {
                    cpu_chg = false;
                    const uint32_t jm = __ballot_sync(FULL, job);
                    bool want = job;
                    if ((uint32_t)__popc(jm) > P.cpu_cores) {
                        const int64_t prio = KIND == K_STATIC ? -(int64_t)static_level : urg ? cpu_prio : 0;
                        __syncwarp();   // Phase B's reads of the snapshot slots are done
                        snapA[lane] = prio;
                        snapB[lane] = job_ready;
                        __syncwarp();
                        uint32_t better = 0, mm = jm & ~lbit();
                        while (mm) {
                            const int o = __ffs(mm) - 1;
                            mm &= mm - 1;
                            const int64_t po = snapA[o], ro = snapB[o];
                            better += (po > prio || (po == prio && (ro < job_ready || (ro == job_ready && o < lane)))) ? 1u : 0u;
                        }
                        want = job && better < P.cpu_cores;
                        __syncwarp();
                    }
                    if (want && !job_run) { job_run = true; run_start = t; cpu_next = t + job_rem; dc = dsat(job_rem); }
                    else if (job && !want && job_run) { job_run = false; job_rem -= t - run_start; cpu_next = INF64; dc = D_INF; }
                }
            }

            // cudaFree barriers (R28): while a request is queued or served nothing starts;
            // the (request time, chain)-first request is served once no kernel runs
            if (has_free) {
                const uint32_t fw = __ballot_sync(FULL, pc == PC_FREE_WAIT);
                const uint32_t fr = __ballot_sync(FULL, pc == PC_FREE_RET);
                if (fw | fr) {
                    bar_prev = true;
                    if (!fr && !__any_sync(FULL, head_end != INF64)) {
                        const bool w8 = (fw >> lane) & 1u;
                        const int64_t rq = w8 ? free_req : INF64;
                        const int64_t mrq = warp_min_nonneg(rq);
                        const int head = __ffs(__ballot_sync(FULL, w8 && free_req == mrq)) - 1;
                        if (lane == head) { pc = PC_FREE_RET; cpu_next = t + P.free_ns; dc = dsat(P.free_ns); }
                    }
                    continue;   // no dispatch during a barrier
                }
                if (bar_prev) { bar_prev = false; dirty = true; }   // released: waiting heads may start
            }

            // Phase C: dispatch waiting stream heads by (level, ready, chain) under capacity (R20).
            // Runs only when a kernel retired or a stream got a new head: otherwise every
            // waiting head was already found not to fit and `used` has not decreased.
            // The greedy scan in key order starts, each time, the smallest-key head that
            // fits the capacity left (heads that do not fit stay unfit as `used` grows).
            if (PK && (c_always || __any_sync(FULL, dirty))) {
                // both halves: a half that is not dirty has no head that fits (fit = 0); a lane with no
                // waiting head has head_u = 0xFFFF, which never fits
                for (;;) {
                    const uint32_t fitw = __ballot_sync(FULL, used + head_u <= 1000u);
                    if (!fitw) break;
                    const uint32_t fit = fitw & hmask;
                    // some half has two or more fitting heads: read off the (warp-uniform) ballot, no vote
                    const uint32_t f0 = fitw & 0xFFFFu, f1 = fitw >> 16;
                    const bool any_multi = ((f0 & (f0 - 1u)) | (f1 & (f1 - 1u))) != 0u;
                    int wl = fit ? __ffs(fit) - 1 : -1;
                    if (any_multi) {
                        const bool in = (fit >> lane) & 1u;
                        const uint64_t key = ((uint64_t)level << 56) | ((uint64_t)head_ready << 5) | (uint64_t)lane;
                        const uint32_t hi = in ? (uint32_t)(key >> 32) : 0xFFFFFFFFu;
                        const uint32_t mh = hmin(hi);
                        const uint32_t ml = hmin((in && hi == mh) ? (uint32_t)key : 0xFFFFFFFFu);
                        if (fit) wl = (int)(ml & 31u);
                    }
                    const uint32_t uw = __shfl_sync(FULL, head_u, wl >= 0 ? wl : lane);
                    if (lane == wl) start_head(t, used);
                    if (wl >= 0) used += uw;
                    URG_DASSERT(used <= 1000u, INV_CAPACITY);
                    if (!any_multi) break;   // each half started its only fitting head (others did not fit)
                }
            } else if (!PK && (c_always || dirty)) {
#ifdef URG_STATS
                ++st_dispatch;
#endif
                bool waiting = true;   // head_u = 0xFFFF (never fits) unless a head waits
                if (has_copy) {   // R31: the copy engine runs one memcpy at a time, (ready, chain) first
                    const bool cw = head_u != 0xFFFFu && head_copy;
                    if (__any_sync(FULL, cw) && !__any_sync(FULL, head_end != INF64 && head_copy)) {
                        const int64_t mr = warp_min_nonneg(cw ? head_ready : INF64);
                        const int wl = __ffs(__ballot_sync(FULL, cw && head_ready == mr)) - 1;
                        if (lane == wl) start_head(t, used);
                    }
                    waiting = !head_copy;   // memcpys never take compute capacity
                }
                for (;;) {
                    const uint32_t fit = __ballot_sync(FULL, waiting && used + head_u <= 1000u);
                    if (!fit) break;
                    int wl;
                    if ((fit & (fit - 1)) == 0) wl = __ffs(fit) - 1;
                    else {
                        const bool in = (fit >> lane) & 1u;
                        const uint64_t key = ((uint64_t)level << 56) | ((uint64_t)head_ready << 5) | (uint64_t)lane;
                        const uint32_t hi = in ? (uint32_t)(key >> 32) : 0xFFFFFFFFu;
                        const uint32_t mh = __reduce_min_sync(FULL, hi);
                        const uint32_t ml = __reduce_min_sync(FULL, (in && hi == mh) ? (uint32_t)key : 0xFFFFFFFFu);
                        wl = (int)(ml & 31u);
                    }
                    const uint32_t u_run = used;
                    used += __shfl_sync(FULL, head_u, wl);
                    URG_DASSERT(used <= 1000u, INV_CAPACITY);
                    if (lane == wl) start_head(t, u_run);
                    if ((fit & (fit - 1)) == 0) break;   // the others did not fit before; `used` only grew
                }
            }
        }

        if (CAL) {   // sample count of this scenario; no records or aggregates
            if (lane == 0) P.cal_buf[jw] = (int64_t)cal_n;
            continue;
        }
        // ---- A11: end of horizon accounting (R7) and per-scenario records ----
        uint32_t n_total = rac->total, n_miss = rac->miss, n_early = rac->early, n_unfin = rac->unfin,
                 hash = rac->hash;
        uint32_t n_launch = rac->launches + (launched - k_first);   // + the current instance's
        const uint64_t sum_rt = rac->sum_rt;
        if (te) {   // R32: the chain's early exits and launches, summed over its threads
            uint32_t e_sum = 0, l_sum = 0;
            for (uint32_t o = 0; o < C; ++o) {
                const uint32_t co = __shfl_sync(FULL, cid, (int)o);
                const uint32_t eo = __shfl_sync(FULL, n_early, (int)o), lo = __shfl_sync(FULL, n_launch, (int)o);
                if (co == cid) { e_sum += eo; l_sum += lo; }
            }
            if (valid && last_stage) { n_early = e_sum; n_launch = l_sum; }
            else n_launch = 0;   // counted once, on the chain's last stage (the warp's launch total)
        }
        if (valid && last_stage) {
            if (te) {   // R32: instances [0, expect) are recorded; later admitted ones are unfinished
                for (uint32_t i = expect; arrival(i) < H; ++i) ++n_unfin;
                n_total = expect + n_unfin;
            } else {
                uint32_t first_unstarted = inst;
                if (pc != PC_ARRIVE && pc != PC_DONE) { ++n_unfin; first_unstarted = inst + 1; }
                if (pc != PC_DONE)
                    for (uint32_t i = first_unstarted; arrival(i) < H; ++i) { ++n_unfin; ++n_total; }
            }
            n_miss += n_unfin;
            URG_DASSERT(n_miss <= n_total && n_early + n_unfin <= n_miss, INV_COUNTS);
            if (records) {
                uint4 *r = (uint4 *)(records + ((uint64_t)jw * NC + cid) * 8);
                r[0] = make_uint4(n_total, n_miss, n_early, n_unfin);
                r[1] = make_uint4(n_launch, hash, (uint32_t)sum_rt, (uint32_t)(sum_rt >> 32));
            }
            // A12: aggregates (integer sums: order-independent, R23)
            unsigned long long *a = agg + (uint64_t)cid * stride;
            atomicAdd(&a[0], (unsigned long long)n_total);
            atomicAdd(&a[1], (unsigned long long)n_miss);
            atomicAdd(&a[2], (unsigned long long)n_early);
            atomicAdd(&a[3], (unsigned long long)n_unfin);
            atomicAdd(&a[4], (unsigned long long)sum_rt);
            if (n_total) atomicAdd(&a[5 + P.rt_bins + (uint64_t)100 * n_miss / n_total], 1ull);
        }
        {   // the warp's launch events of this scenario (pair): one global add
            const uint32_t nl = __reduce_add_sync(FULL, n_launch);
            if (lane == 0 && nl) atomicAdd(&agg[(uint64_t)NC * stride + URG_COLL_BINS + 0], (unsigned long long)nl);
        }
    }
    if (PK) my_steps += __shfl_sync(FULL, my_steps, 16);   // the upper half's steps
    if (lane == 0) {
        if (CAL) return;
        atomicAdd(&agg[(uint64_t)NC * stride + URG_COLL_BINS + 1], my_steps);
#ifdef URG_STATS
        atomicAdd(&work[4], st_single); atomicAdd(&work[5], st_multi);
        atomicAdd(&work[6], st_dispatch); atomicAdd(&work[7], st_rebase);
#endif
    }
}


#undef busy_launch

// ---------------------------------------------------------------------------
// instantiation rows: 0 FIFO, 1 STATIC, 2 + f UrgenGo with flags f (0..15);
// columns: (per-kernel factor table) + 2 * (throughput build)
// ---------------------------------------------------------------------------
// rows 18 + f: the calibration build of UrgenGo with flags f (latency build only);
// rows 34..37: the classical policies EDF, SJF, HRRN, LCUF (R27)
#define URG_SIM_ROWS 38
template <int ROW>
struct UrgRow {
    static constexpr int K = ROW == 0 ? K_FIFO : ROW == 1 ? K_STATIC : ROW < 34 ? K_URGENGO : K_EDF + (ROW - 34);
    static constexpr int F = ROW < 2 || ROW >= 34 ? 0 : ROW < 18 ? ROW - 2 : ROW - 18;
    static constexpr bool C = ROW >= 18 && ROW < 34;
    // col: bit 0 per-kernel factor table, bit 1 throughput build, bit 2 extended model,
    // bit 3 two scenarios per warp (throughput core build only), bit 4 small latency core build
    static const void *get(uint32_t col)
    {
        if constexpr (!C) {
            if ((col & 30u) == 16u)   // bit 4: the small latency core build
                return (col & 1u) ? (const void *)urg_sim_kernel<K, F, true, false, false, false, false, true>
                                  : (const void *)urg_sim_kernel<K, F, false, false, false, false, false, true>;
            if ((col & 14u) == 10u)
                return (col & 1u) ? (const void *)urg_sim_kernel<K, F, true, true, false, false, true>
                                  : (const void *)urg_sim_kernel<K, F, false, true, false, false, true>;
        }
        if constexpr (C) {   // the calibration build: latency variant, extended model
            return (col & 1u) ? (const void *)urg_sim_kernel<K, F, true, false, true, true>
                              : (const void *)urg_sim_kernel<K, F, false, false, true, true>;
        } else {
            switch (col & 7u) {
            case 0: return (const void *)urg_sim_kernel<K, F, false, false, false, false>;
            case 1: return (const void *)urg_sim_kernel<K, F, true, false, false, false>;
            case 2: return (const void *)urg_sim_kernel<K, F, false, true, false, false>;
            case 3: return (const void *)urg_sim_kernel<K, F, true, true, false, false>;
            case 4: return (const void *)urg_sim_kernel<K, F, false, false, false, true>;
            case 5: return (const void *)urg_sim_kernel<K, F, true, false, false, true>;
            case 6: return (const void *)urg_sim_kernel<K, F, false, true, false, true>;
            default: return (const void *)urg_sim_kernel<K, F, true, true, false, true>;
            }
        }
    }
};
