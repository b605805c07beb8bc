// Device template ("blob") layout and kernel parameters -- internal to liburg.so.
//
// The workload template is packed once on the host (urg_api.cu) into one
// 16-byte-aligned blob, copied to HBM at urg_create_workload, and staged whole
// into each CTA's shared memory by the simulation kernel (row A0).
#pragma once
#include <stdint.h>

#define URG_BLOB_MAGIC 0x55524731u   // "URG1"
#define URG_QTABLE 4096              // quantile-table entries (12-bit index)
#define URG_MAX_BLOB_BYTES (160u * 1024u)
#define URG_COLL_BINS 33             // aggregate: kernel-collision histogram bins (R24)
#define URG_SNAP_BYTES_PER_LANE 144u  // per lane: laxity, two policy keys (8 B each), level, mailbox (4 B each),
                                     // the template variant's two estimate totals (16 B), the lane's current
                                     // blocks of four per-kernel (R4) and four sync-cost (R5) Philox words,
                                     // P' and H_stop (8 B each, read on the rare path), t_arr and D'
                                     // (throughput UrgenGo build), the R22 record counters (32 B)

enum { URG_TAG_ARR = 1, URG_TAG_TIGHT = 2, URG_TAG_INST = 3, URG_TAG_KERN = 4, URG_TAG_SYNC = 5, URG_TAG_NOISE = 6 };

struct __align__(16) UrgChainRec {     // 80 B, one per thread (lane): a chain, or one task of it (R32)
    int64_t period_ns, deadline_ns, offset_ns;
    uint32_t num_tasks, task_base;     // the chain's tasks [task_base, task_base + num_tasks)
    uint32_t num_kernels, kern_base;   // the chain's kernels [kern_base, kern_base + num_kernels)
    uint32_t cpu_sigma_ppm, gpu_sigma_ppm;
    uint32_t chain_id;                 // chain of this thread (randomness, records)
    uint32_t stage, stage_end;         // tasks [stage, stage_end) it runs per instance
    uint32_t k_first;                  // chain-local index of the first kernel of task `stage`
    int64_t cpu_est_total;             // CPU estimates of tasks >= stage (Eq. 2 start value)
    int64_t pad_;
};

struct __align__(16) UrgVarRec {       // 16 B, per (template variant, thread), global memory (R33)
    int64_t gpu_est_total;             // kernel estimates of the variant from k_first on (Eq. 2 start value)
    int64_t gpu_est_chain;             // all kernel estimates of the chain in the variant (LCUF key, R27)
};

struct __align__(16) UrgTaskRec {      // 16 B
    uint32_t cpu_nominal_ns, cpu_estimate_ns, num_kernels, flags;   // flags bit 0: ends with cudaFree (R28)
};

struct __align__(16) UrgKernRec {      // 16 B: one LDS.128 per access
    uint32_t nominal_ns, estimate_ns, util_permille, flags;   // flags bit 0: memcpy (R31)
};

struct __align__(16) UrgBlobHeader {   // 64 B
    uint32_t magic, num_chains, num_tasks, num_kernels;
    uint32_t off_chains, off_tasks, off_kerns, off_inst_q;   // byte offsets; 0 = absent table
    uint32_t off_kern_q, total_bytes, reserved0, reserved1;
    uint32_t reserved[4];
};

struct UrgSimParams {
    // workload scalars
    uint32_t num_chains, num_prio, rt_bins, agg_stride;
    int64_t launch_ns, launch_akb_ns, sync_lo_ns, sync_hi_ns, jitter_ns, rt_bin_ns;
    // policy
    uint32_t kind, flags, sync_mode, util_exempt;
    int64_t delta_eval_ns, lax_threshold_ns, sleep_ns;
    // batch
    uint64_t seed, scenario_begin, scenario_count;
    int64_t horizon_ns;
    uint32_t fa_num, fa_den, fd_num, fd_den, ftight_permille, tight_explicit, tight_mask;
    // threads: num_lanes = num_chains, or the number of tasks with per-task executors (R32)
    uint32_t num_lanes, task_exec;
    // template variants (R33): [num_variants][nk_total] kernel records and [num_variants][num_lanes]
    // estimate totals, global memory
    const UrgKernRec *kern;
    const UrgVarRec *var;
    uint32_t nk_total, num_variants;
    // staging
    uint32_t blob_bytes, snap_offset, mbar_offset, smem_bytes;
    // estimation noise (R25) and CPU moving-average predictor (R26)
    uint32_t noise_pm, ma_w, ma_max_tasks, ma_slot, ma_offset;
    // cudaFree barriers (R28), CPU cores (R29)
    uint32_t has_free, cpu_cores, alpha_pm;   // + R30 contention alpha (per-mille)
    uint32_t has_copy;                        // R31: some operation is a memcpy
    int64_t free_ns;
    // TH_urgent calibration build only: sampling end, sample rows ([count] counts, then
    // [count][cal_cap] laxities)
    int64_t cal_end;
    int64_t *cal_buf;
    uint64_t cal_cap;
    // host-derived constants of the step loop: the launch call's busy time (lambda, + lambda_akb for
    // UrgenGo) and the delay sleep as saturated 32-bit distances, and R10 as one unsigned compare:
    // urgent(L) <=> (uint64_t)L < lth_excl (= L_th + 1, or 0 when L_th < 0: never urgent)
    int64_t busy_launch_ns;
    uint32_t busy_launch_d32, sleep_d32;
    uint64_t lth_excl;
    // debug build only (-DURG_DEBUG, liburg_debug.so): event trace of one scenario, [0] = row
    // counter, then rows (t, kind, chain, instance, a, b) in the oracle's trace schema
    int64_t *trace_buf;
    uint64_t trace_cap, trace_scn;
};
