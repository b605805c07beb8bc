// urg_sim.cu -- dispatch table of the simulation-kernel instantiations (the kernel itself
// is urg_sim.cuh, instantiated in parallel slices by urg_sim_part.cu) and the Philox
// known-answer test kernel.
#include "urg_sim.cuh"

extern "C" __global__ void urg_philox_kat_kernel(const uint4 *ctr, const uint2 *key, uint4 *out, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = philox4x32_10(ctr[i], key[i]);
}


#define URG_PARTS 13   // build.py PARTS
#define URG_DECL(k) const void *urg_sim_part##k(uint32_t row, uint32_t col);
URG_DECL(0) URG_DECL(1) URG_DECL(2) URG_DECL(3) URG_DECL(4) URG_DECL(5) URG_DECL(6) URG_DECL(7) URG_DECL(8)
URG_DECL(9) URG_DECL(10) URG_DECL(11) URG_DECL(12)
#undef URG_DECL

const void *urg_sim_kernel_for(uint32_t kind, uint32_t flags, bool kern_q, bool wide, bool cal, bool ext, bool pk,
                               bool small)
{
    const uint32_t row = cal                ? 18 + (flags & 15u)
                         : kind == K_FIFO    ? 0
                         : kind == K_STATIC  ? 1
                         : kind == K_URGENGO ? 2 + (flags & 15u)
                                             : 34 + (kind - K_EDF);
    const uint32_t col = (kern_q ? 1u : 0u) + (wide ? 2u : 0u) + (ext ? 4u : 0u) + (pk ? 8u : 0u) + (small ? 16u : 0u);
    const void *(*parts[URG_PARTS])(uint32_t, uint32_t) = {urg_sim_part0, urg_sim_part1, urg_sim_part2,
                                                          urg_sim_part3, urg_sim_part4, urg_sim_part5,
                                                          urg_sim_part6, urg_sim_part7, urg_sim_part8,
                                                          urg_sim_part9, urg_sim_part10, urg_sim_part11,
                                                          urg_sim_part12};
    for (int k = 0; k < URG_PARTS; ++k)
        if (const void *f = parts[k](row, col)) return f;
    return nullptr;
}

// ---------------------------------------------------------------------------
// TH_urgent: exact nearest-rank selection over the calibration samples
// (Q5).  The k-th smallest urgency key, k = floor(95 m / 100)
// + 1, found by an 8-pass radix select on the order-preserving unsigned key (8 bits
// per pass, most significant first): each pass histograms the samples matching the
// prefix found so far, then one thread picks the byte holding rank k.
// ws layout (int64): [0,256) histogram, [256] prefix, [257] mask, [258] k remaining, [259] m
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t cal_ukey(int64_t L) { return (uint64_t)urgency_key(L) ^ 0x8000000000000000ull; }

extern "C" __global__ void urg_cal_hist_kernel(const int64_t *buf, uint64_t count, uint64_t cap, long long *ws, int pass)
{
    __shared__ unsigned long long h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint64_t prefix = (uint64_t)ws[256], mask = (uint64_t)ws[257];
    const int shift = 8 * pass;
    for (uint64_t j = blockIdx.x; j < count; j += gridDim.x) {
        const uint64_t n = (uint64_t)buf[j];
        const int64_t *row = buf + count + j * cap;
        for (uint64_t i = threadIdx.x; i < n && i < cap; i += blockDim.x) {
            const uint64_t u = cal_ukey(row[i]);
            if ((u & mask) == prefix) atomicAdd(&h[(u >> shift) & 0xFFu], 1ull);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (h[i]) atomicAdd((unsigned long long *)&ws[i], h[i]);
}

extern "C" __global__ void urg_cal_pick_kernel(long long *ws, int pass, int pct, long long *result)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (pass == 7) {   // first pass: every sample matched; m and the rank k
        long long m = 0;
        for (int b = 0; b < 256; ++b) m += ws[b];
        long long k = (long long)pct * m / 100 + 1;
        if (k > m) k = m;
        ws[259] = m;
        ws[258] = k;
    }
    long long k = ws[258], cum = 0;
    int bsel = 255;
    for (int b = 0; b < 256; ++b) {
        if (cum + ws[b] >= k) { bsel = b; break; }
        cum += ws[b];
    }
    const int shift = 8 * pass;
    ws[256] = (long long)((uint64_t)ws[256] | ((uint64_t)bsel << shift));
    ws[257] = (long long)((uint64_t)ws[257] | (0xFFull << shift));
    ws[258] = k - cum;
    for (int b = 0; b < 256; ++b) ws[b] = 0;
    if (pass == 0) {   // the selected key -> its laxity (keys of kept samples are >= 0)
        const long long m = ws[259];
        if (m == 0) { result[0] = -1; result[1] = 0; return; }
        const int64_t key = (int64_t)((uint64_t)ws[256] ^ 0x8000000000000000ull);
        result[0] = key == INF64 ? 0 : ((int64_t)1 << 62) - key;
        result[1] = m;
    }
}
