// urg_sim.cu -- dispatch table of the simulation-kernel instantiations (the kernel itself
// is urg_sim.cuh, instantiated in parallel slices by urg_sim_part.cu) and the Philox
// known-answer test kernel.
#include "urg_sim.cuh"

extern "C" __global__ void urg_philox_kat_kernel(const uint4 *ctr, const uint2 *key, uint4 *out, int n)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = philox4x32_10(ctr[i], key[i]);
}


#define URG_PARTS 6
#define URG_DECL(k) const void *urg_sim_part##k(uint32_t row, uint32_t col);
URG_DECL(0) URG_DECL(1) URG_DECL(2) URG_DECL(3) URG_DECL(4) URG_DECL(5)
#undef URG_DECL

const void *urg_sim_kernel_for(uint32_t kind, uint32_t flags, bool kern_q, bool wide)
{
    const uint32_t row = kind == K_FIFO ? 0 : kind == K_STATIC ? 1 : 2 + (flags & 15u);
    const uint32_t col = (kern_q ? 1u : 0u) + (wide ? 2u : 0u);
    const void *(*parts[URG_PARTS])(uint32_t, uint32_t) = {urg_sim_part0, urg_sim_part1, urg_sim_part2,
                                                          urg_sim_part3, urg_sim_part4, urg_sim_part5};
    for (int k = 0; k < URG_PARTS; ++k)
        if (const void *f = parts[k](row, col)) return f;
    return nullptr;
}
