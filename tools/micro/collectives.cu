// Latency of dependent warp collectives on sm_100a (one warp, chained ops, clock64).
#include <cstdio>
#include <cstdint>
#define N 4096
__global__ void k(uint32_t *out, long long *cyc, uint32_t seed)
{
    uint32_t v = threadIdx.x ^ seed;
    long long t0, t1;
    // REDUX.MIN chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = __reduce_min_sync(0xffffffffu, v + threadIdx.x) + 1;
    t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
    // VOTE.ANY chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) v += __any_sync(0xffffffffu, (v & 7) == threadIdx.x);
    t1 = clock64(); if (threadIdx.x == 0) cyc[1] = t1 - t0;
    // BALLOT chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) v += __ballot_sync(0xffffffffu, (v >> threadIdx.x) & 1);
    t1 = clock64(); if (threadIdx.x == 0) cyc[2] = t1 - t0;
    // SHFL chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
    t1 = clock64(); if (threadIdx.x == 0) cyc[3] = t1 - t0;
    // IADD chain (ALU reference)
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = v * 3 + (v >> 2);
    t1 = clock64(); if (threadIdx.x == 0) cyc[4] = t1 - t0;
    // 64-bit compare+select chain
    long long a = v, b = seed;
    t0 = clock64();
    for (int i = 0; i < N; ++i) { a = a < b ? a + 1 : b - 1; b ^= a; }
    t1 = clock64(); if (threadIdx.x == 0) cyc[5] = t1 - t0;
    // REDUX.SUM chain
    t0 = clock64();
    for (int i = 0; i < N; ++i) v = __reduce_add_sync(0xffffffffu, v & 0xff);
    t1 = clock64(); if (threadIdx.x == 0) cyc[6] = t1 - t0;
    // LDS chain
    __shared__ uint32_t sm[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = (i * 7 + 3) & 1023;
    __syncwarp();
    uint32_t p = threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < N; ++i) p = sm[p];
    t1 = clock64(); if (threadIdx.x == 0) cyc[7] = t1 - t0;
    out[threadIdx.x] = v + (uint32_t)a + (uint32_t)b + p;
}
int main()
{
    uint32_t *o; long long *c; cudaMalloc(&o, 128); cudaMalloc(&c, 64 * 8);
    k<<<1, 32>>>(o, c, 1); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 2); cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    const char *n[8] = {"REDUX.MIN", "VOTE.ANY", "BALLOT", "SHFL", "IMAD+SHF+IADD", "i64 cmp/sel/add/xor", "REDUX.SUM", "LDS chain"};
    for (int i = 0; i < 8; ++i) printf("%-22s %6.1f cycles/iter\n", n[i], (double)h[i] / N);
    return 0;
}
