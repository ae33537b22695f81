// Microbenchmark: dependent-chain latency (cycles) of the warp-collective and
// shared-memory operations the planner's step loop is built from.
#include <cstdio>
#include <cstdint>

__global__ void k(uint32_t *out, long long *cyc, int iters) {
    __shared__ uint32_t sm[1024];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i * 7) & 1023;
    __syncwarp();
    uint32_t v = lane;
    long long t0, t1;
    // 0: LDS chain
    t0 = clock64();
    for (int i = 0; i < iters; i++) v = sm[(v + lane) & 1023];
    t1 = clock64(); if (lane == 0) cyc[0] = (t1 - t0) / iters;
    // 1: SHFL chain
    t0 = clock64();
    for (int i = 0; i < iters; i++) v = __shfl_sync(0xffffffffu, v, (v + 1) & 31);
    t1 = clock64(); if (lane == 0) cyc[1] = (t1 - t0) / iters;
    // 2: REDUX chain
    t0 = clock64();
    for (int i = 0; i < iters; i++) v = __reduce_min_sync(0xffffffffu, v + lane);
    t1 = clock64(); if (lane == 0) cyc[2] = (t1 - t0) / iters;
    // 3: VOTE chain
    t0 = clock64();
    for (int i = 0; i < iters; i++) v = __ballot_sync(0xffffffffu, ((v >> lane) & 1) != 0) + lane;
    t1 = clock64(); if (lane == 0) cyc[3] = (t1 - t0) / iters;
    // 4: VOTE + FLO + SHFL (argmin broadcast idiom)
    t0 = clock64();
    for (int i = 0; i < iters; i++) {
        unsigned m = __ballot_sync(0xffffffffu, (v & 1) != 0);
        v = __shfl_sync(0xffffffffu, v + 1, __ffs(m | 1u) - 1);
    }
    t1 = clock64(); if (lane == 0) cyc[4] = (t1 - t0) / iters;
    // 5: syncwarp + STS/LDS round trip
    t0 = clock64();
    for (int i = 0; i < iters; i++) {
        sm[lane] = v; __syncwarp(); v = sm[(lane + 1) & 31] + 1; __syncwarp();
    }
    t1 = clock64(); if (lane == 0) cyc[5] = (t1 - t0) / iters;
    // 6: dependent IADD chain
    t0 = clock64();
    for (int i = 0; i < iters; i++) v = v * 3 + 1;
    t1 = clock64(); if (lane == 0) cyc[6] = (t1 - t0) / iters;
    // 7: 2x REDUX on u64 key (the warp_min idiom)
    unsigned long long kk = ((unsigned long long)v << 32) | lane;
    t0 = clock64();
    for (int i = 0; i < iters; i++) {
        const uint32_t a = __reduce_min_sync(0xffffffffu, (uint32_t)(kk >> 32));
        const uint32_t b = __reduce_min_sync(0xffffffffu, (uint32_t)(kk >> 32) == a ? (uint32_t)kk : 0xffffffffu);
        kk = (((unsigned long long)a << 32) | b) + lane;
    }
    t1 = clock64(); if (lane == 0) cyc[7] = (t1 - t0) / iters;
    // 8: global load chain (L1/L2 hit)
    t0 = clock64();
    for (int i = 0; i < iters; i++) v = out[(v + lane) & 1023];
    t1 = clock64(); if (lane == 0) cyc[8] = (t1 - t0) / iters;
    out[2048 + threadIdx.x] = v + (uint32_t)kk;
}

int main() {
    uint32_t *out; long long *cyc;
    cudaMalloc(&out, 8192 * 4); cudaMalloc(&cyc, 64 * 8);
    uint32_t h[1024]; for (int i = 0; i < 1024; i++) h[i] = (i * 13) & 1023;
    cudaMemcpy(out, h, 4096, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(out, cyc, 1000);
    k<<<1, 32>>>(out, cyc, 1000);
    long long c[9]; cudaMemcpy(c, cyc, 9 * 8, cudaMemcpyDeviceToHost);
    const char *nm[9] = {"LDS", "SHFL", "REDUX", "VOTE", "VOTE+FLO+SHFL", "STS+syncwarp+LDS+syncwarp",
                         "IMAD", "2xREDUX u64 min", "LDG (L1 hit)"};
    for (int i = 0; i < 9; i++) printf("%-28s %lld cycles\n", nm[i], c[i]);
    return 0;
}
