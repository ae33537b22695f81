// Microbenchmark: per-step synchronisation cost of a planner step spread over
// a CTA or a thread-block cluster (design study for the register-resident
// scan engine).  Each iteration models one best-fit step:
//   leader publishes (lo, hi) -> every thread tests K register-resident
//   blocks -> warp REDUX -> CTA reduce -> (cluster: result to the leader)
//   -> leader derives the next (lo, hi).
// Variants:
//   cta  <NT>      one CTA, two __syncthreads per step
//   clu  <CL, NT>  CL CTAs in a cluster; requests / responses through DSMEM
//                  stores + mbarrier arrivals (release/acquire at cluster
//                  scope), CTA reduce inside each CTA
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>

namespace cg = cooperative_groups;

constexpr int K = 8;

__device__ __forceinline__ uint32_t eval_blocks(const uint32_t (&a)[K], const uint32_t (&f)[K],
                                                const uint32_t (&p)[K], uint32_t lo, uint32_t hi) {
    uint32_t best = 0xFFFFFFFFu;
#pragma unroll
    for (int k = 0; k < K; k++) best = (a[k] >= lo && f[k] <= hi) ? min(best, p[k]) : best;
    return best;
}

template <int NT>
__global__ void __launch_bounds__(NT) k_cta(int iters, unsigned long long *cyc, uint32_t *sink) {
    __shared__ uint32_t req[2];
    __shared__ uint32_t wres[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t a[K], f[K], p[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
        a[k] = (tid * K + k) * 7u % 1000u;
        f[k] = a[k] + 1 + (tid * 13u + k) % 50u;
        p[k] = (tid * K + k) * 2654435761u >> 12;
    }
    if (tid == 0) { req[0] = 0; req[1] = 500; }
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        const uint32_t lo = req[0], hi = req[1];
        const uint32_t b = __reduce_min_sync(0xFFFFFFFFu, eval_blocks(a, f, p, lo, hi));
        if (lane == 0) wres[warp] = b;
        __syncthreads();
        if (warp == 0) {
            const uint32_t g = __reduce_min_sync(0xFFFFFFFFu, lane < NT / 32 ? wres[lane] : ~0u);
            if (lane == 0) { req[0] = (g + it) % 900u; req[1] = req[0] + 100u; }
        }
        __syncthreads();
    }
    const long long t1 = clock64();
    if (tid == 0) { cyc[blockIdx.x] = t1 - t0; sink[blockIdx.x] = req[0]; }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
// arrive (release, cluster scope) on the barrier at the same smem offset in
// CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint64_t *bar, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;"
            " selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void st_remote_u32(uint32_t *p, uint32_t rank, uint32_t v) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(p)), "r"(rank));
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(remote), "r"(v) : "memory");
}

template <int CL, int NT>
__global__ void __launch_bounds__(NT) k_clu(int iters, unsigned long long *cyc, uint32_t *sink) {
    __shared__ uint32_t req[2];
    __shared__ uint32_t wres[32];
    __shared__ uint32_t cres[CL];
    __shared__ __align__(8) uint64_t bar_req, bar_rsp;
    cg::cluster_group cluster = cg::this_cluster();
    const uint32_t rank = cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t a[K], f[K], p[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
        const uint32_t g = (rank * NT + tid) * K + k;
        a[k] = g * 7u % 1000u;
        f[k] = a[k] + 1 + (g * 13u) % 50u;
        p[k] = g * 2654435761u >> 12;
    }
    if (tid == 0) {
        mbar_init(&bar_req, 1);
        mbar_init(&bar_rsp, CL);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster.sync();
    uint32_t lo = 0, hi = 500;
    const long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        const uint32_t par = it & 1;
        if (rank == 0 && tid == 0) {
            // publish the request to every CTA (including this one)
            for (uint32_t r = 0; r < CL; r++) {
                st_remote_u32(&req[0], r, lo);
                st_remote_u32(&req[1], r, hi);
                mbar_arrive_remote(&bar_req, r);
            }
        }
        mbar_wait(&bar_req, par);
        const uint32_t l2 = req[0], h2 = req[1];
        const uint32_t b = __reduce_min_sync(0xFFFFFFFFu, eval_blocks(a, f, p, l2, h2));
        if (lane == 0) wres[warp] = b;
        __syncthreads();
        if (warp == 0) {
            const uint32_t g = __reduce_min_sync(0xFFFFFFFFu, lane < NT / 32 ? wres[lane] : ~0u);
            if (lane == 0) {
                st_remote_u32(&cres[rank], 0, g);
                mbar_arrive_remote(&bar_rsp, 0);
            }
        }
        if (rank == 0 && warp == 0) {
            mbar_wait(&bar_rsp, par);
            const uint32_t g = __reduce_min_sync(0xFFFFFFFFu, lane < CL ? cres[lane] : ~0u);
            lo = (g + it) % 900u;
            hi = lo + 100u;
        }
        __syncthreads();  // wres reuse
    }
    const long long t1 = clock64();
    if (tid == 0) { cyc[blockIdx.x] = t1 - t0; sink[blockIdx.x] = lo; }
    cluster.sync();
}

template <typename F>
static double run(F launch, int ctas, int iters, unsigned long long *cyc) {
    launch(iters / 10 + 1);
    launch(iters);
    cudaDeviceSynchronize();
    unsigned long long h[64];
    cudaMemcpy(h, cyc, sizeof(unsigned long long) * ctas, cudaMemcpyDeviceToHost);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return -1; }
    return (double)h[0] / iters;
}

template <int CL, int NT>
static void clu(int iters, unsigned long long *cyc, uint32_t *sink) {
    cudaFuncSetAttribute(k_clu<CL, NT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    auto L = [&](int n) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(CL);
        cfg.blockDim = dim3(NT);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_clu<CL, NT>, n, cyc, sink);
    };
    printf("cluster CL=%2d NT=%4d: %.1f cycles/step\n", CL, NT, run(L, CL, iters, cyc));
}

int main() {
    unsigned long long *cyc;
    uint32_t *sink;
    cudaMalloc(&cyc, 64 * 8);
    cudaMalloc(&sink, 64 * 4);
    const int it = 20000;
    printf("cta NT=  32: %.1f cycles/step\n", run([&](int n) { k_cta<32><<<1, 32>>>(n, cyc, sink); }, 1, it, cyc));
    printf("cta NT= 128: %.1f cycles/step\n", run([&](int n) { k_cta<128><<<1, 128>>>(n, cyc, sink); }, 1, it, cyc));
    printf("cta NT= 256: %.1f cycles/step\n", run([&](int n) { k_cta<256><<<1, 256>>>(n, cyc, sink); }, 1, it, cyc));
    printf("cta NT= 512: %.1f cycles/step\n", run([&](int n) { k_cta<512><<<1, 512>>>(n, cyc, sink); }, 1, it, cyc));
    printf("cta NT=1024: %.1f cycles/step\n", run([&](int n) { k_cta<1024><<<1, 1024>>>(n, cyc, sink); }, 1, it, cyc));
    clu<2, 1024>(it, cyc, sink);
    clu<4, 1024>(it, cyc, sink);
    clu<8, 1024>(it, cyc, sink);
    clu<16, 1024>(it, cyc, sink);
    clu<8, 256>(it, cyc, sink);
    clu<16, 256>(it, cyc, sink);
    return 0;
}
