// Step-latency floor of the best-fit loop on this GPU (SURVEY.md §8(d):
// "the step-latency floor S x t_step,min ... measured by a microbenchmark").
//
// Every step of solve_bestfit (bestfit.py:295-308) is a dependent chain:
//   choose  R3 argmin over the skyline lines   (bestfit.py:115-122)
//   query   R4 best contained block             (bestfit.py:243-262)
//   update  R5/R6 splice of the line list       (bestfit.py:149-201)
// and step k+1's choice depends on step k's update.  The minimal chain one
// warp can run per step, whatever the data structure, is modelled here:
//   choose: one LDS of a line key per lane, REDUX min, VOTE + FLO, SHFL;
//   query : one dependent load of a table entry at an address derived from
//           the choice — from global memory (variant "l2": a 16 MB table,
//           random addresses, so L1 misses and L2 hits, as for the 10^5-block
//           window tables) or shared memory (variant "smem": traces whose
//           tables fit an SM) — then REDUX min over the lanes (the winner);
//   update: STS of the new line + __syncwarp.
// One warp per CTA; `ctas_per_sm` CTAs per SM (148 SMs) give the batched
// throughput ceiling with that many traces resident per SM.
//
// Built by __graft_entry__.build() into tools/ubench/libstepfloor.so and
// called by bench.py (live, on the same GPU as the bench) through
//   int step_floor(int variant, int ctas, int iters,
//                  double *cyc_per_step, double *steps_per_s);
#include <cstdint>
#include <cstdio>

#include <cuda_runtime.h>

namespace {

constexpr int kTableWords = 4 << 20;  // 16 MB of u32

template <bool L2>
__global__ void __launch_bounds__(32) k_step(const uint32_t *__restrict__ table, int iters,
                                             unsigned long long *cyc, uint32_t *sink) {
    __shared__ uint32_t lines[64];
    __shared__ uint32_t stab[8192];
    const int lane = threadIdx.x;
    lines[lane] = (lane * 2654435761u) >> 8;
    lines[32 + lane] = 0;
    for (int i = lane; i < 8192; i += 32) stab[i] = (i * 40503u) & 0xFFFFu;
    __syncwarp();
    uint32_t state = blockIdx.x * 977u + 1;
    const long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        // choose: argmin of the line keys, leftmost lane at the minimum
        const uint32_t key = lines[lane] ^ (state & 0xFFu);
        const uint32_t kmin = __reduce_min_sync(0xFFFFFFFFu, key);
        const int c = __ffs(__ballot_sync(0xFFFFFFFFu, key == kmin)) - 1;
        const uint32_t lo = __shfl_sync(0xFFFFFFFFu, key + state, c);
        // query: one dependent table read per lane, then the warp winner
        uint32_t v;
        if (L2) {
            const uint32_t idx = ((lo * 2654435761u) ^ (uint32_t)(lane * 4099)) & (kTableWords - 1);
            v = table[idx];
        } else {
            v = stab[(lo + lane * 131u) & 8191u];
        }
        const uint32_t best = __reduce_min_sync(0xFFFFFFFFu, v);
        // update: write the replacement line
        if (lane == (int)(best & 31u)) lines[c] = best + it;
        __syncwarp();
        state = best + 1;
    }
    const long long t1 = clock64();
    if (lane == 0) {
        cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
        sink[blockIdx.x] = state;
    }
}

}  // namespace

extern "C" int step_floor(int variant, int ctas, int iters, double *cyc_per_step,
                          double *steps_per_s) {
    uint32_t *table = nullptr, *sink = nullptr;
    unsigned long long *cyc = nullptr;
    if (cudaMalloc(&table, sizeof(uint32_t) * kTableWords) != cudaSuccess) return 1;
    cudaMalloc(&sink, sizeof(uint32_t) * ctas);
    cudaMalloc(&cyc, sizeof(unsigned long long) * ctas);
    cudaMemset(table, 0x5A, sizeof(uint32_t) * kTableWords);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto launch = [&](int n) {
        if (variant == 0) k_step<true><<<ctas, 32>>>(table, n, cyc, sink);
        else k_step<false><<<ctas, 32>>>(table, n, cyc, sink);
    };
    launch(iters / 10 + 1);  // warm the table into L2
    cudaEventRecord(e0);
    launch(iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long *h = new unsigned long long[ctas];
    cudaMemcpy(h, cyc, sizeof(unsigned long long) * ctas, cudaMemcpyDeviceToHost);
    double sum = 0;
    for (int i = 0; i < ctas; i++) sum += (double)h[i];
    delete[] h;
    *cyc_per_step = sum / ctas / iters;
    *steps_per_s = (double)ctas * iters / (ms * 1e-3);
    const cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(table);
    cudaFree(sink);
    cudaFree(cyc);
    return err == cudaSuccess ? 0 : 2;
}

#ifdef STEP_FLOOR_MAIN
int main() {
    for (int v = 0; v < 2; v++)
        for (int c : {1, 148, 148 * 8, 148 * 16, 148 * 32}) {
            double cyc, sps;
            step_floor(v, c, 20000, &cyc, &sps);
            printf("%s ctas=%d: %.1f cycles/step/warp, %.3g steps/s\n", v ? "smem" : "l2", c, cyc,
                   sps);
        }
    return 0;
}
#endif
