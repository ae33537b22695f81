// K0 — planner pre-pass on the device: compressed time ranks, (alloc, id)
// order, priority ranks, and the packed tables K1/K2 read.
//
// Replaces _RemainingBlocks.__init__ (bestfit.py:231-241: sort by
// (alloc, id), int64 columns) and the implicit key of take_best
// (bestfit.py:250-256: lifetime, then size, then smaller id).
//
// Batched form: T traces in CSR (trace_ptr).  Every sort is a stable CUB
// radix sort; the per-trace grouping is restored by a final stable sort on
// the trace index (LSD order), so a single pass handles one or many traces.
#include <cub/block/block_scan.cuh>
#include <cub/cub.cuh>

#include <stdlib.h>

#include <algorithm>

#include "common.h"
#include "plan_types.cuh"
#include "prep.h"

namespace mp {

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t n) {
    int64_t g = (n + kThreads - 1) / kThreads;
    return (int)(g < 1 ? 1 : (g > (1 << 30) ? (1 << 30) : g));
}

__global__ void k_trace_index(const int64_t *__restrict__ trace_ptr, int64_t T,
                              uint32_t *__restrict__ tix, int64_t N) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = T;  // last t with trace_ptr[t] <= i
        while (hi - lo > 1) {
            int64_t mid = (lo + hi) >> 1;
            if (trace_ptr[mid] <= i) lo = mid; else hi = mid;
        }
        tix[i] = (uint32_t)lo;
    }
}

// times[0..N) = alloc, times[N..2N) = free; idx = iota
__global__ void k_fill_times(const int64_t *__restrict__ alloc, const int64_t *__restrict__ free_,
                             int64_t N, int64_t *__restrict__ times, uint32_t *__restrict__ idx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * N;
         i += (int64_t)gridDim.x * blockDim.x) {
        times[i] = i < N ? alloc[i] : free_[i - N];
        idx[i] = (uint32_t)i;
    }
}

__global__ void k_gather_tkey(const uint32_t *__restrict__ idx, const uint32_t *__restrict__ tix,
                              int64_t N, int64_t M, uint32_t *__restrict__ tkey) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = idx[i];
        tkey[i] = tix[v < N ? v : v - N];
    }
}

// flag = 1 where a new (trace, time) group starts in sorted order
__global__ void k_rank_flags(const uint32_t *__restrict__ idx, const int64_t *__restrict__ alloc,
                             const int64_t *__restrict__ free_, const uint32_t *__restrict__ tix,
                             int64_t N, uint32_t *__restrict__ flags) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * N;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = idx[i];
        int64_t tv = v < N ? alloc[v] : free_[v - N];
        uint32_t tt = tix[v < N ? v : v - N];
        uint32_t f = 1;
        if (i > 0) {
            uint32_t u = idx[i - 1];
            int64_t tu = u < N ? alloc[u] : free_[u - N];
            uint32_t tu_t = tix[u < N ? u : u - N];
            f = (tu != tv || tu_t != tt) ? 1u : 0u;
        }
        flags[i] = f;
    }
}

// local rank = inclusive scan - scan at the trace's first sorted element
__global__ void k_rank_scatter(const uint32_t *__restrict__ idx, const uint32_t *__restrict__ scan,
                               const uint32_t *__restrict__ tix,
                               const int64_t *__restrict__ trace_ptr, int64_t N,
                               uint32_t *__restrict__ arank, uint32_t *__restrict__ frank) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * N;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = idx[i];
        int64_t k = v < N ? v : v - N;
        uint32_t t = tix[k];
        uint32_t r = scan[i] - scan[2 * trace_ptr[t]];
        if (v < N) arank[k] = r; else frank[k] = r;
    }
}

__global__ void k_trace_U(const uint32_t *__restrict__ scan, const int64_t *__restrict__ trace_ptr,
                          int64_t T, uint32_t *__restrict__ U) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t a = trace_ptr[t], b = trace_ptr[t + 1];
        U[t] = b > a ? scan[2 * b - 1] - scan[2 * a] + 1 : 0;
    }
}

__global__ void k_iota_keys_arank(const uint32_t *__restrict__ arank, int64_t N,
                                  uint32_t *__restrict__ keys, uint32_t *__restrict__ vals) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = arank[i];
        vals[i] = (uint32_t)i;
    }
}

// descending size / lifetime as ascending complemented unsigned keys
__global__ void k_keys_size(const int64_t *__restrict__ size, int64_t N,
                            uint64_t *__restrict__ keys, uint32_t *__restrict__ vals) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = ~(uint64_t)size[i];
        vals[i] = (uint32_t)i;
    }
}

__global__ void k_keys_life(const uint32_t *__restrict__ vals, const int64_t *__restrict__ alloc,
                            const int64_t *__restrict__ free_, int64_t N,
                            uint64_t *__restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t k = vals[i];
        keys[i] = ~(uint64_t)(free_[k] - alloc[k]);
    }
}

__global__ void k_gather_tix32(const uint32_t *__restrict__ vals, const uint32_t *__restrict__ tix,
                               int64_t N, uint32_t *__restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        keys[i] = tix[vals[i]];
}

// order[p] = k for global position p; write pos/prio inverse maps
__global__ void k_inverse(const uint32_t *__restrict__ order, const uint32_t *__restrict__ tix,
                          const int64_t *__restrict__ trace_ptr, int64_t N,
                          uint32_t *__restrict__ inv) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < N;
         p += (int64_t)gridDim.x * blockDim.x) {
        uint32_t k = order[p];
        inv[k] = (uint32_t)(p - trace_ptr[tix[k]]);
    }
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t *v, uint32_t n, uint32_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (v[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// sorted alloc ranks per position, for the apos/fpos binary searches
__global__ void k_sorted_arank(const uint32_t *__restrict__ order, const uint32_t *__restrict__ arank,
                               int64_t N, uint32_t *__restrict__ sar) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < N;
         p += (int64_t)gridDim.x * blockDim.x)
        sar[p] = arank[order[p]];
}

// LOP table per trace: lop[off_t + r] = first (alloc, id)-position whose
// alloc rank is >= r, for r in [0, U_t] — built by one pass over the sorted
// alloc ranks (each position writes the ranks since its predecessor's), so
// k_pack reads apos/fpos with one load each instead of two binary searches.
// off_t = sum over earlier traces of (U + 1): one block scans the T values.
__global__ void __launch_bounds__(1024) k_lop_offsets(const uint32_t *__restrict__ U, int64_t T,
                                                      uint64_t *__restrict__ off) {
    using BS = cub::BlockScan<uint64_t, 1024>;
    __shared__ typename BS::TempStorage tmp;
    const int64_t per = (T + 1023) / 1024;
    const int64_t lo = threadIdx.x * per, hi = T < lo + per ? T : lo + per;
    uint64_t sum = 0;
    for (int64_t t = lo; t < hi; t++) sum += (uint64_t)U[t] + 1u;
    uint64_t pre = 0, total = 0;
    BS(tmp).ExclusiveSum(sum, pre, total);
    for (int64_t t = lo; t < hi; t++) {
        off[t] = pre;
        pre += (uint64_t)U[t] + 1u;
    }
    if (threadIdx.x == 0) off[T] = total;
}

__global__ void k_lop_fill(const uint32_t *__restrict__ tix, const int64_t *__restrict__ trace_ptr,
                           const uint32_t *__restrict__ sar, const uint32_t *__restrict__ U,
                           const uint64_t *__restrict__ off, int64_t N, uint32_t *__restrict__ lop) {
    for (int64_t P = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; P < N;
         P += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t t = tix[P];
        const int64_t b = trace_ptr[t];
        const uint32_t p = (uint32_t)(P - b), n = (uint32_t)(trace_ptr[t + 1] - b);
        uint32_t *L = lop + off[t];
        const uint32_t cur = sar[P];
        const uint32_t first = p ? sar[P - 1] + 1u : 0u;  // ranks (prev, cur]
        for (uint32_t r = first; r <= cur; r++) L[r] = p;
        if (p + 1 == n)
            for (uint32_t r = cur + 1; r <= U[t]; r++) L[r] = n;
    }
}

__device__ __forceinline__ int64_t gcd64(int64_t a, int64_t b) {
    while (b) {
        int64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

// Per-trace size unit g = gcd(sizes) and total bytes in units (saturating).
// Every skyline height is a sum of sizes, hence a multiple of g; when the
// total is below 2^32 units the planner runs on 32-bit heights and packs
// (height, lo) into one 64-bit argmin key.
//
// Also the trace's time origin tmin = min alloc and span = max free - tmin:
// raw times relative to tmin feed the planner's lifetime-bound pruning,
// which is enabled when the span fits 31 bits.
__global__ void k_trace_scale(const int64_t *__restrict__ trace_ptr,
                              const int64_t *__restrict__ size, const int64_t *__restrict__ alloc,
                              const int64_t *__restrict__ free_, int64_t *__restrict__ unit,
                              uint64_t *__restrict__ total_units, int64_t *__restrict__ tmin,
                              int64_t *__restrict__ tspan) {
    __shared__ int64_t sg[32];
    __shared__ uint64_t ss[32];
    __shared__ int64_t smn[32], smx[32];
    const int64_t t = blockIdx.x;
    const int64_t b = trace_ptr[t], e = trace_ptr[t + 1];
    {
        int64_t mn = INT64_MAX, mx = INT64_MIN;
        for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
            mn = min(mn, alloc[i]);
            mx = max(mx, free_[i]);
        }
        for (int o = 16; o; o >>= 1) {
            mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
            mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
        }
        if ((threadIdx.x & 31) == 0) { smn[threadIdx.x >> 5] = mn; smx[threadIdx.x >> 5] = mx; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); w++) {
                mn = min(mn, smn[w]);
                mx = max(mx, smx[w]);
            }
            tmin[t] = e > b ? mn : 0;
            // overflow-safe span (times are arbitrary int64 ticks)
            const uint64_t sp = (uint64_t)mx - (uint64_t)mn;
            tspan[t] = e > b ? (sp > (uint64_t)INT64_MAX ? INT64_MAX : (int64_t)sp) : 0;
        }
    }
    int64_t g = 0;
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) g = gcd64(size[i], g);
    for (int o = 16; o; o >>= 1) g = gcd64(g, __shfl_xor_sync(0xFFFFFFFFu, g, o));
    if ((threadIdx.x & 31) == 0) sg[threadIdx.x >> 5] = g;
    __syncthreads();
    if (threadIdx.x < 32) {
        g = threadIdx.x < (blockDim.x >> 5) ? sg[threadIdx.x] : 0;
        for (int o = 16; o; o >>= 1) g = gcd64(g, __shfl_xor_sync(0xFFFFFFFFu, g, o));
        if (threadIdx.x == 0) sg[0] = g > 0 ? g : 1;
    }
    __syncthreads();
    g = sg[0];
    const uint64_t cap = uint64_t(1) << 62;
    uint64_t acc = 0;
    for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
        acc += (uint64_t)(size[i] / g);
        if (acc > cap) acc = cap;
    }
    for (int o = 16; o; o >>= 1) {
        acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
        if (acc > cap) acc = cap;
    }
    if ((threadIdx.x & 31) == 0) ss[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t tot = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            tot += ss[w];
            if (tot > cap) tot = cap;
        }
        unit[t] = g;
        total_units[t] = tot;
    }
}

__global__ void k_pack(const uint32_t *__restrict__ tix, const int64_t *__restrict__ trace_ptr,
                       const uint32_t *__restrict__ arank, const uint32_t *__restrict__ frank,
                       const uint32_t *__restrict__ posof, const uint32_t *__restrict__ prio,
                       const uint32_t *__restrict__ sar, const int64_t *__restrict__ size,
                       const int64_t *__restrict__ unit, const int64_t *__restrict__ alloc,
                       const int64_t *__restrict__ free_, const int64_t *__restrict__ tmin,
                       int64_t N, uint2 *__restrict__ ent, Rec *__restrict__ rec,
                       uint2 *__restrict__ raw2, uint32_t *__restrict__ rawpos,
                       const uint32_t *__restrict__ lop, const uint64_t *__restrict__ off) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        uint32_t t = tix[k];
        int64_t b = trace_ptr[t];
        uint32_t n = (uint32_t)(trace_ptr[t + 1] - b);
        const uint32_t *s = sar + b;
        Rec r;
        r.pos = posof[k];
        r.arank = arank[k];
        r.frank = frank[k];
        if (lop) {  // LOP table (k_lop_fill)
            const uint32_t *L = lop + off[t];
            r.apos = L[r.arank];
            r.fpos = L[r.frank];
        } else {
            r.apos = lower_bound_u32(s, n, r.arank);
            r.fpos = lower_bound_u32(s, n, r.frank);
        }
        r.k = (uint32_t)(k - b);
        r.size = size[k] / unit[t];  // in units of the trace's size gcd
        rec[b + prio[k]] = r;
        ent[b + r.pos] = make_uint2(r.frank, prio[k]);
        // raw times relative to the trace origin (meaningful when span < 2^31)
        const uint32_t ra = (uint32_t)(alloc[k] - tmin[t]), rf = (uint32_t)(free_[k] - tmin[t]);
        raw2[b + prio[k]] = make_uint2(ra, rf);
        rawpos[b + r.pos] = ra;
    }
}

// One warp per chunk: bitonic-sort the chunk's 32 (free rank, slot) keys,
// emit SF/SP, the chunk skeleton and the live count.
__global__ void k_chunk_sort(const int64_t *__restrict__ trace_ptr, int64_t T,
                             const uint2 *__restrict__ ent, uint32_t *__restrict__ sf,
                             uint32_t *__restrict__ sp, uint4 *__restrict__ s0,
                             uint4 *__restrict__ s1, uint2 *__restrict__ s2,
                             const uint32_t *__restrict__ rawpos,
                             uint32_t *__restrict__ cnt, int64_t nchunks) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t cg = warp; cg < nchunks; cg += nw) {
        // owning trace: last t with chunk_base(trace_ptr[t], t) <= cg
        int64_t lo = 0, hi = T;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (chunk_base(trace_ptr[mid], mid) <= cg) lo = mid; else hi = mid;
        }
        const int64_t t = lo, b = trace_ptr[t], n = trace_ptr[t + 1] - b;
        const int64_t j = cg - chunk_base(b, t);
        uint32_t key = 0xFFFFFFFFu, pr = kDead;
        if (j < ((n + 31) >> 5)) {  // else: gap chunk between traces (never read)
            const int64_t p = 32 * j + lane;
            if (p < n) {
                const uint2 e = ent[b + p];
                key = (e.x << 5) | (uint32_t)lane;
                pr = e.y;
            }
        }
        // bitonic sort ascending by key across the warp (payload pr)
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (int jj = k >> 1; jj > 0; jj >>= 1) {
                const uint32_t ok = __shfl_xor_sync(0xFFFFFFFFu, key, jj);
                const uint32_t op = __shfl_xor_sync(0xFFFFFFFFu, pr, jj);
                const bool up = ((lane & k) == 0);
                const bool lower = ((lane & jj) == 0);
                const bool take = (lower == up) ? ok < key : ok > key;
                if (take) { key = ok; pr = op; }
            }
        }
        sf[32 * cg + lane] = key;
        sp[32 * cg + lane] = pr;
        const uint32_t nlive = skel_store(key, pr, lane, s0, s1, s2, cg);
        if (lane == 0 && j < ((n + 31) >> 5)) s2[cg].y = rawpos[b + 32 * j];
        if (lane == 0) cnt[cg] = nlive;
    }
}

// One warp per group of 32 chunks: the group skeleton (plan_types.cuh).
__global__ void k_group_skel(const int64_t *__restrict__ trace_ptr, int64_t T,
                             const uint4 *__restrict__ s0, const uint32_t *__restrict__ rawpos,
                             uint4 *__restrict__ gs, int64_t ngroups) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t gg = warp; gg < ngroups; gg += nw) {
        int64_t lo = 0, hi = T;  // owning trace: last t with group_base <= gg
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (group_base(trace_ptr[mid], mid) <= gg) lo = mid; else hi = mid;
        }
        const int64_t t = lo, b = trace_ptr[t], n = trace_ptr[t + 1] - b;
        const int64_t nch = (n + 31) >> 5, g = gg - group_base(b, t);
        if (g >= ((nch + 31) >> 5)) {  // gap group between traces (never read)
            if (lane == 0) gs[gg] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0u);
            continue;
        }
        group_store(s0 + chunk_base(b, t), nch, gs + group_base(b, t), g, lane);
        __syncwarp();
        // GS.w: relative raw alloc time of the group's first position
        if (lane == 0) gs[gg].w = rawpos[b + 1024 * g];
    }
}

// Batch-wide key ranges for the composite-key sorts: [0] min alloc,
// [1] max free, [2] max lifetime, [3] max size, [4] OR of all sizes (its
// trailing zeros divide every size: dropped from the priority key).
__global__ void k_ranges(const int64_t *__restrict__ alloc, const int64_t *__restrict__ free_,
                         const int64_t *__restrict__ size, int64_t N,
                         unsigned long long *__restrict__ out) {
    int64_t mn = INT64_MAX, mx = INT64_MIN, ml = 0, ms = 0;
    unsigned long long so = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        mn = min(mn, alloc[i]);
        mx = max(mx, free_[i]);
        ml = max(ml, free_[i] - alloc[i]);
        ms = max(ms, size[i]);
        so |= (unsigned long long)size[i];
    }
    for (int o = 16; o; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
        ml = max(ml, __shfl_xor_sync(0xFFFFFFFFu, ml, o));
        ms = max(ms, __shfl_xor_sync(0xFFFFFFFFu, ms, o));
        so |= __shfl_xor_sync(0xFFFFFFFFu, so, o);
    }
    if ((threadIdx.x & 31) == 0) {
        // order-preserving unsigned images of the signed values
        atomicMin(out + 0, (unsigned long long)mn ^ 0x8000000000000000ull);
        atomicMax(out + 1, (unsigned long long)mx ^ 0x8000000000000000ull);
        atomicMax(out + 2, (unsigned long long)ml);
        atomicMax(out + 3, (unsigned long long)ms);
        atomicOr(out + 4, so);
    }
}

// Raw-time ranks: when the batch's time span fits kRankBits - 1 bits, the
// time relative to the trace's first alloc is already an order-preserving
// rank that fits the window keys, so the rank compression (one sort of all
// 2N times, flags, scan, scatter) is skipped.  The best-fit loop only
// compares times (bestfit.py:115-122, :157, :215), so any strictly
// monotone relabelling gives the same plan.
__global__ void k_raw_ranks(const int64_t *__restrict__ alloc, const int64_t *__restrict__ free_,
                            const uint32_t *__restrict__ tix, const int64_t *__restrict__ tmin,
                            int64_t N, uint32_t *__restrict__ arank, uint32_t *__restrict__ frank) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = tmin[tix[i]];
        arank[i] = (uint32_t)(alloc[i] - m);
        frank[i] = (uint32_t)(free_[i] - m);
    }
}

// U = rank of the trace's last time + 1 (the sentinel line's lo is U - 1).
__global__ void k_raw_U(const int64_t *__restrict__ trace_ptr, const int64_t *__restrict__ tspan,
                        int64_t T, uint32_t *__restrict__ U) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T;
         t += (int64_t)gridDim.x * blockDim.x)
        U[t] = trace_ptr[t + 1] > trace_ptr[t] ? (uint32_t)tspan[t] + 1u : 0u;
}

// composite (trace, time - tmin) keys over alloc ∪ free; idx = iota
__global__ void k_time_keys(const int64_t *__restrict__ alloc, const int64_t *__restrict__ free_,
                            const uint32_t *__restrict__ tix, int64_t N, int64_t tmin, int tbits,
                            uint64_t *__restrict__ keys, uint32_t *__restrict__ idx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * N;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i < N ? i : i - N;
        const int64_t t = i < N ? alloc[k] : free_[k];
        keys[i] = ((uint64_t)tix[k] << tbits) | (uint64_t)(t - tmin);
        idx[i] = (uint32_t)i;
    }
}

// composite (trace, alloc rank) keys
__global__ void k_arank_keys(const uint32_t *__restrict__ arank, const uint32_t *__restrict__ tix,
                             int64_t N, int rbits, uint32_t *__restrict__ keys,
                             uint32_t *__restrict__ vals) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = (tix[i] << rbits) | arank[i];
        vals[i] = (uint32_t)i;
    }
}

// composite (trace, lifetime desc, size desc) keys; ids ascend by stability
__global__ void k_prio_keys(const int64_t *__restrict__ alloc, const int64_t *__restrict__ free_,
                            const int64_t *__restrict__ size, const uint32_t *__restrict__ tix,
                            int64_t N, int lbits, int sbits, int sshift, uint64_t lmax,
                            uint64_t smax, uint64_t *__restrict__ keys,
                            uint32_t *__restrict__ vals) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t life = (uint64_t)(free_[i] - alloc[i]), sz = (uint64_t)size[i];
        keys[i] = ((uint64_t)tix[i] << (lbits + sbits)) | ((lmax - life) << sbits) |
                  ((smax - sz) >> sshift);
        vals[i] = (uint32_t)i;
    }
}

inline int bits_for_u64(uint64_t v) {  // bits to hold 0..v
    int b = 0;
    while (b < 64 && (v >> b)) b++;
    return b;
}

inline int bits_for(int64_t T) {
    int b = 1;
    while ((int64_t(1) << b) < T) b++;
    return b;
}

}  // namespace

size_t prep_scratch_bytes(int64_t N, int64_t T) {
    size_t M = (size_t)2 * N;
    size_t b = 0;
    b += Carver::need<uint32_t>(N);         // tix
    b += Carver::need<int64_t>(M) * 2;      // times in/out
    b += Carver::need<uint32_t>(M) * 2;     // idx in/out
    b += Carver::need<uint32_t>(M) * 2;     // tkeys / flags+scan (reused)
    b += Carver::need<uint32_t>(N) * 6;     // arank frank posof prio sar order
    b += Carver::need<uint64_t>(N) * 2;     // 64-bit keys in/out
    // CUB temp: radix sort of M pairs + scan of M items
    size_t t1 = 0, t2 = 0, t3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, (const int64_t *)nullptr, (int64_t *)nullptr,
                                    (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)M);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                    (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)M);
    cub::DeviceScan::InclusiveSum(nullptr, t3, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                  (int)M);
    size_t tmax = t1 > t2 ? t1 : t2;
    tmax = tmax > t3 ? tmax : t3;
    b += Carver::need<char>(tmax);
    b += Carver::need<uint32_t>(T);  // U
    return b + 4096;
}

thread_local int g_prep_k = 0;
int prep_launches() { return g_prep_k; }

int prep_run(const PrepIn &in, PrepOut &out, void *scratch, size_t scratch_bytes,
             cudaStream_t s) {
    const int64_t N = in.N, T = in.T, M = 2 * N;
    if (N == 0) {
        if (T > 0) {
            MP_CUDA(cudaMemsetAsync(out.U, 0, sizeof(uint32_t) * T, s));
            MP_CUDA(cudaMemsetAsync(out.total_units, 0, sizeof(uint64_t) * T, s));
        }
        return MP_OK;
    }
    if (M >= (int64_t(1) << 31)) {
        set_error("batch too large for 32-bit ranks");
        return MP_ERR_INVALID;
    }
    g_prep_k = 0;
    Carver cv(scratch, scratch_bytes);
    uint32_t *tix = cv.take<uint32_t>(N);
    int64_t *times = cv.take<int64_t>(M), *times_s = cv.take<int64_t>(M);
    uint32_t *idx = cv.take<uint32_t>(M), *idx_s = cv.take<uint32_t>(M);
    uint32_t *tk = cv.take<uint32_t>(M), *tk_s = cv.take<uint32_t>(M);
    uint32_t *arank = cv.take<uint32_t>(N), *frank = cv.take<uint32_t>(N);
    uint32_t *posof = cv.take<uint32_t>(N), *prio = cv.take<uint32_t>(N);
    uint32_t *sar = cv.take<uint32_t>(N), *order = cv.take<uint32_t>(N);
    uint64_t *k64 = cv.take<uint64_t>(N), *k64_s = cv.take<uint64_t>(N);
    size_t tbytes = 0;
    {
        size_t t1 = 0, t2 = 0, t3 = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, t1, (const int64_t *)nullptr, (int64_t *)nullptr,
                                        (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)M);
        cub::DeviceRadixSort::SortPairs(nullptr, t2, (const uint64_t *)nullptr,
                                        (uint64_t *)nullptr, (const uint32_t *)nullptr,
                                        (uint32_t *)nullptr, (int)M);
        cub::DeviceScan::InclusiveSum(nullptr, t3, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                      (int)M);
        tbytes = t1 > t2 ? t1 : t2;
        tbytes = tbytes > t3 ? tbytes : t3;
    }
    void *tmp = cv.take<char>(tbytes);
    if (cv.off > cv.cap) {
        set_error("prep scratch too small");
        return MP_ERR_CUDA;
    }
    const int tb = bits_for(T);
    const int g1 = grid_for(N), g2 = grid_for(M);

    k_trace_index<<<g1, kThreads, 0, s>>>(in.trace_ptr, T, tix, N);
    g_prep_k++;

    // Large batches: one composite-key sort per ordering instead of a full
    // 64-bit sort plus a stable regroup by trace, with the key widths cut to
    // the batch's actual ranges (one small reduction + one host sync).
    bool comp = false, raw = false;
    int tbits = 0, lbits = 0, sbits = 0, sshift = 0;
    uint64_t lmax = 0, smax = 0;
    int64_t tmin = 0;
    if (T > 1 && N >= (int64_t(1) << 16)) {
        unsigned long long *rng = reinterpret_cast<unsigned long long *>(k64_s);
        const unsigned long long init[5] = {~0ull, 0ull, 0ull, 0ull, 0ull};
        MP_CUDA(cudaMemcpyAsync(rng, init, sizeof(init), cudaMemcpyHostToDevice, s));
        k_ranges<<<std::min(g1, 148 * 8), kThreads, 0, s>>>(in.alloc, in.free_, in.size, N, rng);
        g_prep_k++;
        unsigned long long h[5];
        MP_CUDA(cudaMemcpyAsync(h, rng, sizeof(h), cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
        tmin = (int64_t)(h[0] ^ 0x8000000000000000ull);
        const int64_t tmax = (int64_t)(h[1] ^ 0x8000000000000000ull);
        const uint64_t span = (uint64_t)tmax - (uint64_t)tmin;
        tbits = bits_for_u64(span);
        lmax = h[2];
        smax = h[3];
        sshift = h[4] ? __builtin_ctzll(h[4]) : 0;
        lbits = bits_for_u64(lmax);
        sbits = bits_for_u64(smax >> sshift);
        comp = tb + tbits <= 64 && tb + lbits + sbits <= 64 && tmax >= tmin;
        raw = comp && tbits < kRankBits - 1 && !getenv("MEMPLAN_DENSE_RANKS");
    }
    // ---- compressed time ranks over alloc ∪ free, per trace ----
    size_t tb_ = tbytes;
    uint32_t *rk_idx = idx_s;
    if (raw) {
        k_trace_scale<<<(unsigned)T, kThreads, 0, s>>>(in.trace_ptr, in.size, in.alloc, in.free_,
                                                      out.unit, out.total_units, out.tmin,
                                                      out.tspan);
        g_prep_k++;
        k_raw_ranks<<<g1, kThreads, 0, s>>>(in.alloc, in.free_, tix, out.tmin, N, arank, frank);
        g_prep_k++;
        k_raw_U<<<grid_for(T), kThreads, 0, s>>>(in.trace_ptr, out.tspan, T, out.U);
        g_prep_k++;
    } else {
    if (comp) {
        uint64_t *tk64 = reinterpret_cast<uint64_t *>(times), *tk64_s = reinterpret_cast<uint64_t *>(times_s);
        k_time_keys<<<g2, kThreads, 0, s>>>(in.alloc, in.free_, tix, N, tmin, tbits, tk64, idx);
        g_prep_k++;
        MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb_, tk64, tk64_s, idx, idx_s, (int)M, 0,
                                                tb + tbits, s));
    } else {
        k_fill_times<<<g2, kThreads, 0, s>>>(in.alloc, in.free_, N, times, idx);
        g_prep_k++;
        MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb_, times, times_s, idx, idx_s, (int)M, 0, 64,
                                                s));
    }
    if (!comp && T > 1) {
        k_gather_tkey<<<g2, kThreads, 0, s>>>(idx_s, tix, N, M, tk);
        g_prep_k++;
        tb_ = tbytes;
        MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb_, tk, tk_s, idx_s, idx, (int)M, 0, tb, s));
        rk_idx = idx;
    }
    uint32_t *flags = tk, *scan = tk_s;
    k_rank_flags<<<g2, kThreads, 0, s>>>(rk_idx, in.alloc, in.free_, tix, N, flags);
    g_prep_k++;
    tb_ = tbytes;
    MP_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb_, flags, scan, (int)M, s));
    k_rank_scatter<<<g2, kThreads, 0, s>>>(rk_idx, scan, tix, in.trace_ptr, N, arank, frank);
    g_prep_k++;
    k_trace_U<<<grid_for(T), kThreads, 0, s>>>(scan, in.trace_ptr, T, out.U);
    g_prep_k++;
    }

    // ---- (alloc, id) order: stable by alloc rank, then stable by trace ----
    uint32_t *ka = tk, *ka_s = tk_s, *va = idx, *va_s = idx_s;
    // ranks < 2n+1 per trace (dense) or <= the batch's time span (raw)
    const int rbits = raw ? std::max(1, tbits) : bits_for_u64((uint64_t)(2 * N + 2));
    const bool comp32 = comp && tb + rbits <= 32;
    if (comp32) {
        k_arank_keys<<<g1, kThreads, 0, s>>>(arank, tix, N, rbits, ka, va);
        g_prep_k++;
        tb_ = tbytes;
        MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb_, ka, ka_s, va, va_s, (int)N, 0,
                                                tb + rbits, s));
    } else {
        k_iota_keys_arank<<<g1, kThreads, 0, s>>>(arank, N, ka, va);
        g_prep_k++;
        tb_ = tbytes;
        MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb_, ka, ka_s, va, va_s, (int)N, 0, 32, s));
    }
    uint32_t *ord = va_s;
    if (!comp32 && T > 1) {
        k_gather_tix32<<<g1, kThreads, 0, s>>>(va_s, tix, N, ka);
        g_prep_k++;
        tb_ = tbytes;
        MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb_, ka, ka_s, va_s, va, (int)N, 0, tb, s));
        ord = va;
    }
    MP_CUDA(cudaMemcpyAsync(order, ord, sizeof(uint32_t) * N, cudaMemcpyDeviceToDevice, s));
    k_inverse<<<g1, kThreads, 0, s>>>(order, tix, in.trace_ptr, N, posof);
    g_prep_k++;
    k_sorted_arank<<<g1, kThreads, 0, s>>>(order, arank, N, sar);
    g_prep_k++;

    // ---- priority order: stable size desc, then stable lifetime desc, then trace ----
    uint32_t *vp = idx, *vp_s = idx_s;
    uint32_t *pord = nullptr;
    if (comp) {
        k_prio_keys<<<g1, kThreads, 0, s>>>(in.alloc, in.free_, in.size, tix, N, lbits, sbits,
                                            sshift, lmax, smax, k64, vp);
        g_prep_k++;
        tb_ = tbytes;
        MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb_, k64, k64_s, vp, vp_s, (int)N, 0,
                                                tb + lbits + sbits, s));
        pord = vp_s;
    } else {
    k_keys_size<<<g1, kThreads, 0, s>>>(in.size, N, k64, vp);
    g_prep_k++;
    tb_ = tbytes;
    MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb_, k64, k64_s, vp, vp_s, (int)N, 0, 64, s));
    k_keys_life<<<g1, kThreads, 0, s>>>(vp_s, in.alloc, in.free_, N, k64);
    g_prep_k++;
    tb_ = tbytes;
    MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb_, k64, k64_s, vp_s, vp, (int)N, 0, 64, s));
    pord = vp;
    if (T > 1) {
        k_gather_tix32<<<g1, kThreads, 0, s>>>(vp, tix, N, tk);
        g_prep_k++;
        tb_ = tbytes;
        MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb_, tk, tk_s, vp, vp_s, (int)N, 0, tb, s));
        pord = vp_s;
    }
    }
    k_inverse<<<g1, kThreads, 0, s>>>(pord, tix, in.trace_ptr, N, prio);
    g_prep_k++;

    if (!raw) {
        k_trace_scale<<<(unsigned)T, kThreads, 0, s>>>(in.trace_ptr, in.size, in.alloc, in.free_,
                                                      out.unit, out.total_units, out.tmin,
                                                      out.tspan);
        g_prep_k++;
    }
    // LOP table in the dead time-sort buffers (times + times_s: 8N words)
    // when the ranks span at most ~4 per block (dense ranks: U <= 2n; raw
    // ranks: U = time span + 1) — else the binary searches
    uint32_t *lop = nullptr;
    const uint64_t *loff = nullptr;
    if (T + 1 <= N && !getenv("MEMPLAN_NO_LOP")) {
        uint64_t *offd = k64_s;
        k_lop_offsets<<<1, 1024, 0, s>>>(out.U, T, offd);
        g_prep_k++;
        uint64_t total = 0;
        MP_CUDA(cudaMemcpyAsync(&total, offd + T, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
        if (total <= (uint64_t)(8 * N)) {
            lop = reinterpret_cast<uint32_t *>(times);  // times_s follows contiguously
            loff = offd;
            k_lop_fill<<<g1, kThreads, 0, s>>>(tix, in.trace_ptr, sar, out.U, offd, N, lop);
            g_prep_k++;
        }
    }
    k_pack<<<g1, kThreads, 0, s>>>(tix, in.trace_ptr, arank, frank, posof, prio, sar, in.size,
                                   out.unit, in.alloc, in.free_, out.tmin, N, out.ent, out.rec,
                                   out.raw2, out.rawpos, lop, loff);
    g_prep_k++;
    if (out.sf) {
        const int64_t chunks = out.nchunks;
        const int blocks = (int)std::min<int64_t>((chunks + 7) / 8, 148 * 64);
        k_chunk_sort<<<blocks, 256, 0, s>>>(in.trace_ptr, T, out.ent, out.sf, out.sp, out.s0,
                                            out.s1, out.s2, out.rawpos, out.cnt, chunks);
        g_prep_k++;
        const int gblocks = (int)std::min<int64_t>((out.ngroups + 7) / 8, 148 * 64);
        k_group_skel<<<gblocks, 256, 0, s>>>(in.trace_ptr, T, out.s0, out.rawpos, out.gs,
                                             out.ngroups);
        g_prep_k++;
    }
    MP_CUDA(cudaGetLastError());
    return MP_OK;
}

}  // namespace mp
