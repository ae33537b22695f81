// K0 for one small trace inside one CTA (the fused small-trace path).
//
// Same outputs as prep_run (prep.cu) restricted to what the TIER_SCAN
// planner reads — compressed time ranks, the (alloc, id) order, priority
// ranks (lifetime desc, size desc, id asc: bestfit.py:216, :250-256), the
// winner records, raw times, the chunk-sorted table rows and the per-trace
// scalars — but computed by one CTA with block-wide radix sorts in shared
// memory instead of device-wide sorts, so a batch of small traces (or one
// single small trace) needs one launch and no host round trip before
// planning.  Included by plan.cu only.
#pragma once
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

namespace mp {

constexpr int kFusedMaxThreads = 256;

struct FusedIn {
    const int64_t *alloc, *free_, *size;  // batch columns (device)
    uint2 *ent;                           // window entries in (alloc, id) order (TIER_WARP)
    int64_t *unit, *tmin, *tspan;         // per trace outputs
    uint64_t *total_units;
    uint32_t *U;
};

__device__ __forceinline__ int64_t gcd64f(int64_t a, int64_t b) {
    while (b) {
        const int64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

__device__ __forceinline__ int bits_u64(uint64_t v) { return v ? 64 - __clzll((long long)v) : 0; }

// Shared-memory footprint of prep_small<THREADS, ITEMS> for traces of at
// most THREADS * ITEMS / 2 blocks.
template <int THREADS, int ITEMS> struct SmallPrep {
    static constexpr int C = THREADS * ITEMS;  // sort capacity (2n)
    static constexpr int NMAX = C / 2;
    using SortT = cub::BlockRadixSort<uint64_t, THREADS, ITEMS, uint32_t>;
    using ScanT = cub::BlockScan<uint32_t, THREADS>;
    union Temp {
        typename SortT::TempStorage sort;
        typename ScanT::TempStorage scan;
    };
    struct Shared {
        Temp temp;
        uint64_t last_key[THREADS];
        uint32_t arank[NMAX], frank[NMAX], posof[NMAX], sar[NMAX], prio[NMAX];
        uint2 ent[NMAX];
        uint32_t U;
    };
};

template <int THREADS, int ITEMS>
__device__ void prep_small(const int64_t *trace_ptr, const FusedIn &in, uint32_t *sf, uint32_t *sp,
                           Rec *rec, uint2 *raw2, int t, unsigned char *smem_raw) {
    using P = SmallPrep<THREADS, ITEMS>;
    constexpr int NWARP = THREADS / 32;
    typename P::Shared &sh = *reinterpret_cast<typename P::Shared *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t b = trace_ptr[t];
    const int n = (int)(trace_ptr[t + 1] - b);
    const int64_t *A = in.alloc + b, *F = in.free_ + b, *S = in.size + b;

    // ---- ranges, gcd (trace scalars; k_trace_scale in prep.cu) ----
    int64_t mn = INT64_MAX, mx = INT64_MIN, g = 0, lm = 0, sm = 0;
    for (int i = tid; i < n; i += THREADS) {
        mn = min(mn, A[i]);
        mx = max(mx, F[i]);
        g = gcd64f(S[i], g);
        lm = max(lm, F[i] - A[i]);
        sm = max(sm, S[i]);
    }
    for (int o = 16; o; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
        g = gcd64f(g, __shfl_xor_sync(0xFFFFFFFFu, g, o));
        lm = max(lm, __shfl_xor_sync(0xFFFFFFFFu, lm, o));
        sm = max(sm, __shfl_xor_sync(0xFFFFFFFFu, sm, o));
    }
    __shared__ int64_t red5[5][NWARP];
    if (lane == 0) {
        red5[0][warp] = mn; red5[1][warp] = mx; red5[2][warp] = g;
        red5[3][warp] = lm; red5[4][warp] = sm;
    }
    __syncthreads();
    mn = red5[0][0]; mx = red5[1][0]; g = red5[2][0]; lm = red5[3][0]; sm = red5[4][0];
    for (int w = 1; w < NWARP; w++) {
        mn = min(mn, red5[0][w]); mx = max(mx, red5[1][w]); g = gcd64f(g, red5[2][w]);
        lm = max(lm, red5[3][w]); sm = max(sm, red5[4][w]);
    }
    if (g <= 0) g = 1;
    const int64_t tmin = mn;
    const uint64_t span = (uint64_t)mx - (uint64_t)mn;
    // total size in units of g, saturating at 2^62 (selects the height width)
    const uint64_t cap = uint64_t(1) << 62;
    uint64_t acc = 0;
    for (int i = tid; i < n; i += THREADS) {
        acc += (uint64_t)(S[i] / g);
        if (acc > cap) acc = cap;
    }
    for (int o = 16; o; o >>= 1) {
        acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
        if (acc > cap) acc = cap;
    }
    __syncthreads();
    if (lane == 0) red5[0][warp] = (int64_t)acc;
    __syncthreads();
    if (tid == 0) {
        uint64_t tot = 0;
        for (int w = 0; w < NWARP; w++) {
            tot += (uint64_t)red5[0][w];
            if (tot > cap) tot = cap;
        }
        in.unit[t] = g;
        in.total_units[t] = tot;
        in.tmin[t] = tmin;
        in.tspan[t] = span > (uint64_t)INT64_MAX ? INT64_MAX : (int64_t)span;
    }

    // ---- compressed time ranks over alloc ∪ free (stable sort, then ranks) ----
    uint64_t key[ITEMS];
    uint32_t val[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        const int i = tid * ITEMS + k;  // blocked arrangement
        if (i < 2 * n) {
            const int64_t tv = i < n ? A[i] : F[i - n];
            key[k] = (uint64_t)tv - (uint64_t)tmin;
            val[k] = (uint32_t)i;
        } else {
            key[k] = ~0ull;
            val[k] = 0xFFFFFFFFu;
        }
    }
    const int tbits = max(1, bits_u64(span));
    typename P::SortT(sh.temp.sort).Sort(key, val, 0, tbits);
    sh.last_key[tid] = key[ITEMS - 1];
    __syncthreads();
    uint32_t flag[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        const int p = tid * ITEMS + k;
        const uint64_t prev = k ? key[k - 1] : (tid ? sh.last_key[tid - 1] : ~0ull);
        flag[k] = (p < 2 * n && (p == 0 || key[k] != prev)) ? 1u : 0u;
    }
    uint32_t incl[ITEMS];
    typename P::ScanT(sh.temp.scan).InclusiveSum(flag, incl);
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        const int p = tid * ITEMS + k;
        if (p < 2 * n) {
            const uint32_t r = incl[k] - 1, v = val[k];
            if (v < (uint32_t)n) sh.arank[v] = r;
            else sh.frank[v - n] = r;
            if (p == 2 * n - 1) sh.U = incl[k];
        }
    }
    __syncthreads();

    // ---- (alloc, id) order: stable sort on the alloc rank ----
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        const int i = tid * ITEMS + k;
        key[k] = i < n ? (uint64_t)sh.arank[i] : ~0ull;
        val[k] = (uint32_t)i;
    }
    typename P::SortT(sh.temp.sort).Sort(key, val, 0, max(1, bits_u64((uint64_t)(2 * n))));
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        const int p = tid * ITEMS + k;
        if (p < n) {
            sh.posof[val[k]] = (uint32_t)p;
            sh.sar[p] = (uint32_t)key[k];
        }
    }
    __syncthreads();

    // ---- priority order: size desc, then (stable) lifetime desc; ids ascend ----
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        const int i = tid * ITEMS + k;
        key[k] = i < n ? (uint64_t)(sm - S[i]) : ~0ull;
        val[k] = (uint32_t)i;
    }
    typename P::SortT(sh.temp.sort).Sort(key, val, 0, max(1, bits_u64((uint64_t)sm)));
    __syncthreads();
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        const int p = tid * ITEMS + k;
        const uint32_t v = val[k];
        key[k] = p < n ? (uint64_t)(lm - (F[v] - A[v])) : ~0ull;
    }
    typename P::SortT(sh.temp.sort).Sort(key, val, 0, max(1, bits_u64((uint64_t)lm)));
#pragma unroll
    for (int k = 0; k < ITEMS; k++) {
        const int p = tid * ITEMS + k;
        if (p < n) sh.prio[val[k]] = (uint32_t)p;
    }
    __syncthreads();

    // ---- records, raw times, window entries ----
    for (int i = tid; i < n; i += THREADS) {
        Rec r;
        r.pos = sh.posof[i];
        r.arank = sh.arank[i];
        r.frank = sh.frank[i];
        uint32_t lo = 0, hi = (uint32_t)n;  // first position with alloc rank >= arank
        while (lo < hi) {
            const uint32_t m = (lo + hi) >> 1;
            if (sh.sar[m] < r.arank) lo = m + 1; else hi = m;
        }
        r.apos = lo;
        lo = 0; hi = (uint32_t)n;  // ... >= frank
        while (lo < hi) {
            const uint32_t m = (lo + hi) >> 1;
            if (sh.sar[m] < r.frank) lo = m + 1; else hi = m;
        }
        r.fpos = lo;
        r.k = (uint32_t)i;
        r.size = S[i] / g;
        const uint32_t pr = sh.prio[i];
        rec[b + pr] = r;
        raw2[b + pr] = make_uint2((uint32_t)(A[i] - tmin), (uint32_t)(F[i] - tmin));
        sh.ent[r.pos] = make_uint2(r.frank, pr);
        in.ent[b + r.pos] = make_uint2(r.frank, pr);
    }
    if (tid == 0) in.U[t] = sh.U;
    __syncthreads();

    // ---- chunk-sorted table rows (k_chunk_sort without skeletons) ----
    const int64_t cb = chunk_base(b, t);
    const int nch = (n + 31) >> 5;
    for (int j = warp; j < nch; j += NWARP) {
        const int p = 32 * j + lane;
        uint32_t k = 0xFFFFFFFFu, pr = kDead;
        if (p < n) {
            k = (sh.ent[p].x << 5) | (uint32_t)lane;
            pr = sh.ent[p].y;
        }
#pragma unroll
        for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
            for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                const uint32_t ok = __shfl_xor_sync(0xFFFFFFFFu, k, jj);
                const uint32_t op = __shfl_xor_sync(0xFFFFFFFFu, pr, jj);
                const bool up = ((lane & kk) == 0);
                const bool lower = ((lane & jj) == 0);
                const bool take = (lower == up) ? ok < k : ok > k;
                if (take) { k = ok; pr = op; }
            }
        }
        sf[32 * (cb + j) + lane] = k;
        sp[32 * (cb + j) + lane] = pr;
    }
    __syncthreads();
}

}  // namespace mp
