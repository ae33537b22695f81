// K3 — GPU plan validator; K4 — peak-live-bytes lower bound.
//
// K3 replaces verify_plan (verifier.py:44-81) over colliding_pairs
// (core.py:227-249).  The reference materialises the pair set E as Python
// tuples (|E| ~ n^2/4), which is infeasible beyond ~10^4 blocks; here blocks
// are sorted by alloc time and every colliding pair (p, q), p < q in that
// order, is enumerated exactly once as q in (p, end_p) with
// end_p = first position whose alloc >= free_p — each warp owns one p and
// its lanes sweep the contiguous q-range (coalesced loads of the
// alloc-sorted columns).  A pair is a violation when its address ranges
// [off, off+size) intersect; records are gathered (capped) and sorted by
// (i, j) on the host exactly as verifier.py:57 orders them.
//
// K4 replaces clique_lower_bound (core.py:252-268): events sorted by time
// with frees before allocs at equal ticks (stable radix sort of
// [frees | allocs]), inclusive prefix sum of +-size, max with 0.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "common.h"

namespace mp {

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t n) {
    int64_t g = (n + kThreads - 1) / kThreads;
    return (int)(g < 1 ? 1 : (g > 65535 * 16 ? 65535 * 16 : g));
}

__global__ void k_iota_alloc(const int64_t *__restrict__ alloc, int64_t n, int64_t *__restrict__ keys,
                             uint32_t *__restrict__ idx) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = alloc[i];
        idx[i] = (uint32_t)i;
    }
}

struct Col {
    int64_t a, f, o, s;
};

__global__ void k_gather_cols(const uint32_t *__restrict__ idx, const int64_t *__restrict__ alloc,
                              const int64_t *__restrict__ free_, const int64_t *__restrict__ size,
                              const int64_t *__restrict__ off, int64_t n, Col *__restrict__ cols) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = idx[p];
        cols[p] = Col{alloc[k], free_[k], off[k], size[k]};
    }
}

__global__ void k_pair_end(const Col *__restrict__ cols, int64_t n, uint32_t *__restrict__ endp) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = cols[p].f;
        int64_t lo = p + 1, hi = n;  // first q > p with alloc_q >= f
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (cols[mid].a < f) lo = mid + 1; else hi = mid;
        }
        endp[p] = (uint32_t)lo;
    }
}

struct ViolRec {
    int64_t i, j, bytes, ticks;
};

__global__ void k_pairs(const Col *__restrict__ cols, const uint32_t *__restrict__ idx,
                        const uint32_t *__restrict__ endp, int64_t n,
                        unsigned long long *__restrict__ count, ViolRec *__restrict__ out,
                        int64_t cap) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t p = warp; p < n; p += nwarps) {
        const Col cp = cols[p];
        const int64_t ep = cp.o + cp.s;
        const int64_t e = endp[p];
        for (int64_t q = p + 1 + lane; q < e; q += 32) {
            const Col cq = cols[q];
            const int64_t lo = max(cp.o, cq.o);
            const int64_t hi = min(ep, cq.o + cq.s);
            if (hi > lo) {
                const unsigned long long slot = atomicAdd(count, 1ull);
                if ((int64_t)slot < cap) {
                    const int64_t ki = idx[p] + 1, kj = idx[q] + 1;
                    ViolRec r;
                    r.i = min(ki, kj);
                    r.j = max(ki, kj);
                    r.bytes = hi - lo;
                    r.ticks = min(cp.f, cq.f) - max(cp.a, cq.a);
                    out[slot] = r;
                }
            }
        }
    }
}

// per-block partials: peak, min offset, used (128-bit as lo/hi with carry)
struct Part {
    int64_t peak, minoff;
    unsigned long long used_lo, used_hi;
};

__device__ __forceinline__ void add128(unsigned long long &lo, unsigned long long &hi,
                                       unsigned long long blo, unsigned long long bhi) {
    const unsigned long long s = lo + blo;
    hi += bhi + (s < lo ? 1ull : 0ull);
    lo = s;
}

__global__ void k_stats(const int64_t *__restrict__ alloc, const int64_t *__restrict__ free_,
                        const int64_t *__restrict__ size, const int64_t *__restrict__ off, int64_t n,
                        Part *__restrict__ parts) {
    int64_t pk = 0, mo = INT64_MAX;
    unsigned long long ulo = 0, uhi = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = off[k], s = size[k];
        pk = max(pk, o + s);
        mo = min(mo, o);
        const unsigned long long life = (unsigned long long)(free_[k] - alloc[k]);
        const unsigned long long us = (unsigned long long)s;
        add128(ulo, uhi, us * life, __umul64hi(us, life));
    }
    for (int o = 16; o; o >>= 1) {
        pk = max(pk, __shfl_xor_sync(0xFFFFFFFFu, pk, o));
        mo = min(mo, __shfl_xor_sync(0xFFFFFFFFu, mo, o));
        const unsigned long long a = __shfl_xor_sync(0xFFFFFFFFu, ulo, o);
        const unsigned long long b = __shfl_xor_sync(0xFFFFFFFFu, uhi, o);
        // xor-butterfly: every lane ends with the full sum
        add128(ulo, uhi, a, b);
    }
    __shared__ Part sp[kThreads / 32];
    if ((threadIdx.x & 31) == 0) sp[threadIdx.x >> 5] = Part{pk, mo, ulo, uhi};
    __syncthreads();
    if (threadIdx.x == 0) {
        Part r = sp[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) {
            r.peak = max(r.peak, sp[w].peak);
            r.minoff = min(r.minoff, sp[w].minoff);
            add128(r.used_lo, r.used_hi, sp[w].used_lo, sp[w].used_hi);
        }
        parts[blockIdx.x] = r;
    }
}

__global__ void k_lb_events(const int64_t *__restrict__ alloc, const int64_t *__restrict__ free_,
                            const int64_t *__restrict__ size, int64_t n, int64_t *__restrict__ t,
                            int64_t *__restrict__ dv) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 2 * n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n) { t[i] = free_[i]; dv[i] = -size[i]; }       // frees first
        else { t[i] = alloc[i - n]; dv[i] = size[i - n]; }
    }
}

struct MaxOp {
    __device__ __forceinline__ int64_t operator()(int64_t a, int64_t b) const { return a > b ? a : b; }
};

// stage host arrays into one device buffer when MP_DEVICE_PTRS is not set
struct Staged {
    Scratch buf;
    const int64_t *p[4] = {nullptr, nullptr, nullptr, nullptr};
    int stage(const int64_t *const *src, int count, int64_t n, bool dev, cudaStream_t s) {
        if (dev) {
            for (int i = 0; i < count; i++) p[i] = src[i];
            return MP_OK;
        }
        const size_t nb = sizeof(int64_t) * (size_t)n;
        MP_TRY(buf.alloc((nb + 256) * count, s));
        Carver cv(buf.ptr, buf.bytes);
        for (int i = 0; i < count; i++) {
            int64_t *d = cv.take<int64_t>(n);
            if (n) MP_CUDA(cudaMemcpyAsync(d, src[i], nb, cudaMemcpyHostToDevice, s));
            p[i] = d;
        }
        return MP_OK;
    }
};

}  // namespace

int verify_run(const int64_t *alloc, const int64_t *free_, const int64_t *size,
               const int64_t *offsets, int64_t n, mp_verify_report *out, mp_violation *viol_out,
               int64_t viol_cap, int flags, cudaStream_t s) {
    *out = mp_verify_report{};
    out->offsets_ok = 1;
    if (n == 0) return MP_OK;
    if (n >= (int64_t(1) << 31)) {
        set_error("too many blocks");
        return MP_ERR_INVALID;
    }
    const bool dev = (flags & MP_DEVICE_PTRS) != 0;
    Staged in;
    const int64_t *src[4] = {alloc, free_, size, offsets};
    MP_TRY(in.stage(src, 4, n, dev, s));
    const int64_t *A = in.p[0], *F = in.p[1], *S = in.p[2], *O = in.p[3];

    size_t tsort = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tsort, (const int64_t *)nullptr, (int64_t *)nullptr,
                                    (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)n);
    const int gs = std::min(grid_for(n), 148 * 8);
    const int64_t cap = std::max<int64_t>(viol_cap, 0);
    const size_t bytes = Carver::need<int64_t>(n) * 2 + Carver::need<uint32_t>(n) * 3 +
                         Carver::need<Col>(n) + Carver::need<char>(tsort) +
                         Carver::need<ViolRec>(cap + 1) + Carver::need<unsigned long long>(1) +
                         Carver::need<Part>(gs) + 4096;
    Scratch sc;
    MP_TRY(sc.alloc(bytes, s));
    Carver cv(sc.ptr, sc.bytes);
    int64_t *keys = cv.take<int64_t>(n), *keys_s = cv.take<int64_t>(n);
    uint32_t *idx = cv.take<uint32_t>(n), *idx_s = cv.take<uint32_t>(n);
    uint32_t *endp = cv.take<uint32_t>(n);
    Col *cols = cv.take<Col>(n);
    void *tmp = cv.take<char>(tsort);
    ViolRec *vr = cv.take<ViolRec>(cap + 1);
    unsigned long long *cnt = cv.take<unsigned long long>(1);
    Part *parts = cv.take<Part>(gs);

    const int g = grid_for(n);
    k_iota_alloc<<<g, kThreads, 0, s>>>(A, n, keys, idx);
    MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tsort, keys, keys_s, idx, idx_s, (int)n, 0, 64, s));
    k_gather_cols<<<g, kThreads, 0, s>>>(idx_s, A, F, S, O, n, cols);
    k_pair_end<<<g, kThreads, 0, s>>>(cols, n, endp);
    MP_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s));
    {
        const int warps_per_block = kThreads / 32;
        int64_t blocks = (n + warps_per_block - 1) / warps_per_block;
        blocks = std::min<int64_t>(blocks, 148 * 64);
        k_pairs<<<(unsigned)blocks, kThreads, 0, s>>>(cols, idx_s, endp, n, cnt, vr, cap);
    }
    k_stats<<<gs, kThreads, 0, s>>>(A, F, S, O, n, parts);
    MP_CUDA(cudaGetLastError());

    unsigned long long hcnt = 0;
    std::vector<Part> hp((size_t)gs);
    MP_CUDA(cudaMemcpyAsync(&hcnt, cnt, sizeof(hcnt), cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaMemcpyAsync(hp.data(), parts, sizeof(Part) * gs, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    Part tot = hp[0];
    for (int i = 1; i < gs; i++) {
        tot.peak = std::max(tot.peak, hp[i].peak);
        tot.minoff = std::min(tot.minoff, hp[i].minoff);
        unsigned long long lo = tot.used_lo + hp[i].used_lo;
        tot.used_hi += hp[i].used_hi + (lo < tot.used_lo ? 1ull : 0ull);
        tot.used_lo = lo;
    }
    out->n_violations = (int64_t)hcnt;
    out->peak_recomputed = tot.peak;
    out->offsets_ok = tot.minoff >= 0 ? 1 : 0;
    out->used_lo = tot.used_lo;
    out->used_hi = tot.used_hi;
    const int64_t stored = std::min<int64_t>((int64_t)hcnt, cap);
    if (stored > 0 && viol_out) {
        std::vector<ViolRec> h((size_t)stored);
        MP_CUDA(cudaMemcpy(h.data(), vr, sizeof(ViolRec) * stored, cudaMemcpyDeviceToHost));
        std::sort(h.begin(), h.end(), [](const ViolRec &x, const ViolRec &y) {
            return x.i != y.i ? x.i < y.i : x.j < y.j;
        });
        for (int64_t k = 0; k < stored; k++)
            viol_out[k] = mp_violation{h[k].i, h[k].j, h[k].bytes, h[k].ticks};
    }
    return MP_OK;
}

int clique_lb_run(const int64_t *alloc, const int64_t *free_, const int64_t *size, int64_t n,
                  int64_t *lb_out, int flags, cudaStream_t s) {
    const bool dev = (flags & MP_DEVICE_PTRS) != 0;
    if (n == 0) {
        if (dev) MP_CUDA(cudaMemsetAsync(lb_out, 0, sizeof(int64_t), s));
        else *lb_out = 0;
        return MP_OK;
    }
    Staged in;
    const int64_t *src[3] = {alloc, free_, size};
    MP_TRY(in.stage(src, 3, n, dev, s));
    const int64_t m = 2 * n;
    size_t t1 = 0, t2 = 0, t3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, (const int64_t *)nullptr, (int64_t *)nullptr,
                                    (const int64_t *)nullptr, (int64_t *)nullptr, (int)m);
    cub::DeviceScan::InclusiveSum(nullptr, t2, (const int64_t *)nullptr, (int64_t *)nullptr, (int)m);
    cub::DeviceReduce::Reduce(nullptr, t3, (const int64_t *)nullptr, (int64_t *)nullptr, (int)m,
                              MaxOp(), int64_t(0));
    const size_t tb = std::max(t1, std::max(t2, t3));
    Scratch sc;
    MP_TRY(sc.alloc(Carver::need<int64_t>(m) * 4 + Carver::need<char>(tb) +
                        Carver::need<int64_t>(1) + 1024, s));
    Carver cv(sc.ptr, sc.bytes);
    int64_t *t = cv.take<int64_t>(m), *ts = cv.take<int64_t>(m);
    int64_t *dv = cv.take<int64_t>(m), *dvs = cv.take<int64_t>(m);
    void *tmp = cv.take<char>(tb);
    int64_t *res = cv.take<int64_t>(1);
    k_lb_events<<<grid_for(m), kThreads, 0, s>>>(in.p[0], in.p[1], in.p[2], n, t, dv);
    size_t b = tb;
    MP_CUDA(cub::DeviceRadixSort::SortPairs(tmp, b, t, ts, dv, dvs, (int)m, 0, 64, s));
    b = tb;
    MP_CUDA(cub::DeviceScan::InclusiveSum(tmp, b, dvs, dv, (int)m, s));
    b = tb;
    MP_CUDA(cub::DeviceReduce::Reduce(tmp, b, dv, res, (int)m, MaxOp(), int64_t(0), s));
    if (dev) {
        MP_CUDA(cudaMemcpyAsync(lb_out, res, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
        if (!(flags & MP_ASYNC)) MP_CUDA(cudaStreamSynchronize(s));
    } else {
        MP_CUDA(cudaMemcpyAsync(lb_out, res, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
    }
    return MP_OK;
}

}  // namespace mp

extern "C" {

int mp_verify(const int64_t *alloc, const int64_t *free_, const int64_t *size,
              const int64_t *offsets, int64_t n, mp_verify_report *out, mp_violation *viol_out,
              int64_t viol_cap, int flags, int device, mp_stream_t stream) {
    MP_TRY(mp::use_device(device));
    return mp::verify_run(alloc, free_, size, offsets, n, out, viol_out, viol_cap, flags,
                          (cudaStream_t)stream);
}

int mp_clique_lower_bound(const int64_t *alloc, const int64_t *free_, const int64_t *size,
                          int64_t n, int64_t *lb_out, int flags, int device, mp_stream_t stream) {
    MP_TRY(mp::use_device(device));
    return mp::clique_lb_run(alloc, free_, size, n, lb_out, flags, (cudaStream_t)stream);
}

}  // extern "C"
