// K1/K2 — best-fit skyline planner on sm_100a ("sorted-skyline warp engine").
//
// Replaces solve_bestfit (bestfit.py:276-309) with OffsetLineSet
// (bestfit.py:61-201) and _RemainingBlocks.take_best (bestfit.py:243-262).
// Output is bit-identical to the reference: same offset per id, same peak.
//
// One warp owns one trace and runs the reference's dependent step loop; all
// lanes execute every step uniformly (no single-lane pointer chasing):
//
//  skyline   lines kept as a compact, time-sorted array: line i spans
//            [LO[i], LO[i+1]) at height H[i]; LOP[i] is the first (alloc,id)
//            position with alloc >= LO[i].  A sentinel at index L holds
//            (t_hi, n).  Heights are in units of the trace's size gcd, so for
//            all realistic traces they fit 32 bits and (H, LO) packs into one
//            u64 argmin key.
//  choose    rule R3 (bestfit.py:115-122): warp argmin of (height, lo) —
//            per-lane min over strided lines + two redux.sync.min.
//  query     rule R4 (bestfit.py:243-256): the window is positions
//            [LOP[c], LOP[c+1]); a block fits iff its free rank <= hi.
//            Entries at positions >= LOP[c+1] can never fit (alloc >= hi), so
//            only the window's left edge needs a position mask.  Full 32-entry
//            chunks are answered from a per-chunk summary (min/max free rank
//            of live entries, best live priority): all-fit -> summary, none
//            -> skip, straddling -> scanned by the whole warp.  The winner is
//            the minimum priority rank = max (lifetime, size, -id).
//  update    place (R6, :149-178) and lift_up (R5, :180-201) both replace
//            the chosen line (and at most one right neighbour) by <= 3 lines;
//            the tail shifts by d in [-2, 2] with warp-parallel copies.
//
// The loop bound assert (R8, bestfit.py:297) and IllegalLift (:185-186)
// are reported through the per-trace status word.
#include <algorithm>
#include <vector>

#include "common.h"
#include "plan.h"
#include "plan_types.cuh"
#include "prep.h"

namespace mp {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

struct PlanArgs {
    const int64_t *trace_ptr;
    uint2 *ent;               // mutable window table (global), N
    const Rec *rec;           // N
    const uint32_t *U;        // T
    const int64_t *unit;      // T
    int64_t *offsets;         // N (id order per trace)
    int64_t *peaks;           // T
    int64_t *stats;           // T * ST_N
    const int32_t *tlist;     // optional subset of traces (grid = its length)
    unsigned char *lines_g;   // global line storage when !LINES_SMEM
    uint4 *summ_g;            // global chunk summaries when !summ_smem
    int lcap;                 // line slots per trace (excluding sentinel)
    int ent_cap;              // entries cached in smem per trace (ENT_SMEM)
    int summ_smem;            // chunk summaries in shared memory
    int rec_smem;             // winner records in shared memory
};

__device__ __forceinline__ size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Line key = (height, lo) packed so that one unsigned compare orders lines by
// rule R3 (lowest height, then leftmost).  32-bit heights -> u64 keys;
// 64-bit heights -> 128-bit keys (96 significant bits).
template <typename HT> struct KeyT;

template <> struct KeyT<uint32_t> {
    using K = unsigned long long;
    static __device__ __forceinline__ K make(uint32_t h, uint32_t lo) {
        return ((K)h << 32) | lo;
    }
    static __device__ __forceinline__ uint32_t h(K k) { return (uint32_t)(k >> 32); }
    static __device__ __forceinline__ uint32_t lo(K k) { return (uint32_t)k; }
    static __device__ __forceinline__ K none() { return ~0ull; }
    static __device__ __forceinline__ K warp_min(K k) {
        const uint32_t a = __reduce_min_sync(kFull, (uint32_t)(k >> 32));
        const uint32_t b = __reduce_min_sync(kFull, (uint32_t)(k >> 32) == a ? (uint32_t)k
                                                                              : 0xFFFFFFFFu);
        return make(a, b);
    }
};

template <> struct KeyT<uint64_t> {
    using K = unsigned __int128;
    static __device__ __forceinline__ K make(uint64_t h, uint32_t lo) {
        return ((K)h << 32) | lo;
    }
    static __device__ __forceinline__ uint64_t h(K k) { return (uint64_t)(k >> 32); }
    static __device__ __forceinline__ uint32_t lo(K k) { return (uint32_t)k; }
    static __device__ __forceinline__ K none() { return ~(K)0; }
    static __device__ __forceinline__ K warp_min(K k) {
        const uint32_t w2 = (uint32_t)(k >> 64), w1 = (uint32_t)(k >> 32), w0 = (uint32_t)k;
        const uint32_t a = __reduce_min_sync(kFull, w2);
        const uint32_t b = __reduce_min_sync(kFull, w2 == a ? w1 : 0xFFFFFFFFu);
        const uint32_t c = __reduce_min_sync(kFull, (w2 == a && w1 == b) ? w0 : 0xFFFFFFFFu);
        return ((K)a << 64) | ((K)b << 32) | c;
    }
};

template <bool ENT_SMEM>
__device__ __forceinline__ uint2 load_ent(const uint2 *ent, int p, int n) {
    if (ENT_SMEM) return ent[p];  // smem copy is padded with dead entries
    return p < n ? ent[p] : make_uint2(kDead, kDead);
}

template <typename HT, bool ENT_SMEM, bool LINES_SMEM>
__global__ void __launch_bounds__(32) k_plan_sorted(PlanArgs a) {
    using KO = KeyT<HT>;
    using K = typename KO::K;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x;
    const int t = a.tlist ? a.tlist[blockIdx.x] : (int)blockIdx.x;
    const int64_t base = a.trace_ptr[t];
    const int n = (int)(a.trace_ptr[t + 1] - base);
    int64_t *st = a.stats + (int64_t)t * ST_N;
    if (n == 0) {  // R1: empty instance -> {} / peak 0 (bestfit.py:285-286)
        if (lane == 0) {
            a.peaks[t] = 0;
            st[ST_STEPS] = 0; st[ST_LIFTS] = 0; st[ST_MAXLINES] = 0; st[ST_STATUS] = PS_OK;
        }
        return;
    }
    const int lcap = a.lcap;
    const int nch = (n + 31) >> 5;
    const int64_t unit = a.unit[t];

    // ---- carve shared memory: lines | summaries | entries | records ----
    size_t off = 0;
    K *KEY;
    uint32_t *LOP;
    {
        const size_t kb = align16((size_t)(lcap + 1) * sizeof(K));
        const size_t stride = kb + align16((size_t)(lcap + 1) * 4);
        unsigned char *lb = LINES_SMEM ? smem : a.lines_g + (size_t)blockIdx.x * stride;
        KEY = reinterpret_cast<K *>(lb);
        LOP = reinterpret_cast<uint32_t *>(lb + kb);
        if (LINES_SMEM) off = stride;
    }
    uint4 *summ;
    if (a.summ_smem) {
        summ = reinterpret_cast<uint4 *>(smem + off);
        off += (size_t)nch * sizeof(uint4);
    } else {
        summ = a.summ_g + (base >> 5) + t;
    }
    uint2 *ent;
    if (ENT_SMEM) {
        ent = reinterpret_cast<uint2 *>(smem + off);
        off += align16((size_t)nch * 32 * sizeof(uint2));
        const uint2 *src = a.ent + base;
        for (int i = lane; i < nch * 32; i += 32) ent[i] = i < n ? src[i] : make_uint2(kDead, kDead);
    } else {
        ent = a.ent + base;
    }
    const uint4 *rec4;
    if (a.rec_smem) {
        uint4 *dst = reinterpret_cast<uint4 *>(smem + off);
        const uint4 *src = reinterpret_cast<const uint4 *>(a.rec + base);
        for (int i = lane; i < 2 * n; i += 32) dst[i] = src[i];
        rec4 = dst;
    } else {
        rec4 = reinterpret_cast<const uint4 *>(a.rec + base);
    }
    __syncwarp();
    // chunk summaries: (min live free rank, max live free rank, best live prio)
    for (int j = 0; j < nch; j++) {
        const uint2 e = load_ent<ENT_SMEM>(ent, (j << 5) + lane, n);
        const bool live = e.x != kDead;
        const uint32_t mn = __reduce_min_sync(kFull, live ? e.x : 0xFFFFFFFFu);
        const uint32_t mx = __reduce_max_sync(kFull, live ? e.x : 0u);
        const uint32_t bp = __reduce_min_sync(kFull, e.y);
        if (lane == 0) summ[j] = make_uint4(mn, mx, bp, 0);
    }
    // R2: one line over the whole span at height 0 (bestfit.py:287-289)
    int nl = 1;
    if (lane == 0) {
        KEY[0] = KO::make(0, 0); LOP[0] = 0;
        KEY[1] = KO::make(0, a.U[t] - 1); LOP[1] = (uint32_t)n;  // sentinel
    }
    __syncwarp();

    HT peak = 0;
    int64_t steps = 0, lifts = 0;
    int placed = 0, status = PS_OK, maxl = 1;
    const int64_t bound = 3 * (int64_t)n + 4;
    // the lowest line is known without a scan after a place that leaves a
    // shoulder: the shoulder keeps the chosen (minimal) height and nothing
    // else at that height lies to its left
    bool known = true;
    int c = 0;
    K ck = KO::make(0, 0);

    while (placed < n) {
        if (++steps > bound) { status = PS_LOOP_BOUND; break; }  // R8

        // ---- choose (R3): argmin of the packed (height, lo) keys ----
        if (!known) {
            K bk = KO::none();
            int bi = 0;
            for (int i0 = lane; i0 < nl; i0 += 128) {
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int i = i0 + 32 * u;
                    const K k = i < nl ? KEY[i] : KO::none();
                    if (k < bk) { bk = k; bi = i; }
                }
            }
            ck = KO::warp_min(bk);
            c = __shfl_sync(kFull, bi, __ffs(__ballot_sync(kFull, bk == ck)) - 1);
        }
        const HT ch = KO::h(ck);
        const uint32_t clo = KO::lo(ck);
        const bool hasP = c > 0, hasN = c + 1 < nl;
        const K kn = KEY[c + 1];
        const K kp = hasP ? KEY[c - 1] : KO::none();
        const uint32_t clop = LOP[c], chip = LOP[c + 1];
        const uint32_t chi = KO::lo(kn);
        const HT hN = KO::h(kn), hP = KO::h(kp);

        // ---- query (R4): best contained block, records prefetched ----
        uint32_t best = 0xFFFFFFFFu;
        if (clop < chip) {
            const int c0 = (int)(clop >> 5), c1 = (int)((chip - 1) >> 5);
            {
                const int p = (c0 << 5) + lane;
                const uint2 e = load_ent<ENT_SMEM>(ent, p, n);
                if (p >= (int)clop && e.x <= chi) best = e.y;
            }
            for (int jb = c0 + 1; jb <= c1; jb += 32) {
                const int j = jb + lane;
                bool strad = false;
                if (j <= c1) {
                    const uint4 sm = summ[j];
                    if (sm.x <= chi) {
                        if (sm.y <= chi) best = min(best, sm.z);
                        else strad = true;
                    }
                }
                unsigned m = __ballot_sync(kFull, strad);
                while (m) {
                    const int k0 = __ffs(m) - 1;
                    m &= m - 1;
                    const uint2 e0 = load_ent<ENT_SMEM>(ent, ((jb + k0) << 5) + lane, n);
                    if (m) {
                        const int k1 = __ffs(m) - 1;
                        m &= m - 1;
                        const uint2 e1 = load_ent<ENT_SMEM>(ent, ((jb + k1) << 5) + lane, n);
                        if (e1.x <= chi) best = min(best, e1.y);
                    }
                    if (e0.x <= chi) best = min(best, e0.y);
                }
            }
        }
        uint4 r0 = make_uint4(0, 0, 0, 0), r1 = make_uint4(0, 0, 0, 0);
        if (best != 0xFFFFFFFFu) {  // prefetch this lane's candidate record
            r0 = rec4[2 * best];
            r1 = rec4[2 * best + 1];
        }
        const uint32_t gbest = __reduce_min_sync(kFull, best);

        // ---- replacement of lines [c, c+e] by m new lines ----
        K nk0 = 0, nk1 = 0, nk2 = 0;
        uint32_t np0 = 0, np1 = 0, np2 = 0;
        int m = 0, e = 0, cnext = c;
        if (gbest == 0xFFFFFFFFu) {
            // lift_up (R5)
            ++lifts;
            if (!hasP && !hasN) { status = PS_ILLEGAL_LIFT; break; }
            const bool intoN = !hasP || (hasN && hP > hN);
            const bool intoP = !intoN && (!hasN || hP < hN);
            e = intoP ? 0 : 1;
            m = intoN ? 1 : 0;
            nk0 = KO::make(hN, clo);
            np0 = clop;
            known = false;
        } else {
            // place (R6)
            const int src = __ffs(__ballot_sync(kFull, best == gbest)) - 1;
            const uint32_t rpos = __shfl_sync(kFull, r0.x, src);
            const uint32_t rar = __shfl_sync(kFull, r0.y, src);
            const uint32_t rfr = __shfl_sync(kFull, r0.z, src);
            const uint32_t rap = __shfl_sync(kFull, r0.w, src);
            const uint32_t rfp = __shfl_sync(kFull, r1.x, src);
            const uint32_t rk = __shfl_sync(kFull, r1.y, src);
            HT rsz = (HT)__shfl_sync(kFull, r1.z, src);
            if (sizeof(HT) == 8)
                rsz |= (HT)((uint64_t)__shfl_sync(kFull, r1.w, src) << 32);
            const HT newh = ch + rsz;
            if (lane == 0) a.offsets[base + rk] = (int64_t)ch * unit;
            peak = max(peak, newh);
            ++placed;
            // retire the winner and refresh its chunk summary
            {
                const int j = (int)(rpos >> 5);
                const int p = (j << 5) + lane;
                uint2 en = load_ent<ENT_SMEM>(ent, p, n);
                if (p == (int)rpos) {
                    en = make_uint2(kDead, kDead);
                    ent[p] = en;
                }
                const bool live = en.x != kDead;
                const uint32_t mn = __reduce_min_sync(kFull, live ? en.x : 0xFFFFFFFFu);
                const uint32_t mx = __reduce_max_sync(kFull, live ? en.x : 0u);
                const uint32_t bp = __reduce_min_sync(kFull, en.y);
                if (lane == 0) summ[j] = make_uint4(mn, mx, bp, 0);
            }
            const bool hasL = clo < rar, hasR = rfr < chi;
            const bool mP = !hasL && hasP && hP == newh;  // flush re-merge (:171-174)
            const bool mN = !hasR && hasN && hN == newh;  // (:175-177)
            e = mN ? 1 : 0;
            const K kL = ck, kRa = KO::make(newh, rar), kR = KO::make(ch, rfr);
            // sequence: [L?] [raised unless merged into P] [R?]
            nk0 = hasL ? kL : (!mP ? kRa : kR);
            np0 = hasL ? clop : (!mP ? rap : rfp);
            nk1 = hasL ? (!mP ? kRa : kR) : kR;
            np1 = hasL ? (!mP ? rap : rfp) : rfp;
            nk2 = kR;
            np2 = rfp;
            m = (hasL ? 1 : 0) + (mP ? 0 : 1) + (hasR ? 1 : 0);
            known = hasL || hasR;
            ck = hasL ? kL : kR;
            // index of the predicted next line: L stays at c; R follows raised
            cnext = hasL ? c : c + (mP ? 0 : 1);
        }

        // ---- apply: shift the tail [c+1+e, nl] (incl. sentinel) by d ----
        const int d = m - 1 - e;
        if (nl + d > lcap) { status = PS_LINES_OVERFLOW; break; }
        if (d != 0) {
            const int from = c + 1 + e, to = nl;  // inclusive
            const int nblk = (to - from) >> 7;
            for (int q = 0; q <= nblk; q++) {
                // d < 0: front to back; d > 0: back to front (no overwrite)
                const int b = from + 128 * (d < 0 ? q : nblk - q);
                K vk[4];
                uint32_t vp[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int i = b + lane + 32 * u;
                    if (i <= to) { vk[u] = KEY[i]; vp[u] = LOP[i]; }
                }
                __syncwarp();
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int i = b + lane + 32 * u;
                    if (i <= to) { KEY[i + d] = vk[u]; LOP[i + d] = vp[u]; }
                }
                __syncwarp();
            }
        }
        if (lane < m) {
            KEY[c + lane] = lane == 0 ? nk0 : (lane == 1 ? nk1 : nk2);
            LOP[c + lane] = lane == 0 ? np0 : (lane == 1 ? np1 : np2);
        }
        nl += d;
        maxl = max(maxl, nl);
        c = cnext;
        __syncwarp();
    }
    if (lane == 0) {
        a.peaks[t] = (int64_t)peak * unit;  // R7: max(offset + size)
        st[ST_STEPS] = steps;
        st[ST_LIFTS] = lifts;
        st[ST_MAXLINES] = maxl;
        st[ST_STATUS] = status;
    }
}

template <typename HT, bool E, bool Ls>
int launch_one(const PlanArgs &a, int grid, size_t smem, cudaStream_t s) {
    auto fn = k_plan_sorted<HT, E, Ls>;
    if (smem > 48 * 1024)
        MP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<grid, 32, smem, s>>>(a);
    MP_CUDA(cudaGetLastError());
    return MP_OK;
}

template <typename HT>
int launch_ht(const PlanArgs &a, int grid, bool ent_smem, bool lines_smem, size_t smem,
              cudaStream_t s) {
    if (ent_smem && lines_smem) return launch_one<HT, true, true>(a, grid, smem, s);
    if (ent_smem) return launch_one<HT, true, false>(a, grid, smem, s);
    if (lines_smem) return launch_one<HT, false, true>(a, grid, smem, s);
    return launch_one<HT, false, false>(a, grid, smem, s);
}

int launch_plan(const PlanArgs &a, int grid, bool h32, bool ent_smem, bool lines_smem,
                size_t smem, cudaStream_t s) {
    return h32 ? launch_ht<uint32_t>(a, grid, ent_smem, lines_smem, smem, s)
               : launch_ht<uint64_t>(a, grid, ent_smem, lines_smem, smem, s);
}

thread_local mp_plan_info g_info;

size_t smem_limit(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    return v > 0 ? (size_t)v : 48 * 1024;
}

inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

struct Layout {
    bool lines_smem, summ_smem, ent_smem, rec_smem;
    size_t smem;
};

// Shared memory priority: skyline lines > chunk summaries > window entries >
// winner records.
// per line: packed key (8 B for 32-bit heights, 16 B for 64-bit) + LOP (4 B)
size_t lines_bytes(int lcap, size_t hbytes) {
    const size_t kbytes = hbytes == 4 ? 8 : 16;
    return a16((size_t)(lcap + 1) * kbytes) + a16((size_t)(lcap + 1) * 4);
}

Layout choose_layout(int64_t nmax, int lcap, size_t hbytes, size_t lim, bool force_global,
                     bool lines_global = false) {
    Layout l{};
    const size_t lines_b = lines_bytes(lcap, hbytes);
    const int64_t nch = (nmax + 31) / 32;
    const size_t summ_b = (size_t)nch * 16;
    const size_t ent_b = a16((size_t)nch * 32 * 8);
    const size_t rec_b = (size_t)nmax * 32;
    if (force_global) return l;
    size_t used = 0;
    if (!lines_global && lines_b <= lim) { l.lines_smem = true; used += lines_b; }
    if (used + summ_b <= lim) { l.summ_smem = true; used += summ_b; }
    if (used + ent_b <= lim) { l.ent_smem = true; used += ent_b; }
    if (used + rec_b <= lim) { l.rec_smem = true; used += rec_b; }
    l.smem = used;
    return l;
}

}  // namespace

const mp_plan_info &last_plan_info() { return g_info; }

int plan_device(const int64_t *trace_ptr_d, const int64_t *trace_ptr_h, int64_t T,
                const int64_t *alloc_d, const int64_t *free_d, const int64_t *size_d,
                int64_t *offsets_d, int64_t *peaks_d, int flags, int device, cudaStream_t s) {
    g_info = mp_plan_info{};
    if (T <= 0) return MP_OK;
    const int64_t N = trace_ptr_h[T] - trace_ptr_h[0];
    if (trace_ptr_h[0] != 0) {
        set_error("trace_ptr[0] must be 0");
        return MP_ERR_INVALID;
    }
    int64_t nmax = 0;
    for (int64_t t = 0; t < T; t++) nmax = std::max(nmax, trace_ptr_h[t + 1] - trace_ptr_h[t]);
    if (nmax >= (int64_t(1) << 30)) {
        set_error("trace too large");
        return MP_ERR_INVALID;
    }
    const size_t prep_b = prep_scratch_bytes(N, T);
    const size_t tab_b = Carver::need<uint2>(N) + Carver::need<Rec>(N) +
                         Carver::need<uint32_t>(T) + Carver::need<int64_t>(T) +
                         Carver::need<uint64_t>(T) + Carver::need<int64_t>(T * ST_N) +
                         Carver::need<uint4>(N / 32 + T + 1);
    Scratch sc;
    MP_TRY(sc.alloc(prep_b + tab_b, s));
    Carver cv(sc.ptr, prep_b + tab_b);
    PrepOut po;
    po.ent = cv.take<uint2>(N);
    po.rec = cv.take<Rec>(N);
    po.U = cv.take<uint32_t>(T);
    po.unit = cv.take<int64_t>(T);
    po.total_units = cv.take<uint64_t>(T);
    int64_t *stats = cv.take<int64_t>(T * ST_N);
    uint4 *summ_g = cv.take<uint4>(N / 32 + T + 1);
    void *prep_ws = cv.base + cv.off;
    size_t prep_ws_b = cv.cap - cv.off;

    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
    cudaEventRecord(e0, s);
    PrepIn pi{trace_ptr_d, alloc_d, free_d, size_d, N, T};
    int rc = prep_run(pi, po, prep_ws, prep_ws_b, s);
    if (rc != MP_OK) return rc;
    cudaEventRecord(e1, s);

    // 32-bit heights when every trace's total bytes fit 2^32 size units
    std::vector<uint64_t> tot((size_t)T);
    MP_CUDA(cudaMemcpyAsync(tot.data(), po.total_units, sizeof(uint64_t) * T,
                            cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    bool h32 = true;
    for (int64_t t = 0; t < T; t++) h32 = h32 && tot[t] < (uint64_t(1) << 32);
    const size_t hb = h32 ? 4 : 8;

    const size_t lim = smem_limit(device);
    const bool force_global = (flags & MP_FORCE_GLOBAL) != 0;
    const int64_t lneed = 2 * nmax + 2;  // worst case 2n+1 lines
    const int lcap_s = (int)std::min<int64_t>(lneed, 4096);
    Layout lay = choose_layout(nmax, lcap_s, hb, lim, force_global);

    PlanArgs a{};
    a.trace_ptr = trace_ptr_d;
    a.ent = po.ent;
    a.rec = po.rec;
    a.U = po.U;
    a.unit = po.unit;
    a.offsets = offsets_d;
    a.peaks = peaks_d;
    a.stats = stats;
    a.tlist = nullptr;
    a.summ_g = summ_g;
    a.lcap = lay.lines_smem ? lcap_s : (int)lneed;
    a.ent_cap = (int)nmax;
    a.summ_smem = lay.summ_smem;
    a.rec_smem = lay.rec_smem;
    const size_t line_bytes_g = lines_bytes(a.lcap, hb);
    Scratch lines_sc;
    if (!lay.lines_smem) {
        MP_TRY(lines_sc.alloc((size_t)T * line_bytes_g, s));
        a.lines_g = lines_sc.as<unsigned char>();
    }
    MP_TRY(launch_plan(a, (int)T, h32, lay.ent_smem, lay.lines_smem, lay.smem, s));

    // ---- collect status; re-run overflowed traces with global lines ----
    std::vector<int64_t> hst((size_t)T * ST_N);
    MP_CUDA(cudaMemcpyAsync(hst.data(), stats, sizeof(int64_t) * T * ST_N,
                            cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    std::vector<int32_t> redo;
    for (int64_t t = 0; t < T; t++)
        if (hst[t * ST_N + ST_STATUS] == PS_LINES_OVERFLOW) redo.push_back((int32_t)t);
    Layout lay2 = lay;
    if (!redo.empty()) {
        // restart overflowed traces from fresh tables with 2n+2 global lines
        rc = prep_run(pi, po, prep_ws, prep_ws_b, s);
        if (rc != MP_OK) return rc;
        Scratch tl;
        MP_TRY(tl.alloc(sizeof(int32_t) * redo.size(), s));
        MP_CUDA(cudaMemcpyAsync(tl.ptr, redo.data(), sizeof(int32_t) * redo.size(),
                                cudaMemcpyHostToDevice, s));
        PlanArgs b = a;
        b.tlist = tl.as<int32_t>();
        b.lcap = (int)lneed;
        lay2 = choose_layout(nmax, b.lcap, hb, lim, force_global, /*lines_global=*/true);
        b.summ_smem = lay2.summ_smem;
        b.rec_smem = lay2.rec_smem;
        Scratch lg;
        MP_TRY(lg.alloc(redo.size() * lines_bytes(b.lcap, hb), s));
        b.lines_g = lg.as<unsigned char>();
        MP_TRY(launch_plan(b, (int)redo.size(), h32, lay2.ent_smem, false, lay2.smem, s));
        MP_CUDA(cudaMemcpyAsync(hst.data(), stats, sizeof(int64_t) * T * ST_N,
                                cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
    }
    cudaEventRecord(e2, s);
    cudaEventSynchronize(e2);
    float ms_prep = 0, ms_plan = 0;
    cudaEventElapsedTime(&ms_prep, e0, e1);
    cudaEventElapsedTime(&ms_plan, e1, e2);
    cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2);
    g_info.prep_ms = ms_prep;
    g_info.plan_ms = ms_plan;
    g_info.engine = (h32 ? 16 : 0) | (lay.lines_smem ? 8 : 0) | (lay.summ_smem ? 4 : 0) |
                    (lay.ent_smem ? 2 : 0) | (lay.rec_smem ? 1 : 0) | (redo.empty() ? 0 : 32);
    g_info.cluster = 1;
    for (int64_t t = 0; t < T; t++) {
        g_info.steps += hst[t * ST_N + ST_STEPS];
        g_info.lifts += hst[t * ST_N + ST_LIFTS];
        g_info.max_lines = std::max(g_info.max_lines, hst[t * ST_N + ST_MAXLINES]);
        int64_t stv = hst[t * ST_N + ST_STATUS];
        if (stv == PS_LOOP_BOUND) {
            set_error("best-fit loop exceeded its iteration bound");
            return MP_ERR_LOOP_BOUND;
        }
        if (stv == PS_ILLEGAL_LIFT) {
            set_error("cannot lift the only offset line");
            return MP_ERR_ILLEGAL_LIFT;
        }
        if (stv != PS_OK) {
            set_error("planner status " + std::to_string(stv));
            return MP_ERR_CUDA;
        }
    }
    return MP_OK;
}

}  // namespace mp
