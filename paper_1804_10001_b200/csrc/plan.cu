// K1/K2 — best-fit skyline planner on sm_100a.
//
// Replaces solve_bestfit (bestfit.py:276-309) with OffsetLineSet
// (bestfit.py:61-201) and _RemainingBlocks.take_best (bestfit.py:243-262).
//
// Engine "warp" (this file): one warp owns one trace.  The skyline lives in
// shared memory as slot arrays (lo, hi, lop, hip, prev, next, height); the
// window table (free rank, priority rank) in (alloc, id) order lives in
// shared memory when it fits, otherwise in global memory (L2-resident).
// Per step, all lanes:
//   1. choose   — lexicographic argmin (height, lo) over line slots with
//                 three redux.sync.min passes (rule R3, bestfit.py:115-122);
//   2. scan     — the line's window [lop, hip) for entries with free <= hi,
//                 min priority rank via redux.sync.min (R4, :243-256);
//   3. update   — lane 0 splices place (R6, :149-178) or lift_up (R5,
//                 :180-201); the winner's entry is overwritten with kDead.
// The loop bound assert (R8, :297) and IllegalLift (:185-186) are reported
// through the per-trace status word.
#include <algorithm>
#include <vector>

#include "common.h"
#include "plan.h"
#include "plan_types.cuh"
#include "prep.h"

namespace mp {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int64_t kDeadH = INT64_MAX;

struct Lines {
    uint32_t *lo, *hi, *lop, *hip;
    int32_t *prv, *nxt;
    int64_t *h;
    __device__ __forceinline__ void bind(unsigned char *base, int cap) {
        lo = reinterpret_cast<uint32_t *>(base);
        hi = lo + cap;
        lop = hi + cap;
        hip = lop + cap;
        prv = reinterpret_cast<int32_t *>(hip + cap);
        nxt = prv + cap;
        h = reinterpret_cast<int64_t *>(nxt + cap);  // cap even -> 8B aligned
    }
};

struct PlanArgs {
    const int64_t *trace_ptr;
    uint2 *ent;          // mutable window table (global), N
    const Rec *rec;      // N
    const uint32_t *U;   // T
    int64_t *offsets;    // N (CSR-aligned with inputs, id order per trace)
    int64_t *peaks;      // T
    int64_t *stats;      // T * ST_N
    const int32_t *tlist;  // optional subset of traces (grid = its length)
    unsigned char *lines_g;  // global line storage (LINES_SMEM == false)
    int lcap;                // line slots per trace
    int ent_cap;             // entries cached in smem per trace (ENT_SMEM)
};

template <bool ENT_SMEM, bool LINES_SMEM>
__global__ void __launch_bounds__(32) k_plan_warp(PlanArgs a) {
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
    uint2 *ent;
    size_t ent_bytes = 0;
    if (ENT_SMEM) {
        ent = reinterpret_cast<uint2 *>(smem);
        ent_bytes = ((size_t)a.ent_cap * sizeof(uint2) + 15) & ~size_t(15);
        const uint2 *src = a.ent + base;
        for (int i = lane; i < n; i += 32) ent[i] = src[i];
    } else {
        ent = a.ent + base;
    }
    Lines L;
    L.bind(LINES_SMEM ? smem + ent_bytes
                      : a.lines_g + (size_t)blockIdx.x * (size_t)a.lcap * kLineBytes,
           a.lcap);
    const Rec *rec = a.rec + base;
    const int lcap = a.lcap;

    // R2: one line over the whole span at height 0 (bestfit.py:287-289)
    if (lane == 0) {
        L.lo[0] = 0; L.hi[0] = a.U[t] - 1; L.lop[0] = 0; L.hip[0] = (uint32_t)n;
        L.prv[0] = -1; L.nxt[0] = -1; L.h[0] = 0;
    }
    __syncwarp();
    int hwm = 1, maxhwm = 1;
    int freelist = -1;  // lane 0 only; threaded through L.nxt
    int64_t peak = 0, steps = 0, lifts = 0;
    int placed = 0, status = PS_OK;
    const int64_t bound = 3 * (int64_t)n + 4;

    while (placed < n) {
        if (++steps > bound) { status = PS_LOOP_BOUND; break; }  // R8
        // ---- 1. choose: argmin (height, lo) over live slots ----
        int64_t bh = kDeadH;
        uint32_t blo = 0xFFFFFFFFu;
        int bs = 0;
        for (int s = lane; s < hwm; s += 32) {
            int64_t h = L.h[s];
            uint32_t lo = L.lo[s];
            if (h < bh || (h == bh && lo < blo)) { bh = h; blo = lo; bs = s; }
        }
        const uint32_t hh = (uint32_t)((uint64_t)bh >> 32), hl = (uint32_t)bh;
        const uint32_t mhh = __reduce_min_sync(kFull, hh);
        const uint32_t mhl = __reduce_min_sync(kFull, hh == mhh ? hl : 0xFFFFFFFFu);
        const bool eqh = (hh == mhh) && (hl == mhl);
        const uint32_t mlo = __reduce_min_sync(kFull, eqh ? blo : 0xFFFFFFFFu);
        const unsigned who = __ballot_sync(kFull, eqh && blo == mlo);
        const int c = __shfl_sync(kFull, bs, __ffs(who) - 1);
        const int64_t ch = (int64_t)(((uint64_t)mhh << 32) | mhl);
        const uint32_t clo = mlo, chi = L.hi[c], clop = L.lop[c], chip = L.hip[c];

        // ---- 2. scan the window for the best contained block ----
        uint32_t best = 0xFFFFFFFFu;
        {
            int p = (int)clop + lane;
            const int e = (int)chip;
            for (; p + 96 < e; p += 128) {
                uint2 e0 = ent[p], e1 = ent[p + 32], e2 = ent[p + 64], e3 = ent[p + 96];
                if (e0.x <= chi) best = min(best, e0.y);
                if (e1.x <= chi) best = min(best, e1.y);
                if (e2.x <= chi) best = min(best, e2.y);
                if (e3.x <= chi) best = min(best, e3.y);
            }
            for (; p < e; p += 32) {
                uint2 e0 = ent[p];
                if (e0.x <= chi) best = min(best, e0.y);
            }
        }
        best = __reduce_min_sync(kFull, best);

        if (best == 0xFFFFFFFFu) {
            // ---- 3a. lift_up (R5) ----
            ++lifts;
            if (lane == 0) {
                const int P = L.prv[c], N = L.nxt[c];
                if (P < 0 && N < 0) {
                    status = PS_ILLEGAL_LIFT;
                } else if (P < 0 || (N >= 0 && L.h[P] > L.h[N])) {  // into next
                    L.lo[N] = clo; L.lop[N] = clop; L.prv[N] = P;
                    if (P >= 0) L.nxt[P] = N;
                    L.h[c] = kDeadH; L.nxt[c] = freelist; freelist = c;
                } else if (N < 0 || L.h[P] < L.h[N]) {  // into prev
                    L.hi[P] = chi; L.hip[P] = chip; L.nxt[P] = N;
                    if (N >= 0) L.prv[N] = P;
                    L.h[c] = kDeadH; L.nxt[c] = freelist; freelist = c;
                } else {  // equal neighbours: merge all three at prev height
                    const int NN = L.nxt[N];
                    L.hi[P] = L.hi[N]; L.hip[P] = L.hip[N]; L.nxt[P] = NN;
                    if (NN >= 0) L.prv[NN] = P;
                    L.h[c] = kDeadH; L.nxt[c] = freelist; freelist = c;
                    L.h[N] = kDeadH; L.nxt[N] = freelist; freelist = N;
                }
            }
            status = __shfl_sync(kFull, status, 0);
            if (status != PS_OK) break;
        } else {
            // ---- 3b. place (R6) ----
            const Rec r = rec[best];
            const int64_t newh = ch + r.size;
            if (lane == 0) {
                ent[r.pos] = make_uint2(kDead, kDead);
                a.offsets[base + r.k] = ch;
                const int P = L.prv[c], N = L.nxt[c];
                int left = -1, right = -1;
                if (clo < r.arank) {
                    if (freelist >= 0) { left = freelist; freelist = L.nxt[left]; }
                    else if (hwm < lcap) left = hwm++;
                    if (left >= 0) {
                        L.lo[left] = clo; L.hi[left] = r.arank; L.lop[left] = clop;
                        L.hip[left] = r.apos; L.h[left] = ch;
                        L.prv[left] = P; L.nxt[left] = c;
                        if (P >= 0) L.nxt[P] = left;
                    } else {
                        status = PS_LINES_OVERFLOW;
                    }
                }
                if (r.frank < chi && status == PS_OK) {
                    if (freelist >= 0) { right = freelist; freelist = L.nxt[right]; }
                    else if (hwm < lcap) right = hwm++;
                    if (right >= 0) {
                        L.lo[right] = r.frank; L.hi[right] = chi; L.lop[right] = r.fpos;
                        L.hip[right] = chip; L.h[right] = ch;
                        L.prv[right] = c; L.nxt[right] = N;
                        if (N >= 0) L.prv[N] = right;
                    } else {
                        status = PS_LINES_OVERFLOW;
                    }
                }
                L.lo[c] = r.arank; L.hi[c] = r.frank; L.lop[c] = r.apos; L.hip[c] = r.fpos;
                L.h[c] = newh;
                L.prv[c] = left >= 0 ? left : P;
                L.nxt[c] = right >= 0 ? right : N;
                // flush re-merge of the raised segment (bestfit.py:171-177)
                if (left < 0 && P >= 0 && L.h[P] == newh) {
                    const int PP = L.prv[P];
                    L.lo[c] = L.lo[P]; L.lop[c] = L.lop[P]; L.prv[c] = PP;
                    if (PP >= 0) L.nxt[PP] = c;
                    L.h[P] = kDeadH; L.nxt[P] = freelist; freelist = P;
                }
                if (right < 0 && N >= 0 && L.h[N] == newh) {
                    const int NN = L.nxt[N];
                    L.hi[c] = L.hi[N]; L.hip[c] = L.hip[N]; L.nxt[c] = NN;
                    if (NN >= 0) L.prv[NN] = c;
                    L.h[N] = kDeadH; L.nxt[N] = freelist; freelist = N;
                }
            }
            peak = max(peak, newh);
            ++placed;
            status = __shfl_sync(kFull, status, 0);
            if (status != PS_OK) break;
        }
        hwm = __shfl_sync(kFull, hwm, 0);
        maxhwm = max(maxhwm, hwm);
        __syncwarp();
    }
    if (lane == 0) {
        a.peaks[t] = peak;  // R7: max(offset + size)
        st[ST_STEPS] = steps;
        st[ST_LIFTS] = lifts;
        st[ST_MAXLINES] = maxhwm;
        st[ST_STATUS] = status;
    }
}

template <bool E, bool Ls>
int launch_warp(const PlanArgs &a, int grid, size_t smem, cudaStream_t s) {
    auto fn = k_plan_warp<E, Ls>;
    if (smem > 48 * 1024)
        MP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<grid, 32, smem, s>>>(a);
    MP_CUDA(cudaGetLastError());
    return MP_OK;
}

int launch_plan(const PlanArgs &a, int grid, bool ent_smem, bool lines_smem, size_t smem,
                cudaStream_t s) {
    if (ent_smem && lines_smem) return launch_warp<true, true>(a, grid, smem, s);
    if (ent_smem) return launch_warp<true, false>(a, grid, smem, s);
    if (lines_smem) return launch_warp<false, true>(a, grid, smem, s);
    return launch_warp<false, false>(a, grid, smem, s);
}

thread_local mp_plan_info g_info;

size_t smem_limit(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    return v > 0 ? (size_t)v : 48 * 1024;
}

}  // namespace

const mp_plan_info &last_plan_info() { return g_info; }

// Device-pointer core: all arrays already in HBM.  `trace_ptr_h` is the host
// copy of the CSR offsets (used to size the launch).
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
    // scratch: prep workspace + tables + U + stats + (maybe) global lines
    const size_t prep_b = prep_scratch_bytes(N, T);
    const size_t tab_b = Carver::need<uint2>(N) + Carver::need<Rec>(N) +
                         Carver::need<uint32_t>(T) + Carver::need<int64_t>(T * ST_N);
    Scratch sc;
    MP_TRY(sc.alloc(prep_b + tab_b, s));
    Carver cv(sc.ptr, prep_b + tab_b);
    PrepOut po;
    po.ent = cv.take<uint2>(N);
    po.rec = cv.take<Rec>(N);
    po.U = cv.take<uint32_t>(T);
    int64_t *stats = cv.take<int64_t>(T * ST_N);
    void *prep_ws = cv.base + cv.off;
    size_t prep_ws_b = cv.cap - cv.off;

    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
    cudaEventRecord(e0, s);
    PrepIn pi{trace_ptr_d, alloc_d, free_d, size_d, N, T};
    int rc = prep_run(pi, po, prep_ws, prep_ws_b, s);
    if (rc != MP_OK) return rc;
    cudaEventRecord(e1, s);

    // ---- choose the engine configuration ----
    const size_t lim = smem_limit(device);
    const bool force_global = (flags & MP_FORCE_GLOBAL) != 0;
    // realistic skylines stay small (<= a few hundred lines); worst case 2n+1
    int64_t lneed = 2 * nmax + 2;
    int lcap_s = (int)std::min<int64_t>(lneed, 2048);
    lcap_s += lcap_s & 1;
    size_t lines_b = (size_t)lcap_s * kLineBytes;
    size_t ent_b = ((size_t)nmax * sizeof(uint2) + 15) & ~size_t(15);
    bool ent_smem = !force_global && ent_b + lines_b <= lim;
    bool lines_smem = !force_global && lines_b <= lim;
    size_t smem = (ent_smem ? ent_b : 0) + (lines_smem ? lines_b : 0);

    PlanArgs a{};
    a.trace_ptr = trace_ptr_d;
    a.ent = po.ent;
    a.rec = po.rec;
    a.U = po.U;
    a.offsets = offsets_d;
    a.peaks = peaks_d;
    a.stats = stats;
    a.tlist = nullptr;
    a.lcap = lines_smem ? lcap_s : (int)(lneed + (lneed & 1));
    a.ent_cap = (int)nmax;
    Scratch lines_sc;
    if (!lines_smem) {
        MP_TRY(lines_sc.alloc((size_t)T * a.lcap * kLineBytes, s));
        a.lines_g = lines_sc.as<unsigned char>();
    }
    MP_TRY(launch_plan(a, (int)T, ent_smem, lines_smem, smem, s));

    // ---- collect status; re-run overflowed traces with global lines ----
    std::vector<int64_t> hst((size_t)T * ST_N);
    MP_CUDA(cudaMemcpyAsync(hst.data(), stats, sizeof(int64_t) * T * ST_N,
                            cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    std::vector<int32_t> redo;
    for (int64_t t = 0; t < T; t++)
        if (hst[t * ST_N + ST_STATUS] == PS_LINES_OVERFLOW) redo.push_back((int32_t)t);
    if (!redo.empty()) {
        // the table copy in global was mutated by ENT_SMEM=false runs only;
        // overflowed traces must restart from a fresh table: rerun prep.
        rc = prep_run(pi, po, prep_ws, prep_ws_b, s);
        if (rc != MP_OK) return rc;
        Scratch tl;
        MP_TRY(tl.alloc(sizeof(int32_t) * redo.size(), s));
        MP_CUDA(cudaMemcpyAsync(tl.ptr, redo.data(), sizeof(int32_t) * redo.size(),
                                cudaMemcpyHostToDevice, s));
        PlanArgs b = a;
        b.tlist = tl.as<int32_t>();
        b.lcap = (int)(lneed + (lneed & 1));
        Scratch lg;
        MP_TRY(lg.alloc(redo.size() * (size_t)b.lcap * kLineBytes, s));
        b.lines_g = lg.as<unsigned char>();
        size_t smem2 = ent_smem ? ent_b : 0;
        MP_TRY(launch_plan(b, (int)redo.size(), ent_smem, false, smem2, s));
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
    g_info.engine = (ent_smem ? 1 : 0) | (lines_smem ? 2 : 0);
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
