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
#include <math.h>
#include <stdlib.h>

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
    uint32_t *sf, *sp, *pm;   // chunk-sorted window table (global), 32 per chunk
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

// One skyline line: packed (height, lo) key and LOP, 16 B (32 B for wide keys)
template <typename K> struct __align__(16) LineRec {
    K key;
    uint32_t lop;
};

// Chunk-sorted window table views (see plan_types.cuh).
struct Tab {
    uint32_t *sf, *sp, *pm;
};

// Mark the winner's slot dead, recompute the chunk's prefix minima and its
// summary (one warp).  rpos is the winner's (alloc,id) position.
__device__ __forceinline__ void retire_entry(const Tab &tb, uint4 *summ, uint32_t rpos, int lane) {
    const int j = (int)(rpos >> 5);
    const uint32_t key = tb.sf[32 * j + lane];
    uint32_t pr = tb.sp[32 * j + lane];
    if ((key & 31u) == (rpos & 31u) && key != 0xFFFFFFFFu) {
        pr = kDead;
        tb.sp[32 * j + lane] = kDead;
    }
    uint32_t m = pr;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(kFull, m, o);
        if (lane >= o) m = min(m, v);
    }
    tb.pm[32 * j + lane] = m;
    const unsigned live = __ballot_sync(kFull, pr != kDead);
    const uint32_t fr = key >> 5;
    const uint32_t mn = live ? __shfl_sync(kFull, fr, __ffs(live) - 1) : 0xFFFFFFFFu;
    const uint32_t mx = live ? __shfl_sync(kFull, fr, 31 - __clz(live)) : 0u;
    const uint32_t bp = __shfl_sync(kFull, m, 31);
    if (lane == 0) summ[j] = make_uint4(mn, mx, bp, (uint32_t)__popc(live));
}

// Step state shared between the leader warp and the query warps.
template <typename K> struct StepShared {
    K ck;                 // chosen line key
    uint32_t clop, chip;  // chosen line window [clop, chip)
    uint32_t chi;         // chosen line hi (free-rank threshold)
    int done;             // loop exit flag (set by the leader)
    uint32_t wbest[32];   // per-warp best priority rank
    uint4 wrec[32][2];    // per-warp prefetched winner record
    unsigned long long wlive[32];
};

// Best contained block among the window chunks this warp handles.
//  - left partial chunk c0 (warp 0, cooperative): slots whose position is
//    below clop are outside the window;
//  - every other chunk j in (c0, c1] (one lane each): summary says none /
//    all fit, or it straddles and a 5-step binary search over the chunk's
//    sorted free ranks gives the fitting prefix, whose best priority is
//    PM[count-1].  Positions >= chip can never fit (alloc >= hi), so the
//    right end needs no mask.
template <bool STATS, int NW>
__device__ __forceinline__ uint32_t query_window(const uint4 *summ, const Tab &tb, int c0, int c1,
                                                 uint32_t chi, uint32_t clop, uint32_t chip,
                                                 int warp, int lane, unsigned long long &wlive) {
    uint32_t best = 0xFFFFFFFFu;
    const uint32_t thr = (chi << 5) | 31u;
    if (warp == 0) {
        const uint32_t key = tb.sf[32 * c0 + lane];
        const uint32_t pr = tb.sp[32 * c0 + lane];
        const uint32_t slot = key & 31u;
        if (slot >= (clop & 31u) && key <= thr) best = pr;
        if (STATS) {
            const uint32_t pos = 32u * (uint32_t)c0 + slot;
            wlive += __popc(__ballot_sync(kFull, key != 0xFFFFFFFFu && pr != kDead &&
                                                     pos >= clop && pos < chip));
            if (c1 > c0) {
                const uint32_t k2 = tb.sf[32 * c1 + lane];
                const uint32_t p2 = tb.sp[32 * c1 + lane];
                const uint32_t pos2 = 32u * (uint32_t)c1 + (k2 & 31u);
                wlive += __popc(__ballot_sync(kFull, k2 != 0xFFFFFFFFu && p2 != kDead && pos2 < chip));
            }
        }
    }
    for (int jb = c0 + 1 + 32 * warp; jb <= c1; jb += 32 * NW) {
        const int j = jb + lane;
        if (STATS) {
            const uint32_t w = (j < c1) ? summ[j].w : 0u;
            wlive += __reduce_add_sync(kFull, w);
        }
        if (j <= c1) {
            const uint4 sm = summ[j];
            if (sm.x <= chi) {
                if (sm.y <= chi) {
                    best = min(best, sm.z);
                } else {
                    const uint32_t *row = tb.sf + 32 * j;
                    int cnt = row[15] <= thr ? 16 : 0;
                    cnt += row[cnt + 7] <= thr ? 8 : 0;
                    cnt += row[cnt + 3] <= thr ? 4 : 0;
                    cnt += row[cnt + 1] <= thr ? 2 : 0;
                    cnt += row[cnt] <= thr ? 1 : 0;
                    if (cnt > 0) best = min(best, tb.pm[32 * j + cnt - 1]);
                }
            }
        }
    }
    return best;
}

template <typename HT, bool TAB_SMEM, bool LINES_SMEM, bool STATS, int NW>
__global__ void __launch_bounds__(32 * NW) k_plan_sorted(PlanArgs a) {
    using KO = KeyT<HT>;
    using K = typename KO::K;
    using LR = LineRec<K>;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ StepShared<K> ss;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int t = a.tlist ? a.tlist[blockIdx.x] : (int)blockIdx.x;
    const int64_t base = a.trace_ptr[t];
    const int n = (int)(a.trace_ptr[t + 1] - base);
    int64_t *st = a.stats + (int64_t)t * ST_N;
    if (n == 0) {  // R1: empty instance -> {} / peak 0 (bestfit.py:285-286)
        if (threadIdx.x == 0) {
            a.peaks[t] = 0;
            st[ST_STEPS] = 0; st[ST_LIFTS] = 0; st[ST_MAXLINES] = 0; st[ST_STATUS] = PS_OK;
            st[ST_WLIVE] = 0;
        }
        return;
    }
    const int lcap = a.lcap;
    const int nch = (n + 31) >> 5;
    const int64_t unit = a.unit[t];
    const int64_t cb = chunk_base(base, t);
    unsigned long long wlive = 0;  // STATS: live entries in the reference's windows

    // ---- carve shared memory: lines | summaries | table | records ----
    size_t off = 0;
    LR *L;
    {
        const size_t stride = align16((size_t)(lcap + 1) * sizeof(LR));
        L = reinterpret_cast<LR *>(LINES_SMEM ? smem : a.lines_g + (size_t)blockIdx.x * stride);
        if (LINES_SMEM) off = stride;
    }
    uint4 *summ;
    if (a.summ_smem) {
        summ = reinterpret_cast<uint4 *>(smem + off);
        off += (size_t)nch * sizeof(uint4);
        const uint4 *src = a.summ_g + cb;
        for (int i = threadIdx.x; i < nch; i += 32 * NW) summ[i] = src[i];
    } else {
        summ = a.summ_g + cb;
    }
    Tab tb;
    if (TAB_SMEM) {
        uint32_t *d = reinterpret_cast<uint32_t *>(smem + off);
        tb.sf = d;
        tb.sp = d + 32 * nch;
        tb.pm = d + 64 * nch;
        off += (size_t)nch * 32 * 12;
        const uint4 *s0 = reinterpret_cast<const uint4 *>(a.sf + 32 * cb);
        const uint4 *s1 = reinterpret_cast<const uint4 *>(a.sp + 32 * cb);
        const uint4 *s2 = reinterpret_cast<const uint4 *>(a.pm + 32 * cb);
        for (int i = threadIdx.x; i < nch * 8; i += 32 * NW) {
            reinterpret_cast<uint4 *>(tb.sf)[i] = s0[i];
            reinterpret_cast<uint4 *>(tb.sp)[i] = s1[i];
            reinterpret_cast<uint4 *>(tb.pm)[i] = s2[i];
        }
    } else {
        tb.sf = a.sf + 32 * cb;
        tb.sp = a.sp + 32 * cb;
        tb.pm = a.pm + 32 * cb;
    }
    const uint4 *rec4;
    if (a.rec_smem) {
        uint4 *dst = reinterpret_cast<uint4 *>(smem + off);
        const uint4 *src = reinterpret_cast<const uint4 *>(a.rec + base);
        for (int i = threadIdx.x; i < 2 * n; i += 32 * NW) dst[i] = src[i];
        rec4 = dst;
    } else {
        rec4 = reinterpret_cast<const uint4 *>(a.rec + base);
    }
    // R2: one line over the whole span at height 0 (bestfit.py:287-289)
    if (threadIdx.x == 0) {
        L[0].key = KO::make(0, 0); L[0].lop = 0;
        L[1].key = KO::make(0, a.U[t] - 1); L[1].lop = (uint32_t)n;  // sentinel
        ss.done = 0;
    }
    __syncthreads();

    // leader-warp state (warp 0; uniform across its lanes)
    int nl = 1;
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
    HT hP = 0, hN = 0;
    bool hasP = false, hasN = false;
    uint32_t clop = 0, chip = 0, chi = 0;

    for (;;) {
        // ======== leader: choose (R3) ========
        if (warp == 0) {
            if (placed >= n || ++steps > bound) {
                if (placed < n) status = PS_LOOP_BOUND;  // R8
                if (lane == 0) ss.done = 1;
            } else {
                if (!known) {
                    K bk = KO::none();
                    int bi = 0;
                    for (int i0 = lane; i0 < nl; i0 += 128) {
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            const int i = i0 + 32 * u;
                            const K k = i < nl ? L[i].key : KO::none();
                            if (k < bk) { bk = k; bi = i; }
                        }
                    }
                    ck = KO::warp_min(bk);
                    c = __shfl_sync(kFull, bi, __ffs(__ballot_sync(kFull, bk == ck)) - 1);
                }
                hasP = c > 0;
                hasN = c + 1 < nl;
                const LR ln = L[c + 1];
                const K kp = hasP ? L[c - 1].key : KO::none();
                clop = L[c].lop;
                chip = ln.lop;
                chi = KO::lo(ln.key);
                hN = KO::h(ln.key);
                hP = KO::h(kp);
                if (NW > 1 && lane == 0) {
                    ss.clop = clop; ss.chip = chip; ss.chi = chi;
                }
            }
        }
        if (NW > 1) __syncthreads();  // [A] choice published
        if (NW > 1 ? ss.done : (placed >= n || status != PS_OK)) break;

        // ======== all warps: query (R4) ========
        uint32_t qlop, qhip, qchi;
        if (NW > 1) { qlop = ss.clop; qhip = ss.chip; qchi = ss.chi; }
        else { qlop = clop; qhip = chip; qchi = chi; }
        uint32_t best = 0xFFFFFFFFu;
        if (qlop < qhip) {
            const int c0 = (int)(qlop >> 5), c1 = (int)((qhip - 1) >> 5);
            best = query_window<STATS, NW>(summ, tb, c0, c1, qchi, qlop, qhip, warp, lane, wlive);
        }
        // every lane prefetches its own candidate's record before the
        // reductions, so the L2 latency overlaps them and barrier [B]
        uint4 r0 = make_uint4(0, 0, 0, 0), r1 = make_uint4(0, 0, 0, 0);
        if (best != 0xFFFFFFFFu) {
            r0 = rec4[2 * best];
            r1 = rec4[2 * best + 1];
        }
        const uint32_t wb = __reduce_min_sync(kFull, best);
        uint32_t gbest;
        if (NW > 1) {
            if (best == wb && best != 0xFFFFFFFFu) {
                ss.wrec[warp][0] = r0;
                ss.wrec[warp][1] = r1;
            }
            if (lane == 0) ss.wbest[warp] = wb;
            __syncthreads();  // [B] per-warp winners published
            const uint32_t mine = lane < NW ? ss.wbest[lane] : 0xFFFFFFFFu;
            gbest = __reduce_min_sync(kFull, mine);
            int ww = -1;
            if (gbest != 0xFFFFFFFFu) ww = __ffs(__ballot_sync(kFull, mine == gbest)) - 1;
            if (ww == warp) {
                // the winning warp retires the entry while the leader
                // rewrites the skyline
                retire_entry(tb, summ, ss.wrec[warp][0].x, lane);
            }
            if (warp != 0) continue;
            if (gbest != 0xFFFFFFFFu) {
                r0 = ss.wrec[ww][0];
                r1 = ss.wrec[ww][1];
            }
        } else {
            gbest = wb;
            if (gbest != 0xFFFFFFFFu) {
                const int src = __ffs(__ballot_sync(kFull, best == gbest)) - 1;
                r0.x = __shfl_sync(kFull, r0.x, src);
                r0.y = __shfl_sync(kFull, r0.y, src);
                r0.z = __shfl_sync(kFull, r0.z, src);
                r0.w = __shfl_sync(kFull, r0.w, src);
                r1.x = __shfl_sync(kFull, r1.x, src);
                r1.y = __shfl_sync(kFull, r1.y, src);
                r1.z = __shfl_sync(kFull, r1.z, src);
                if (sizeof(HT) == 8) r1.w = __shfl_sync(kFull, r1.w, src);
            }
        }

        // ======== leader: replacement of lines [c, c+e] by m new lines ========
        K nk0 = 0, nk1 = 0, nk2 = 0;
        uint32_t np0 = 0, np1 = 0, np2 = 0;
        int m = 0, e = 0, cnext = c;
        if (gbest == 0xFFFFFFFFu) {
            // lift_up (R5)
            ++lifts;
            if (!hasP && !hasN) {
                status = PS_ILLEGAL_LIFT;
                placed = n;  // leave through the done path next round
                continue;
            }
            const bool intoN = !hasP || (hasN && hP > hN);
            const bool intoP = !intoN && (!hasN || hP < hN);
            e = intoP ? 0 : 1;
            m = intoN ? 1 : 0;
            nk0 = KO::make(hN, KO::lo(ck));
            np0 = clop;
            known = false;
        } else {
            // place (R6)
            const uint32_t rpos = r0.x, rar = r0.y, rfr = r0.z, rap = r0.w, rfp = r1.x,
                           rk = r1.y;
            HT rsz = (HT)r1.z;
            if (sizeof(HT) == 8) rsz |= (HT)((uint64_t)r1.w << 32);
            const HT ch = KO::h(ck);
            const uint32_t clo = KO::lo(ck);
            const HT newh = ch + rsz;
            if (lane == 0) a.offsets[base + rk] = (int64_t)ch * unit;
            peak = max(peak, newh);
            ++placed;
            if (NW == 1) retire_entry(tb, summ, rpos, lane);
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
        if (nl + d > lcap) {
            status = PS_LINES_OVERFLOW;
            placed = n;
            continue;
        }
        if (d != 0) {
            const int from = c + 1 + e, to = nl;  // inclusive
            const int nblk = (to - from) >> 7;
            for (int q = 0; q <= nblk; q++) {
                // d < 0: front to back; d > 0: back to front (no overwrite)
                const int b = from + 128 * (d < 0 ? q : nblk - q);
                LR v[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int i = b + lane + 32 * u;
                    if (i <= to) v[u] = L[i];
                }
                __syncwarp();
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int i = b + lane + 32 * u;
                    if (i <= to) L[i + d] = v[u];
                }
                __syncwarp();
            }
        }
        if (lane < m) {
            LR v;
            v.key = lane == 0 ? nk0 : (lane == 1 ? nk1 : nk2);
            v.lop = lane == 0 ? np0 : (lane == 1 ? np1 : np2);
            L[c + lane] = v;
        }
        nl += d;
        maxl = max(maxl, nl);
        c = cnext;
        __syncwarp();
    }
    if (STATS && NW > 1) {
        if (lane == 0) ss.wlive[warp] = wlive;
        __syncthreads();
        if (threadIdx.x == 0)
            for (int w = 1; w < NW; w++) wlive += ss.wlive[w];
    }
    if (threadIdx.x == 0) {
        a.peaks[t] = (int64_t)peak * unit;  // R7: max(offset + size)
        st[ST_STEPS] = steps;
        st[ST_LIFTS] = lifts;
        st[ST_MAXLINES] = maxl;
        st[ST_STATUS] = status;
        st[ST_WLIVE] = (int64_t)wlive;
    }
}

thread_local int64_t g_launches = 0;
thread_local int g_nwarps = 1;  // warps per trace chosen by plan_device
thread_local int g_carveout = -1;  // shared-memory carveout percent (-1: driver default)

template <typename HT, bool E, bool Ls, bool ST, int NW>
int launch_nw(const PlanArgs &a, int grid, size_t smem, cudaStream_t s) {
    auto fn = k_plan_sorted<HT, E, Ls, ST, NW>;
    if (smem > 48 * 1024)
        MP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // keep only the shared memory the resident CTAs need: the rest is L1,
    // which caches the L2-resident window table between steps
    MP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, g_carveout));
    fn<<<grid, 32 * NW, smem, s>>>(a);
    MP_CUDA(cudaGetLastError());
    g_launches++;
    return MP_OK;
}


template <typename HT, bool E, bool Ls, bool ST>
int launch_one(const PlanArgs &a, int grid, size_t smem, cudaStream_t s) {
    switch (g_nwarps) {
        case 1: return launch_nw<HT, E, Ls, ST, 1>(a, grid, smem, s);
        case 4: return launch_nw<HT, E, Ls, ST, 4>(a, grid, smem, s);
        case 8: return launch_nw<HT, E, Ls, ST, 8>(a, grid, smem, s);
        default: return launch_nw<HT, E, Ls, ST, 16>(a, grid, smem, s);
    }
}

template <typename HT, bool ST>
int launch_ht(const PlanArgs &a, int grid, bool ent_smem, bool lines_smem, size_t smem,
              cudaStream_t s) {
    if (ent_smem && lines_smem) return launch_one<HT, true, true, ST>(a, grid, smem, s);
    if (ent_smem) return launch_one<HT, true, false, ST>(a, grid, smem, s);
    if (lines_smem) return launch_one<HT, false, true, ST>(a, grid, smem, s);
    return launch_one<HT, false, false, ST>(a, grid, smem, s);
}

int launch_plan(const PlanArgs &a, int grid, bool h32, bool ent_smem, bool lines_smem,
                size_t smem, cudaStream_t s, bool stats) {
    if (stats)
        return h32 ? launch_ht<uint32_t, true>(a, grid, ent_smem, lines_smem, smem, s)
                   : launch_ht<uint64_t, true>(a, grid, ent_smem, lines_smem, smem, s);
    return h32 ? launch_ht<uint32_t, false>(a, grid, ent_smem, lines_smem, smem, s)
               : launch_ht<uint64_t, false>(a, grid, ent_smem, lines_smem, smem, s);
}

thread_local mp_plan_info g_info;

size_t smem_limit(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    return v > 0 ? (size_t)v : 48 * 1024;
}

inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

struct Layout {
    bool lines_smem, summ_smem, tab_smem, rec_smem;
    size_t smem;
};

// Shared memory priority: skyline lines > chunk summaries > chunk-sorted
// window table > winner records.
// per line: LineRec = packed key + LOP, 16 B (32 B for 64-bit heights)
size_t lines_bytes(int lcap, size_t hbytes) {
    const size_t lr = hbytes == 4 ? 16 : 32;
    return a16((size_t)(lcap + 1) * lr);
}

Layout choose_layout(int64_t nmax, int lcap, size_t hbytes, size_t lim, bool force_global,
                     bool lines_global = false) {
    Layout l{};
    const size_t lines_b = lines_bytes(lcap, hbytes);
    const int64_t nch = (nmax + 31) / 32;
    const size_t summ_b = (size_t)nch * 16;
    const size_t tab_b = (size_t)nch * 32 * 12;
    const size_t rec_b = (size_t)nmax * 32;
    if (force_global) return l;
    size_t used = 0;
    if (!lines_global && lines_b <= lim) { l.lines_smem = true; used += lines_b; }
    if (used + summ_b <= lim) { l.summ_smem = true; used += summ_b; }
    if (used + tab_b <= lim) { l.tab_smem = true; used += tab_b; }
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
    if (2 * nmax + 2 >= (int64_t(1) << kRankBits)) {
        set_error("trace too large (free ranks must fit 27 bits: n < 2^26)");
        return MP_ERR_INVALID;
    }
    const int64_t nchunks = N / 32 + T + 1;
    const size_t prep_b = prep_scratch_bytes(N, T);
    const size_t tab_b = Carver::need<uint2>(N) + Carver::need<Rec>(N) +
                         Carver::need<uint32_t>(T) + Carver::need<int64_t>(T) +
                         Carver::need<uint64_t>(T) + Carver::need<int64_t>(T * ST_N) +
                         Carver::need<uint4>(nchunks) + 3 * Carver::need<uint32_t>(32 * nchunks);
    Scratch sc;
    MP_TRY(sc.alloc(prep_b + tab_b, s));
    Carver cv(sc.ptr, prep_b + tab_b);
    PrepOut po;
    po.ent = cv.take<uint2>(N);
    po.sf = cv.take<uint32_t>(32 * nchunks);
    po.sp = cv.take<uint32_t>(32 * nchunks);
    po.pm = cv.take<uint32_t>(32 * nchunks);
    po.rec = cv.take<Rec>(N);
    po.U = cv.take<uint32_t>(T);
    po.unit = cv.take<int64_t>(T);
    po.total_units = cv.take<uint64_t>(T);
    int64_t *stats = cv.take<int64_t>(T * ST_N);
    uint4 *summ_g = cv.take<uint4>(nchunks);
    po.summ = summ_g;
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
    const int lcap_s = (int)std::min<int64_t>(lneed, 2048);
    Layout lay = choose_layout(nmax, lcap_s, hb, lim, force_global);
    // warps per trace: one leader warp always; helper warps split the window
    // query when the entry table lives in L2 (long dependent load chains)
    g_nwarps = lay.tab_smem ? 1 : 8;
    {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        const int64_t per_sm = std::max<int64_t>(1, (T + sms - 1) / sms);
        const double need = (double)per_sm * (double)(lay.smem + 1024 + sizeof(void *) * 256);
        int pct = (int)std::ceil(100.0 * need / (228.0 * 1024.0));
        g_carveout = std::min(100, std::max(0, pct));
    }
    if (const char *env = getenv("MEMPLAN_NWARPS")) {
        const int v = atoi(env);
        if (v == 1 || v == 4 || v == 8 || v == 16) g_nwarps = v;
    }

    PlanArgs a{};
    a.trace_ptr = trace_ptr_d;
    a.sf = po.sf;
    a.sp = po.sp;
    a.pm = po.pm;
    a.rec = po.rec;
    a.U = po.U;
    a.unit = po.unit;
    a.offsets = offsets_d;
    a.peaks = peaks_d;
    a.stats = stats;
    a.tlist = nullptr;
    a.summ_g = summ_g;
    a.lcap = lay.lines_smem ? lcap_s : (int)lneed;
    a.summ_smem = lay.summ_smem;
    a.rec_smem = lay.rec_smem;
    const size_t line_bytes_g = lines_bytes(a.lcap, hb);
    Scratch lines_sc;
    if (!lay.lines_smem) {
        MP_TRY(lines_sc.alloc((size_t)T * line_bytes_g, s));
        a.lines_g = lines_sc.as<unsigned char>();
    }
    const bool stats_on = (flags & MP_STATS) != 0;
    const int64_t launches0 = g_launches;
    cudaEvent_t k0, k1;
    cudaEventCreate(&k0); cudaEventCreate(&k1);
    cudaEventRecord(k0, s);
    MP_TRY(launch_plan(a, (int)T, h32, lay.tab_smem, lay.lines_smem, lay.smem, s, stats_on));
    cudaEventRecord(k1, s);

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
        MP_TRY(launch_plan(b, (int)redo.size(), h32, lay2.tab_smem, false, lay2.smem, s,
                           stats_on));
        MP_CUDA(cudaMemcpyAsync(hst.data(), stats, sizeof(int64_t) * T * ST_N,
                                cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
    }
    cudaEventRecord(e2, s);
    cudaEventSynchronize(e2);
    float ms_prep = 0, ms_plan = 0;
    cudaEventElapsedTime(&ms_prep, e0, e1);
    cudaEventElapsedTime(&ms_plan, e1, e2);
    float ms_kernel = 0;
    cudaEventElapsedTime(&ms_kernel, k0, k1);
    cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e2);
    cudaEventDestroy(k0); cudaEventDestroy(k1);
    g_info.prep_ms = ms_prep;
    g_info.plan_ms = ms_plan;
    g_info.kernel_ms = ms_kernel;
    g_info.launches = prep_launches() + (g_launches - launches0);
    g_info.engine = (h32 ? 16 : 0) | (lay.lines_smem ? 8 : 0) | (lay.summ_smem ? 4 : 0) |
                    (lay.tab_smem ? 2 : 0) | (lay.rec_smem ? 1 : 0) | (redo.empty() ? 0 : 32);
    g_info.cluster = g_nwarps;  // warps per trace (single-CTA engine)
    for (int64_t t = 0; t < T; t++) {
        g_info.steps += hst[t * ST_N + ST_STEPS];
        g_info.lifts += hst[t * ST_N + ST_LIFTS];
        g_info.sum_wlive += hst[t * ST_N + ST_WLIVE];
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
