// K1/K2 — best-fit skyline planner on sm_100a ("skeleton engine", v6).
//
// Replaces solve_bestfit (bestfit.py:276-309) with OffsetLineSet
// (bestfit.py:61-201) and _RemainingBlocks.take_best (bestfit.py:243-262).
// Output is bit-identical to the reference: same offset per id, same peak.
//
// One CTA (normally one warp) owns one trace and runs the reference's
// dependent step loop; a batch launches one CTA per trace.
//
//  skyline   lines kept as a compact, time-sorted array: line i spans
//            [LO[i], LO[i+1]) at height H[i]; LOP[i] is the first (alloc,id)
//            position with alloc >= LO[i]; RAW[i] is LO's raw time.  A
//            sentinel at index L holds (t_hi, n).  Heights are in units of the
//            trace's size gcd, so for realistic traces they fit 32 bits and
//            (H, LO) packs into one u64 argmin key.
//  choose    rule R3 (bestfit.py:115-122): warp argmin of (height, lo).
//            Skipped after a placement that leaves a shoulder (the shoulder
//            is the new lowest-leftmost line).
//  query     rule R4 (bestfit.py:243-256): the window is positions
//            [LOP[c], LOP[c+1]); a block fits iff its free rank <= hi.  Whole
//            groups of 32 chunks, then chunks, are answered from skeletons
//            (plan_types.cuh): nothing fits / the best entry fits -> exact;
//            otherwise a chunk's skeleton names the one 8-slot segment where
//            its fitting prefix ends, and that segment is read from the table
//            only if its prefix minimum can still beat the best so far.
//            Lifetime bounds (priority is lifetime-major; a block of a group
//            or chunk that fits lives at most raw(hi) - its raw alloc
//            origin) skip groups and segments that cannot win.  Winner =
//            minimum priority rank = max (lifetime, size, -id).  Traces of
//            at most kScanMaxBlocks blocks (TIER_SCAN) scan their window rows
//            from shared memory instead and keep no skeletons.
//  update    place (R6, :149-178) and lift_up (R5, :180-201) both replace
//            the chosen line (and at most one right neighbour) by <= 3 lines;
//            the tail shifts by d in [-2, 2] with warp-parallel copies.  The
//            winner's table slot is retired and its chunk and group
//            skeletons rebuilt (one row read, overlapped with the update).
//
// NW = 1: one warp, no block barriers at all.  NW > 1 (tuning): warp 0 leads
// (choose + update), all warps split the window; two barriers per step.
//
// The loop bound assert (R8, bestfit.py:297) and IllegalLift (:185-186)
// are reported through the per-trace status word.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>
#include <type_traits>
#include <vector>

#include <cooperative_groups.h>

#include "common.h"
#include "plan.h"
#include "plan_types.cuh"
#include "prep.h"
#include "fused_prep.cuh"

namespace mp {

namespace cg = cooperative_groups;

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint32_t kNone = 0xFFFFFFFFu;
// pending segment slots per warp (shared memory); a memory round adds at most
// 32 * kG and the list is drained above kPendCap - 32 * kG, so 128 is the
// least that holds kG = 4.  128 rather than 256: +1.8 % batched (16 traces
// per SM keep 1 KB more of their SM's L1 each, and drains come earlier)
constexpr int kPendCap = 128;

// Shared-memory tiers for the window structures: nothing / group skeleton /
// + chunk skeleton / + chunk-sorted table.
// TIER_SCAN: small traces keep the table in shared memory and scan their
// (short) windows row by row — no skeletons to maintain at all.
enum { TIER_GLOBAL = 0, TIER_GROUP = 1, TIER_SKEL = 2, TIER_ALL = 3, TIER_SCAN = 4,
       TIER_WARP = 5 /* TIER_TINY, warp_engine.cuh; host-side label only */,
       TIER_CLU = 6 /* TIER_SKEL in a cluster, table over DSMEM; host-side label */ };
// Flagged groups evaluated per memory round, and pending segments read per
// lane per wave.  Single traces: 4 groups with the chunk skeletons in shared
// memory (tier SKEL), else 3, and 2 segments.  LEAN (the batched kernel
// capped at 128 registers): 2 groups, 1 segment — the smallest memory-level
// parallelism that compiles without spills at 128 registers, which is what
// lets 16 traces share an SM (4 warps per SM sub-partition).
#ifndef MEMPLAN_KG_LEAN
#define MEMPLAN_KG_LEAN 2
#endif
#ifndef MEMPLAN_KG_SKEL
#define MEMPLAN_KG_SKEL 4
#endif
template <int TIER, bool LEAN>
constexpr int kGroupsPerRound = LEAN ? MEMPLAN_KG_LEAN : (TIER == TIER_SKEL ? MEMPLAN_KG_SKEL : 3);
template <bool LEAN> constexpr int kSegsPerLane = LEAN ? 1 : 2;
constexpr int64_t kScanMaxBlocks = 4096;
// Lifetime samples for the pruning bound: every kLtStep-th priority rank's
// lifetime in shared memory.  Lifetimes are non-increasing along priority
// rank (lifetime-major key), so the sample at or after rank e is a LOWER
// bound on e's lifetime — a slightly weaker but memory-round-free bound.
constexpr int kLtShift = 7, kLtStep = 1 << kLtShift;
__host__ __device__ inline size_t lt_bytes(int64_t n) {
    return ((size_t)(n + kLtStep - 1) / kLtStep + 1) * 4u + 15u & ~size_t(15);
}

struct PlanArgs {
    const int64_t *trace_ptr;
    uint32_t *sf, *sp;        // chunk-sorted window table (global), 32 per chunk
    uint4 *s0, *s1;           // chunk skeleton (global), see plan_types.cuh
    uint2 *s2;
    uint4 *gs;                // group skeleton (global)
    uint32_t *cnt;            // live entries per chunk (STATS)
    const Rec *rec;           // N
    const uint2 *raw2;        // N (priority order): raw alloc/free relative to tmin
    const int64_t *tspan;     // T: raw time span (lifetime pruning when < 2^31)
    const uint32_t *U;        // T
    const int64_t *unit;      // T
    int64_t *offsets;         // N (id order per trace)
    int64_t *peaks;           // T
    int64_t *stats;           // T * ST_N
    const int32_t *tlist;     // optional subset of traces (grid = its length)
    unsigned char *lines_g;   // global line storage when !LINES_SMEM
    int lcap;                 // line slots per trace (excluding sentinel)
    int rec_smem;             // winner records in shared memory
    int timing;               // diagnostics: per-phase clock() sums (NW = 1)
    int clu_cshift, clu_pshift;  // cluster tier: chunks / priorities per worker CTA (log2)
    const uint32_t *lt;       // cluster tier: N lifetimes (raw free - raw alloc), priority order
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
    static __device__ __forceinline__ uint32_t warp_min_h(uint32_t h) {
        return __reduce_min_sync(kFull, h);
    }
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
    static __device__ __forceinline__ uint64_t warp_min_h(uint64_t h) {
        const uint32_t a = __reduce_min_sync(kFull, (uint32_t)(h >> 32));
        const uint32_t b = __reduce_min_sync(kFull, (uint32_t)(h >> 32) == a ? (uint32_t)h
                                                                              : 0xFFFFFFFFu);
        return ((uint64_t)a << 32) | b;
    }
    static __device__ __forceinline__ K warp_min(K k) {
        const uint32_t w2 = (uint32_t)(k >> 64), w1 = (uint32_t)(k >> 32), w0 = (uint32_t)k;
        const uint32_t a = __reduce_min_sync(kFull, w2);
        const uint32_t b = __reduce_min_sync(kFull, w2 == a ? w1 : 0xFFFFFFFFu);
        const uint32_t c = __reduce_min_sync(kFull, (w2 == a && w1 == b) ? w0 : 0xFFFFFFFFu);
        return ((K)a << 64) | ((K)b << 32) | c;
    }
};

// One skyline line: packed (height, lo) key, LOP and the raw time of lo
// relative to the trace origin (lifetime pruning); 16 B (32 B for wide keys)
template <typename K> struct __align__(16) LineRec {
    K key;
    uint32_t lop;
    uint32_t raw;
};

// Window structures of one trace (pointers already offset to its chunks).
struct Win {
    uint4 *s0, *s1;      // chunk skeleton (shared or global)
    uint2 *s2;
    uint4 *gs;           // group skeleton (shared or global)
    int nch;             // chunks of this trace
    uint32_t *sf, *sp;   // chunk-sorted table (shared or global)
    uint32_t *cnt;       // live count per chunk (global, STATS only)
    uint64_t keep, stream;  // L2 policies (global tiers)
    // cluster tier (CLU): the table and the per-priority lifetimes live in
    // the shared memory of the cluster's worker CTAs (ranks 1..), read
    // through DSMEM; placed entries are tracked in a per-chunk bitmap in the
    // planner CTA's own shared memory (the remote table stays read-only)
    const uint32_t *lts; // lifetime samples: lts[k] = lifetime of priority rank
                         // min(kLtStep k, n - 1), shared memory (pruning bound)
    uint32_t tab;        // shared::cta offset of each worker's slice
    int cshift, pshift;  // chunks / priorities per worker: 1 << shift
    uint32_t *dead;      // per chunk: bit p = position 32 j + p placed
};

// ---- DSMEM access (cluster tier) ----
__device__ __forceinline__ uint32_t dsm_map(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
__device__ __forceinline__ uint32_t dsm_ld(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 dsm_ld4(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared::cluster.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a));
    return v;
}
// cluster address of chunk j's SF row (its SP row follows the worker's SF
// slice: + (128 << cshift))
__device__ __forceinline__ uint32_t dsm_row(const Win &w, int j) {
    const uint32_t jl = (uint32_t)j & ((1u << w.cshift) - 1u);
    return dsm_map(w.tab + 128u * jl, 1u + ((uint32_t)j >> w.cshift));
}
__device__ __forceinline__ uint32_t dsm_lifetime(const Win &w, uint32_t prio) {
    const uint32_t pl = prio & ((1u << w.pshift) - 1u);
    return dsm_ld(dsm_map(w.tab + (256u << w.cshift) + 4u * pl, 1u + (prio >> w.pshift)));
}
// a placed entry reads as kDead
__device__ __forceinline__ uint32_t dead_mask(uint32_t dm, uint32_t key, uint32_t pr) {
    return (dm >> (key & 31u)) & 1u ? kDead : pr;
}

// L2 cache policies for the global-memory tiers: the group / S0 skeletons are
// the hot, re-read working set of every step (evict_last); everything else
// is evict_normal — evict_first on S1/S2, records and raw times cost 3 % at
// 12 traces per SM (those lines are re-read by later steps of the same trace).
__device__ __forceinline__ uint64_t l2_policy_keep() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_stream() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint4 ldg_hint(const uint4 *ptr, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(ptr), "l"(pol));
    return v;
}
__device__ __forceinline__ uint2 ldg_hint(const uint2 *ptr, uint64_t pol) {
    uint2 v;
    asm volatile("ld.global.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y)
                 : "l"(ptr), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ldg_hint(const uint32_t *ptr, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(ptr), "l"(pol));
    return v;
}
// Skeleton / record loads: plain (shared memory or plain global) or with
// the L2 policy when the structure lives in global memory.
template <bool G, typename T> __device__ __forceinline__ T ldk(const T *p, uint64_t pol) {
    if (G) return ldg_hint(p, pol);
    return *p;
}

// Winner record (priority order) and its raw alloc/free.
__device__ __forceinline__ void load_rec(const uint4 *rec4, const uint2 *raw2, uint32_t b,
                                         bool rec_smem, uint64_t pol, uint4 &r0, uint4 &r1,
                                         uint2 &rw) {
    if (rec_smem) {
        r0 = rec4[2 * b];
        r1 = rec4[2 * b + 1];
    } else {
        r0 = ldg_hint(rec4 + 2 * b, pol);
        r1 = ldg_hint(rec4 + 2 * b + 1, pol);
    }
    rw = ldg_hint(raw2 + b, pol);
}

// Issue the row read of the retired entry's chunk (the data is consumed by
// retire_finish, so the latency overlaps whatever the warp does between).
struct RetireRow {
    uint32_t key, pr;
    int j;
    uint4 gq;  // S0 of chunk 32*(j>>5) + lane (the retired chunk's group)
};

template <bool SG, bool SCAN = false, bool CLU = false>
__device__ __forceinline__ RetireRow retire_load(const Win &w, uint32_t pos, int lane) {
    RetireRow r;
    r.j = (int)(pos >> 5);
    if (CLU) {
        const uint32_t row = dsm_row(w, r.j) + 4u * lane;
        r.key = dsm_ld(row);
        r.pr = dead_mask(w.dead[r.j], r.key, dsm_ld(row + (128u << w.cshift)));
    } else {
        r.key = w.sf[32 * r.j + lane];
        r.pr = w.sp[32 * r.j + lane];
    }
    const int jj = (r.j & ~31) + lane;
    r.gq = make_uint4(kNone, kNone, kNone, 0u);
    if (!SCAN && jj < w.nch) r.gq = ldk<SG>(w.s0 + jj, w.keep);
    return r;
}

// Mark the entry at (alloc,id)-position `pos` dead and rebuild its chunk's
// skeleton (one warp; TIER_SCAN keeps no skeleton).
template <bool STATS, bool SCAN = false, bool CLU = false>
__device__ __forceinline__ void retire_finish(const Win &w, RetireRow r, uint32_t pos, int lane) {
    if ((r.key & 31u) == (pos & 31u) && r.key != kNone) {
        r.pr = kDead;
        if (CLU) w.dead[r.j] |= 1u << (pos & 31u);
        else w.sp[32 * r.j + lane] = kDead;
    }
    if (SCAN) return;
    uint4 q;
    const uint32_t nlive = skel_store(r.key, r.pr, lane, w.s0, w.s1, w.s2, r.j, &q);
    if (STATS && lane == 0) w.cnt[r.j] = nlive;
    // the group's other chunks are unchanged: patch in the new S0 and reduce
    if (lane == (r.j & 31)) r.gq = q;
    group_reduce(r.gq, w.gs, r.j >> 5, lane);
}

// Step state shared between the leader warp and the query warps (NW > 1).
template <typename K> struct StepShared {
    uint32_t clop, chip, chi;  // chosen line window [clop, chip), hi
    uint32_t rawhi;            // raw time of hi (relative)
    int done;                  // loop exit flag (set by the leader)
    uint32_t wbest[32];        // per-warp best priority rank
    uint4 wrec[32][2];         // per-warp prefetched winner record
    uint2 wraw[32];            // and its raw alloc/free
    unsigned long long wst[32][5];  // per-warp STATS counters
};

__device__ __forceinline__ uint32_t fit_min4(uint4 k, uint4 v, uint32_t thr, uint32_t best) {
    best = k.x <= thr ? min(best, v.x) : best;
    best = k.y <= thr ? min(best, v.y) : best;
    best = k.z <= thr ? min(best, v.z) : best;
    best = k.w <= thr ? min(best, v.w) : best;
    return best;
}

// Read the pending segments — DU per lane in flight (32 * DU per wave), each
// as two 16-byte loads of SF and two of SP — skipping segments whose prefix
// minimum cannot beat `bound`, which tightens after every wave.  Returns
// this lane's best fitting priority.
template <int DU, bool CLU = false>
__device__ __forceinline__ uint32_t drain_pending(const Win &w, const uint32_t *pend, int np,
                                                  uint32_t thr, uint32_t bound, int lane) {
    __syncwarp();
    uint32_t best = kNone;
    for (int e0 = 0; e0 < np; e0 += 32 * DU) {
        uint4 k[DU][2], v[DU][2];
        uint32_t dm[DU];
        bool act[DU];
#pragma unroll
        for (int u = 0; u < DU; u++) {
            const int e = e0 + 32 * u + lane;
            act[u] = e < np && pend[kPendCap + e] < bound;
            if (act[u]) {
                const uint32_t code = pend[e];
                if (CLU) {
                    const int j = (int)(code >> 2);
                    const uint32_t row = dsm_row(w, j) + 32u * (code & 3u);
                    k[u][0] = dsm_ld4(row);
                    k[u][1] = dsm_ld4(row + 16u);
                    v[u][0] = dsm_ld4(row + (128u << w.cshift));
                    v[u][1] = dsm_ld4(row + (128u << w.cshift) + 16u);
                    dm[u] = w.dead[j];
                } else {
                    const int idx = 32 * (int)(code >> 2) + 8 * (int)(code & 3u);
                    const uint4 *kp = reinterpret_cast<const uint4 *>(w.sf + idx);
                    const uint4 *vp = reinterpret_cast<const uint4 *>(w.sp + idx);
                    k[u][0] = kp[0];
                    k[u][1] = kp[1];
                    v[u][0] = vp[0];
                    v[u][1] = vp[1];
                }
            }
        }
#pragma unroll
        for (int u = 0; u < DU; u++) {
            if (CLU && act[u]) {
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    v[u][h].x = dead_mask(dm[u], k[u][h].x, v[u][h].x);
                    v[u][h].y = dead_mask(dm[u], k[u][h].y, v[u][h].y);
                    v[u][h].z = dead_mask(dm[u], k[u][h].z, v[u][h].z);
                    v[u][h].w = dead_mask(dm[u], k[u][h].w, v[u][h].w);
                }
            }
            if (act[u]) {
                best = fit_min4(k[u][0], v[u][0], thr, best);
                best = fit_min4(k[u][1], v[u][1], thr, best);
            }
        }
        if (e0 + 32 * DU < np) bound = min(bound, __reduce_min_sync(kFull, best));
    }
    __syncwarp();
    return best;
}

// STATS counters per warp: live window entries, skeleton passes, table
// segments read, edge rows read.
struct QStats {
    unsigned long long wlive = 0, pass = 0, seg = 0, edge = 0;
};

// Evaluate chunk j against threshold thr from its skeleton: exact answers
// fold into `best`; a straddling chunk whose boundary segment may still win
// is appended to the warp's pending list (code = j<<2 | segment, and the
// segment's prefix minimum as the bound it must beat).
// One chunk's skeleton records (loaded together: one memory round).
struct ChunkSk {
    uint4 q;   // {K0, A, P, K15}
    uint4 r;   // {K7, K23, P7, P15}
    uint2 q2;  // {P23, RA}
    bool valid;
};

template <bool SG>
__device__ __forceinline__ ChunkSk load_chunk(const Win &w, int j, bool valid) {
    ChunkSk c;
    c.valid = valid;
    c.q = make_uint4(kNone, kNone, kNone, kNone);
    c.r = make_uint4(0, 0, 0, 0);
    c.q2 = make_uint2(0, 0);
    if (valid) {
        // loading S1/S2 only for straddling chunks costs more in rounds than
        // it saves in bytes (measured at 8 and 28 traces per SM)
        c.q = ldk<SG>(w.s0 + j, w.keep);
        c.r = ldk<SG>(w.s1 + j, w.stream);
        c.q2 = ldk<SG>(w.s2 + j, w.stream);
    }
    return c;
}

template <bool SG>
__device__ __forceinline__ void eval_chunk(const Win &w, int j, bool valid, uint32_t thr,
                                           uint32_t rawhi, uint32_t lstar, uint32_t &best,
                                           uint32_t *pend, int &np, int lane);

__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// PF: the table lives in global memory, so a segment that goes on the
// pending list is prefetched into L2 right away (the drain reads it after
// the remaining passes).
template <bool PF>
__device__ __forceinline__ void eval_loaded(const Win &w, const ChunkSk &c, int j, uint32_t thr,
                                            uint32_t rawhi, uint32_t lstar, uint32_t &best,
                                            uint32_t *pend, int &np, int lane) {
    bool need = false;
    uint32_t code = 0, pe = kNone;
    if (c.valid) {
        const uint4 q = c.q, r = c.r;
        const uint2 q2 = c.q2;
        const uint32_t p23 = q2.x;
        if (q.x <= thr) {
            if (q.y <= thr) {
                best = min(best, q.z);  // the chunk's best live entry fits
            } else {
                // the fitting prefix ends inside segment s; pb / pe = prefix
                // minima before / through segment s
                uint32_t pb, s;
                if (q.w <= thr) {
                    if (r.y <= thr) { s = 3; pb = p23; pe = q.z; }
                    else { s = 2; pb = r.w; pe = p23; }
                } else {
                    if (r.x <= thr) { s = 1; pb = r.z; pe = r.w; }
                    else { s = 0; pb = kNone; pe = r.z; }
                }
                best = min(best, pb);  // slots before segment s all fit
                // segment s may still hold a better fit: its prefix minimum
                // must beat the best, and (lifetime bound) a block of this
                // chunk that fits lives at most rawhi - RA
                if (pe < best && rawhi - q2.y >= lstar) {
                    need = true;
                    code = ((uint32_t)j << 2) | s;
                    if (PF) {
                        prefetch_l2(w.sf + 32 * j + 8 * s);
                        prefetch_l2(w.sp + 32 * j + 8 * s);
                    }
                }
            }
        }
    }
    const unsigned m = __ballot_sync(kFull, need);
    if (m) {
        if (need) {
            const int at = np + __popc(m & ((1u << lane) - 1u));
            pend[at] = code;
            pend[kPendCap + at] = pe;
        }
        np += __popc(m);
    }
}

template <bool SG>
__device__ __forceinline__ void eval_chunk(const Win &w, int j, bool valid, uint32_t thr,
                                           uint32_t rawhi, uint32_t lstar, uint32_t &best,
                                           uint32_t *pend, int &np, int lane) {
    const ChunkSk c = load_chunk<SG>(w, j, valid);
    eval_loaded<false>(w, c, j, thr, rawhi, lstar, best, pend, np, lane);
}

// Best contained block among the window chunks this warp handles (rule R4).
// Returns the warp-wide minimum priority; `lbest` is this lane's candidate
// and the lane holding the warp minimum has prefetched its record into r0/r1.
// TIER_SCAN query: every chunk row of the window, four rows per round.
template <bool STATS, int NW>
__device__ __forceinline__ uint32_t query_scan(const Win &w, const uint4 *rec4, const uint2 *raw2,
                                               int c0, int c1, uint32_t chi, uint32_t clop,
                                               uint32_t chip, int warp, int lane,
                                               uint32_t &lbest, uint4 &r0, uint4 &r1, uint2 &rw,
                                               QStats &qs, bool rec_smem) {
    const uint32_t thr = (chi << 5) | 31u;
    uint32_t best = kNone;
    for (int jb = c0 + 4 * warp; jb <= c1; jb += 4 * NW) {
        uint32_t k[4], p[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int j = jb + u;
            k[u] = kNone;
            p[u] = kDead;
            if (j <= c1) {
                k[u] = w.sf[32 * j + lane];
                p[u] = w.sp[32 * j + lane];
            }
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const uint32_t pos = 32u * (uint32_t)(jb + u) + (k[u] & 31u);
            if (pos >= clop && k[u] <= thr) best = min(best, p[u]);
            if (STATS)
                qs.wlive += __popc(__ballot_sync(kFull, k[u] != kNone && p[u] != kDead &&
                                                            pos >= clop && pos < chip));
        }
        if (STATS) qs.pass++;
    }
    const uint32_t wb = __reduce_min_sync(kFull, best);
    if (!rec_smem && best == wb && wb != kNone) load_rec(rec4, raw2, best, false, w.stream, r0, r1, rw);
    lbest = best;
    return wb;
}

template <bool STATS, int NW, int TIER, bool LEAN, bool CLU = false, bool LTS = true>
__device__ __forceinline__ uint32_t query_window(const Win &w, const uint4 *rec4, const uint2 *raw2,
                                                 uint32_t *pend, int c0, int c1, uint32_t chi,
                                                 uint32_t clop, uint32_t chip, uint32_t rawhi,
                                                 bool prune, int warp, int lane, uint32_t &lbest,
                                                 uint4 &r0, uint4 &r1, uint2 &rw, QStats &qs,
                                                 bool rec_smem) {
    if constexpr (TIER == TIER_SCAN)
        return query_scan<STATS, NW>(w, rec4, raw2, c0, c1, chi, clop, chip, warp, lane, lbest,
                                     r0, r1, rw, qs, rec_smem);
    constexpr int kG = kGroupsPerRound<TIER, LEAN>;
    constexpr int DU = kSegsPerLane<LEAN>;
    const uint32_t thr = (chi << 5) | 31u;
    uint32_t best = kNone;
    const bool partial = (clop & 31u) != 0;
    const int cs = partial ? c0 + 1 : c0;
    // left edge chunk (warp 0): issue the row read now, consume at the end
    bool edge = false;
    uint32_t ek = kNone, ep = kDead;
    // the group skeleton (shared memory from tier GROUP up) says when nothing
    // in the edge chunk's group fits at all: no row read, no chunk pass
    const bool g0_fits = ldk<(TIER < TIER_GROUP)>(w.gs + (c0 >> 5), w.keep).x <= thr;
    if (warp == 0 && partial && (TIER == TIER_ALL || g0_fits)) {  // speculative row read
        edge = true;
        if (CLU) {
            const uint32_t row = dsm_row(w, c0) + 4u * lane;
            ek = dsm_ld(row);
            ep = dead_mask(w.dead[c0], ek, dsm_ld(row + (128u << w.cshift)));
        } else {
            ek = w.sf[32 * c0 + lane];
            ep = w.sp[32 * c0 + lane];
        }
        if (STATS) qs.edge++;
    }
    if (STATS) {
        // live entries of the reference's window: edge chunk rows (warp 0)
        // plus the live counts of the chunks strictly inside
        if (warp == 0) {
            for (int e = 0; e < (c1 > c0 ? 2 : 1); e++) {
                const int cc = e ? c1 : c0;
                uint32_t kk, pp;
                if (CLU) {
                    const uint32_t row = dsm_row(w, cc) + 4u * lane;
                    kk = dsm_ld(row);
                    pp = dead_mask(w.dead[cc], kk, dsm_ld(row + (128u << w.cshift)));
                } else {
                    kk = w.sf[32 * cc + lane];
                    pp = w.sp[32 * cc + lane];
                }
                const uint32_t pos = 32u * (uint32_t)cc + (kk & 31u);
                qs.wlive += __popc(__ballot_sync(kFull, kk != kNone && pp != kDead &&
                                                            pos >= clop && pos < chip));
            }
        }
        for (int jb = c0 + 1 + 32 * warp; jb < c1; jb += 32 * NW) {
            const int j = jb + lane;
            qs.wlive += __reduce_add_sync(kFull, j < c1 ? w.cnt[j] : 0u);
        }
    }
    int np = 0;
    // chunks of the left partial group (warp 0)
    const int gcs = cs >> 5;
    int gf = gcs;
    if (cs <= c1 && (cs & 31)) {
        gf = gcs + 1;
        const bool gfits =
            gcs == (c0 >> 5) ? g0_fits : ldk<(TIER < TIER_GROUP)>(w.gs + gcs, w.keep).x <= thr;
        if (warp == 0 && gfits) {
            const int j = cs + lane;
            if (STATS) qs.pass++;
            eval_chunk<(TIER < TIER_SKEL)>(w, j, j <= c1 && j < 32 * gf, thr, rawhi, 0u, best,
                                            pend, np, lane);
            if (np > kPendCap - 32 * kG) {
                if (STATS) qs.seg += np;
                best = min(best, drain_pending<DU, CLU>(w, pend, np, thr, kNone, lane));
                np = 0;
            }
        }
    }
    // lifetime bound of the best candidate so far (0 = none yet)
    uint32_t lstar = 0, e_used = kNone;
    // whole groups [gf, c1 >> 5] (none when the window is the edge chunk alone)
    const int gl = cs <= c1 ? c1 >> 5 : gf - 1;
    for (int gb = gf + 32 * warp; gb <= gl; gb += 32 * NW) {
        const int g = gb + lane;
        bool scan = false;
        uint32_t graw = 0;
        if (STATS) qs.pass++;
        if (g <= gl) {
            const uint4 G = ldk<(TIER < TIER_GROUP)>(w.gs + g, w.keep);  // {G0, GA, GP, GR}
            if (G.x <= thr) {
                if (G.y <= thr) best = min(best, G.z);  // the group's best entry fits
                else { scan = true; graw = G.w; }
            }
        }
        unsigned m = __ballot_sync(kFull, scan);
        // Lifetime bound: a block of group g that fits [lo, hi) lives at most
        // rawhi - GR(g).  Priority order is lifetime-major, so a group whose
        // bound is below the lifetime of the best candidate so far cannot
        // hold a better one (equal bounds are kept: size and id break
        // lifetime ties).  GR grows left to right, so once a group fails
        // every group to its right fails too; flagged groups are scanned
        // left to right and the bound is re-applied as the best improves —
        // before every memory round that still has flagged groups (waiting
        // for the best's raw times costs less than one skippable round:
        // +3 % over tightening only when 3-4 groups were pending).
        auto tighten = [&]() {
            const uint32_t e = __reduce_min_sync(kFull, best);
            if (e < e_used) {
                e_used = e;
                if (CLU) {
                    lstar = dsm_lifetime(w, e);
                } else if (LTS) {
                    lstar = w.lts[(e >> kLtShift) + 1];  // lower bound, no memory round
                } else {
                    const uint2 er = rec_smem ? raw2[e] : ldg_hint(raw2 + e, w.stream);
                    lstar = er.y - er.x;
                }
                m &= __ballot_sync(kFull, scan && rawhi - graw >= lstar);
            }
        };
        if (lstar) m &= __ballot_sync(kFull, scan && rawhi - graw >= lstar);
        if (prune && m) tighten();
        while (m) {
            // up to kG flagged groups per memory round (left to right)
            ChunkSk ck4[kG];
            int jj[kG];
#pragma unroll
            for (int u = 0; u < kG; u++) {
                jj[u] = -1;
                if (m) {
                    const int g2 = gb + __ffs(m) - 1;
                    m &= m - 1;
                    jj[u] = 32 * g2 + lane;
                }
                ck4[u] = load_chunk<(TIER < TIER_SKEL)>(w, jj[u], jj[u] >= 0 && jj[u] <= c1);
            }
#pragma unroll
            for (int u = 0; u < kG; u++) {
                if (__any_sync(kFull, jj[u] >= 0)) {
                    if (STATS) qs.pass++;
                    eval_loaded<(TIER < TIER_ALL) && !CLU>(w, ck4[u], jj[u], thr, rawhi, lstar,
                                                           best, pend, np, lane);
                }
            }
            if (np > kPendCap - 32 * kG) {
                if (STATS) qs.seg += np;
                best = min(best, drain_pending<DU, CLU>(w, pend, np, thr, kNone, lane));
                np = 0;
            }
            if (prune && m) tighten();
        }
    }
    // the speculative edge row has long arrived: fold it in first
    if (edge && (ek & 31u) >= (clop & 31u) && ek <= thr) best = min(best, ep);
    // provisional warp winner: prefetch its record while the segments load
    const uint32_t wb1 = __reduce_min_sync(kFull, best);
    if (!rec_smem && best == wb1 && best != kNone) {
        load_rec(rec4, raw2, best, false, w.stream, r0, r1, rw);
    }
    if (!np) {
        lbest = best;
        return wb1;
    }
    if (STATS) {
        for (int e = lane; e < np; e += 32)
            qs.seg += __popc(__ballot_sync(__activemask(), pend[kPendCap + e] < wb1));
    }
    const uint32_t b2 = drain_pending<DU, CLU>(w, pend, np, thr, wb1, lane);
    if (b2 < best) best = b2;
    const uint32_t wb = __reduce_min_sync(kFull, best);
    if (!rec_smem && wb != wb1 && best == wb) {  // a pending segment improved it
        load_rec(rec4, raw2, best, false, w.stream, r0, r1, rw);
    }
    lbest = best;
    return wb;
}

// The step loop for trace t, run by threads [0, 32*NW) of the CTA (k_plan
// launches exactly those; the fused small-trace kernel hands its warp 0 in).
// LEAN: 32-bit step counters.  Frees the registers the capped batched kernel
// would otherwise spill; the uncapped single-trace kernels schedule better
// with 64-bit ones (measured, TIER_ALL 10^4: 5-7 %).
template <typename HT, bool LINES_SMEM, bool STATS, int NW, int TIER, bool TIMING,
          bool LEAN = false, bool CLU = false>
__device__ __forceinline__ void plan_trace(const PlanArgs &a, const int t) {
    using Cnt = std::conditional_t<LEAN, int, int64_t>;
    using KO = KeyT<HT>;
    using K = typename KO::K;
    using LR = LineRec<K>;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ StepShared<K> ss;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t base = a.trace_ptr[t];
    const int n = (int)(a.trace_ptr[t + 1] - base);
    int64_t *st = a.stats + (int64_t)t * ST_N;
    if (n == 0) {  // R1: empty instance -> {} / peak 0 (bestfit.py:285-286)
        if (threadIdx.x == 0) {
            a.peaks[t] = 0;
            st[ST_STEPS] = 0; st[ST_LIFTS] = 0; st[ST_MAXLINES] = 0; st[ST_STATUS] = PS_OK;
            for (int k = ST_WLIVE; k < ST_N; k++) st[k] = 0;
        }
        return;
    }
    const int lcap = a.lcap;
    const bool prune = a.tspan[t] < (int64_t(1) << 31);
    const int nch = (n + 31) >> 5;
    const int64_t unit = a.unit[t];
    const int64_t cb = chunk_base(base, t);
    QStats qs;                     // STATS counters (this warp)
    unsigned long long nscan = 0;  // STATS: choose scans (leader)

    // ---- carve shared memory: lines | pending | skeleton | table | records ----
    size_t off = 0;
    LR *L;
    {
        const size_t stride = align16((size_t)(lcap + 1) * sizeof(LR));
        L = reinterpret_cast<LR *>(LINES_SMEM ? smem : a.lines_g + (size_t)blockIdx.x * stride);
        if (LINES_SMEM) off = stride;
    }
    uint32_t *pend = reinterpret_cast<uint32_t *>(smem + off) + warp * 2 * kPendCap;
    off += (size_t)NW * 2 * kPendCap * sizeof(uint32_t);
    Win win;
    if (TIER != TIER_SCAN) {
        uint32_t *lts = reinterpret_cast<uint32_t *>(smem + off);
        off += lt_bytes(n);
        if (prune) {
            const uint2 *rw2 = a.raw2 + base;
            const int ns = (n + kLtStep - 1) / kLtStep;
            for (int k = threadIdx.x; k <= ns; k += 32 * NW) {
                const uint2 v = rw2[min(k * kLtStep, n - 1)];
                lts[k] = v.y - v.x;
            }
        }
        win.lts = lts;
    }
    win.cnt = a.cnt + cb;
    win.keep = l2_policy_keep();
    win.stream = l2_policy_stream();
    win.nch = nch;
    const int ngr = (nch + 31) >> 5;
    const int64_t gbase = group_base(base, t);
    if (TIER >= TIER_GROUP && TIER != TIER_SCAN) {
        uint4 *g = reinterpret_cast<uint4 *>(smem + off);
        off += (size_t)ngr * 16;
        for (int i = threadIdx.x; i < ngr; i += 32 * NW) g[i] = a.gs[gbase + i];
        win.gs = g;
    } else {
        win.gs = a.gs + gbase;
    }
    if (CLU) {  // placed-entry bitmap (the remote table is never written)
        win.dead = reinterpret_cast<uint32_t *>(smem + off);
        off += align16((size_t)nch * 4);
        for (int i = threadIdx.x; i < nch; i += 32 * NW) win.dead[i] = 0;
        win.tab = (uint32_t)__cvta_generic_to_shared(smem);  // workers' slice offset
        win.cshift = a.clu_cshift;
        win.pshift = a.clu_pshift;
    }
    if (TIER >= TIER_SKEL && TIER != TIER_SCAN) {
        uint4 *d = reinterpret_cast<uint4 *>(smem + off);
        off += (size_t)nch * 32 + align16((size_t)nch * 8);
        for (int i = threadIdx.x; i < nch; i += 32 * NW) {
            d[i] = a.s0[cb + i];
            d[nch + i] = a.s1[cb + i];
            reinterpret_cast<uint2 *>(d + 2 * nch)[i] = a.s2[cb + i];
        }
        win.s0 = d;
        win.s1 = d + nch;
        win.s2 = reinterpret_cast<uint2 *>(d + 2 * nch);
    } else {
        win.s0 = a.s0 + cb;
        win.s1 = a.s1 + cb;
        win.s2 = a.s2 + cb;
    }
    if (TIER == TIER_ALL || TIER == TIER_SCAN) {
        uint32_t *d = reinterpret_cast<uint32_t *>(smem + off);
        off += (size_t)nch * 32 * 8;
        const uint4 *s0 = reinterpret_cast<const uint4 *>(a.sf + 32 * cb);
        const uint4 *s1 = reinterpret_cast<const uint4 *>(a.sp + 32 * cb);
        for (int i = threadIdx.x; i < nch * 8; i += 32 * NW) {
            reinterpret_cast<uint4 *>(d)[i] = s0[i];
            reinterpret_cast<uint4 *>(d + 32 * nch)[i] = s1[i];
        }
        win.sf = d;
        win.sp = d + 32 * nch;
    } else {
        win.sf = a.sf + 32 * cb;
        win.sp = a.sp + 32 * cb;
    }
    const uint4 *rec4;
    const uint2 *raw2 = a.raw2 + base;
    if (a.rec_smem) {
        uint2 *rdst = reinterpret_cast<uint2 *>(smem + off + (size_t)n * 32);
        for (int i = threadIdx.x; i < n; i += 32 * NW) rdst[i] = raw2[i];
        raw2 = rdst;
        uint4 *dst = reinterpret_cast<uint4 *>(smem + off);
        const uint4 *src = reinterpret_cast<const uint4 *>(a.rec + base);
        for (int i = threadIdx.x; i < 2 * n; i += 32 * NW) dst[i] = src[i];
        rec4 = dst;
    } else {
        rec4 = reinterpret_cast<const uint4 *>(a.rec + base);
    }
    // R2: one line over the whole span at height 0 (bestfit.py:287-289)
    if (threadIdx.x == 0) {
        L[0].key = KO::make(0, 0); L[0].lop = 0; L[0].raw = 0;
        L[1].key = KO::make(0, a.U[t] - 1); L[1].lop = (uint32_t)n;  // sentinel
        L[1].raw = prune ? (uint32_t)a.tspan[t] : 0u;
        ss.done = 0;
    }
    if (NW > 1) __syncthreads();
    else __syncwarp();

    // leader-warp state (warp 0; uniform across its lanes)
    int nl = 1;
    HT peak = 0;
    Cnt steps = 0, lifts = 0;  // < 3n + 5 < 2^31 (n < 2^26)
    int placed = 0, status = PS_OK, maxl = 1;
    const Cnt bound = 3 * (Cnt)n + 4;
    // the lowest line is known without a scan after a place that leaves a
    // shoulder: the shoulder keeps the chosen (minimal) height and nothing
    // else at that height lies to its left
    bool known = true;
    int c = 0;
    K ck = KO::make(0, 0);
    HT hbase = 0;  // the last chosen height (a lower bound of every line's)
    HT hP = 0, hN = 0;
    bool hasP = false, hasN = false;
    uint32_t clop = 0, chip = 0, chi = 0, craw = 0, rawhi = 0;

    // timing: choose, query, update, retire phases; lift / place step totals
    long long tph[6] = {0, 0, 0, 0, 0, 0};
    long long tc = TIMING ? clock64() : 0, tstep = tc;
    for (;;) {
        // ======== leader: choose (R3) ========
        if (NW == 1 || warp == 0) {
            if (placed >= n || ++steps > bound) {
                if (placed < n) status = PS_LOOP_BOUND;  // R8
                if (NW == 1) break;  // one warp: leave right here
                if (lane == 0) ss.done = 1;
            } else {
                if (!known) {
                    if (STATS) nscan++;
                    if (nl <= 32) {
                        // lane i holds line i (time order), so the leftmost
                        // line of minimal height is the lowest lane whose
                        // height equals the warp minimum: one reduction
                        const K k = lane < nl ? L[lane].key : KO::none();
                        const HT hmin = KO::warp_min_h(KO::h(k));
                        c = __ffs(__ballot_sync(kFull, KO::h(k) == hmin && lane < nl)) - 1;
                        ck = KO::make(hmin, __shfl_sync(kFull, KO::lo(k), c));
                    } else if (sizeof(HT) == 4 && nl <= 128 && [&] {
                        // one reduction over (height relative to the last
                        // choice, saturated) << 7 | line: the lowest height
                        // never decreases; a saturated minimum falls back
                        constexpr uint32_t SAT = (1u << 25) - 1u;
                        uint32_t pk = 0xFFFFFFFFu;
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            const int i = lane + 32 * u;
                            if (i < nl) {
                                const uint32_t rel = (uint32_t)(KO::h(L[i].key) - hbase);
                                pk = min(pk, (min(rel, SAT) << 7) | (uint32_t)i);
                            }
                        }
                        const uint32_t km = __reduce_min_sync(kFull, pk);
                        if ((km >> 7) >= SAT) return false;
                        c = (int)(km & 127u);
                        ck = L[c].key;
                        return true;
                    }()) {
                    } else if (nl <= 128) {
                        // heights first (one reduction), then the leftmost
                        // line at that height (a second reduction over line
                        // indices); independent loads, depth-2 min trees
                        HT hr[4];
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            const int i = lane + 32 * u;
                            hr[u] = i < nl ? KO::h(L[i].key) : ~HT(0);
                        }
                        const HT hmin = KO::warp_min_h(min(min(hr[0], hr[1]), min(hr[2], hr[3])));
                        uint32_t ir[4];
#pragma unroll
                        for (int u = 0; u < 4; u++)
                            ir[u] = hr[u] == hmin ? (uint32_t)(lane + 32 * u) : 0xFFFFFFFFu;
                        c = (int)__reduce_min_sync(kFull, min(min(ir[0], ir[1]), min(ir[2], ir[3])));
                        ck = L[c].key;
                    } else {
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
                }
                hbase = KO::h(ck);
                hasP = c > 0;
                hasN = c + 1 < nl;
                const LR ln = L[c + 1];
                const K kp = hasP ? L[c - 1].key : KO::none();
                clop = L[c].lop;
                craw = L[c].raw;
                rawhi = ln.raw;
                chip = ln.lop;
                chi = KO::lo(ln.key);
                hN = KO::h(ln.key);
                hP = KO::h(kp);
                if (NW > 1 && lane == 0) {
                    ss.clop = clop; ss.chip = chip; ss.chi = chi; ss.rawhi = rawhi;
                }
            }
        }
        if (NW > 1) __syncthreads();  // [A] choice published
        if (NW > 1 && ss.done) break;

        if (TIMING) { const long long t2 = clock64(); tph[0] += t2 - tc; tc = t2; }
        // ======== all warps: query (R4) ========
        uint32_t qlop, qhip, qchi, qraw;
        if (NW > 1) { qlop = ss.clop; qhip = ss.chip; qchi = ss.chi; qraw = ss.rawhi; }
        else { qlop = clop; qhip = chip; qchi = chi; qraw = rawhi; }
        uint32_t lbest = kNone, wb = kNone;
        uint4 r0 = make_uint4(0, 0, 0, 0), r1 = make_uint4(0, 0, 0, 0);
        uint2 rw = make_uint2(0, 0);
        if (qlop < qhip) {
            const int c0 = (int)(qlop >> 5), c1 = (int)((qhip - 1) >> 5);
            wb = query_window<STATS, NW, TIER, LEAN, CLU>(win, rec4, raw2, pend, c0, c1, qchi,
                                                         qlop, qhip, qraw, prune, warp, lane,
                                                         lbest, r0, r1, rw, qs, a.rec_smem != 0);
        }
        uint32_t gbest;
        if (NW > 1) {
            if (lbest == wb && wb != kNone) {
                ss.wrec[warp][0] = r0;
                ss.wrec[warp][1] = r1;
                ss.wraw[warp] = rw;
            }
            if (lane == 0) ss.wbest[warp] = wb;
            __syncthreads();  // [B] per-warp winners published
            const uint32_t mine = lane < NW ? ss.wbest[lane] : kNone;
            gbest = __reduce_min_sync(kFull, mine);
            int ww = -1;
            if (gbest != kNone) ww = __ffs(__ballot_sync(kFull, mine == gbest)) - 1;
            if (gbest != kNone) {
                if (a.rec_smem) {
                    r0 = rec4[2 * gbest];
                    r1 = rec4[2 * gbest + 1];
                    rw = raw2[gbest];
                } else {
                    r0 = ss.wrec[ww][0];
                    r1 = ss.wrec[ww][1];
                    rw = ss.wraw[ww];
                }
            }
            if (ww == warp) {
                // the winning warp retires the entry while the leader
                // rewrites the skyline (both finish before barrier [A])
                const uint32_t pos = r0.x;
                retire_finish<STATS, TIER == TIER_SCAN>(
                    win, retire_load<(TIER < TIER_SKEL), TIER == TIER_SCAN>(win, pos, lane), pos,
                    lane);
            }
            if (warp != 0) continue;
        } else {
            gbest = wb;
            if (gbest != kNone && a.rec_smem) {
                r0 = rec4[2 * gbest];  // shared memory broadcast reads
                r1 = rec4[2 * gbest + 1];
                rw = raw2[gbest];
            } else if (gbest != kNone) {
                const int src = __ffs(__ballot_sync(kFull, lbest == gbest)) - 1;
                r0.x = __shfl_sync(kFull, r0.x, src);
                r0.y = __shfl_sync(kFull, r0.y, src);
                r0.z = __shfl_sync(kFull, r0.z, src);
                r0.w = __shfl_sync(kFull, r0.w, src);
                r1.x = __shfl_sync(kFull, r1.x, src);
                r1.y = __shfl_sync(kFull, r1.y, src);
                r1.z = __shfl_sync(kFull, r1.z, src);
                if (sizeof(HT) == 8) r1.w = __shfl_sync(kFull, r1.w, src);
                rw.x = __shfl_sync(kFull, rw.x, src);
                rw.y = __shfl_sync(kFull, rw.y, src);
            }
        }

        if (TIMING) { const long long t2 = clock64(); tph[1] += t2 - tc; tc = t2; }
        // ======== leader: replacement of lines [c, c+e] by m new lines ========
        K nk0 = 0, nk1 = 0, nk2 = 0;
        uint32_t np0 = 0, np1 = 0, np2 = 0, nr0 = 0, nr1 = 0, nr2 = 0;
        int m = 0, e = 0, cnext = c;
        RetireRow rr{};
        if (gbest == kNone) {
            // lift_up (R5)
            ++lifts;
            if (!hasP && !hasN) {  // lifting the only line (bestfit.py:185-186)
                status = PS_ILLEGAL_LIFT;
                placed = n;  // the loop ends at its next top check; this
            }                // step's harmless splice is discarded with the plan
            const bool intoN = !hasP || (hasN && hP > hN);
            const bool intoP = !intoN && (!hasN || hP < hN);
            e = intoP ? 0 : 1;
            m = intoN ? 1 : 0;
            nk0 = KO::make(hN, KO::lo(ck));
            np0 = clop;
            nr0 = craw;
            known = false;
        } else {
            // place (R6)
            const uint32_t rpos = r0.x, rar = r0.y, rfr = r0.z, rap = r0.w, rfp = r1.x,
                           rk = r1.y;
            if (NW == 1)  // the row read overlaps the skyline update
                rr = retire_load<(TIER < TIER_SKEL), TIER == TIER_SCAN, CLU>(win, rpos, lane);
            HT rsz = (HT)r1.z;
            if (sizeof(HT) == 8) rsz |= (HT)((uint64_t)r1.w << 32);
            const HT ch = KO::h(ck);
            const uint32_t clo = KO::lo(ck);
            const HT newh = ch + rsz;
            if (lane == 0) a.offsets[base + rk] = (int64_t)ch * unit;
            peak = max(peak, newh);
            ++placed;
            const bool hasL = clo < rar, hasR = rfr < chi;
            const bool mP = !hasL && hasP && hP == newh;  // flush re-merge (:171-174)
            const bool mN = !hasR && hasN && hN == newh;  // (:175-177)
            e = mN ? 1 : 0;
            const K kL = ck, kRa = KO::make(newh, rar), kR = KO::make(ch, rfr);
            // sequence: [L?] [raised unless merged into P] [R?]
            nk0 = hasL ? kL : (!mP ? kRa : kR);
            np0 = hasL ? clop : (!mP ? rap : rfp);
            nr0 = hasL ? craw : (!mP ? rw.x : rw.y);
            nk1 = hasL ? (!mP ? kRa : kR) : kR;
            np1 = hasL ? (!mP ? rap : rfp) : rfp;
            nr1 = hasL ? (!mP ? rw.x : rw.y) : rw.y;
            nk2 = kR;
            np2 = rfp;
            nr2 = rw.y;
            m = (hasL ? 1 : 0) + (mP ? 0 : 1) + (hasR ? 1 : 0);
            known = hasL || hasR;
            ck = hasL ? kL : kR;
            // index of the predicted next line: L stays at c; R follows raised
            cnext = hasL ? c : c + (mP ? 0 : 1);
        }

        // ---- apply: shift the tail [c+1+e, nl] (incl. sentinel) by d ----
        const int d = m - 1 - e;
        if (gbest != kNone && nl + d > lcap) {  // only a place grows the skyline
            status = PS_LINES_OVERFLOW;
            placed = n;
            continue;
        }
        if (d != 0 && nl < 32) {
            const int from = c + 1 + e;  // lines [from, nl] (incl. sentinel) move by d
            const bool mv = lane >= from && lane <= nl;
            LR v;
            if (mv) v = L[lane];
            __syncwarp();
            if (mv) L[lane + d] = v;
            __syncwarp();
        } else if (!LEAN && d != 0 && nl - (c + 1 + e) < 32) {
            // short tail of a long skyline (most shifts: the chosen line
            // sits near its end): one line per lane (single-trace kernels;
            // the register-capped batched loop measured slower with it)
            const int i = c + 1 + e + lane;
            const bool mv = i <= nl;
            LR v;
            if (mv) v = L[i];
            __syncwarp();
            if (mv) L[i + d] = v;
            __syncwarp();
        } else if (d != 0) {
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
            v.raw = lane == 0 ? nr0 : (lane == 1 ? nr1 : nr2);
            L[c + lane] = v;
        }
        nl += d;
        maxl = max(maxl, nl);
        c = cnext;
        if (TIMING) { const long long t2 = clock64(); tph[2] += t2 - tc; tc = t2; }
        if (NW == 1 && gbest != kNone)
            retire_finish<STATS, TIER == TIER_SCAN, CLU>(win, rr, r0.x, lane);
        __syncwarp();
        if (TIMING) {
            const long long t2 = clock64();
            tph[3] += t2 - tc;
            tph[gbest == kNone ? 4 : 5] += t2 - tstep;
            tc = tstep = t2;
        }
    }
    if (STATS && NW > 1) {
        if (lane == 0) {
            ss.wst[warp][0] = qs.wlive; ss.wst[warp][1] = qs.pass;
            ss.wst[warp][2] = qs.seg; ss.wst[warp][3] = qs.edge;
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int w = 1; w < NW; w++) {
                qs.wlive += ss.wst[w][0]; qs.pass += ss.wst[w][1];
                qs.seg += ss.wst[w][2]; qs.edge += ss.wst[w][3];
            }
    }
    if (threadIdx.x == 0) {
        a.peaks[t] = (int64_t)peak * unit;  // R7: max(offset + size)
        st[ST_STEPS] = steps;
        st[ST_LIFTS] = lifts;
        st[ST_MAXLINES] = maxl;
        st[ST_STATUS] = status;
        st[ST_WLIVE] = (int64_t)qs.wlive;
        st[ST_SCAN] = (int64_t)nscan;
        st[ST_PASS] = (int64_t)qs.pass;
        st[ST_SEG] = (int64_t)qs.seg;
        st[ST_EDGE] = (int64_t)qs.edge;
        for (int k = 0; k < 6; k++) st[ST_T0 + k] = tph[k];
    }
}

}  // namespace
}  // namespace mp
#include "warp_engine.cuh"
namespace mp {
namespace {

// ---- bulk copies (the TMA engine's cp.async.bulk) into shared memory ----
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
        "r"((uint32_t)__cvta_generic_to_shared(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;"
            " selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    }
}
// bulk copy of `bytes` (multiple of 16, 16-B aligned ends) in <= 64 KB pieces
__device__ __forceinline__ void bulk_copy(void *dst, const void *src, uint32_t bytes,
                                          uint64_t *bar) {
    for (uint32_t o = 0; o < bytes; o += 65536u)
        bulk_g2s(static_cast<char *>(dst) + o, static_cast<const char *>(src) + o,
                 min(65536u, bytes - o), bar);
}

// lifetimes in priority order for the cluster tier's pruning bound
__global__ void k_lifetimes(const uint2 *raw2, uint32_t *lt, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        lt[i] = raw2[i].y - raw2[i].x;
}

// Cluster tier: one thread-block cluster per trace.  Rank 0 runs the TIER_SKEL
// step loop (skeletons, lines, pending list in its own shared memory); ranks
// 1.. hold the chunk-sorted table and the lifetimes in theirs (staged with
// bulk copies) and serve them over DSMEM until the plan is done.
template <bool STATS>
__global__ void __launch_bounds__(32) k_plan_clu(PlanArgs a, int cl) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    cg::cluster_group cluster = cg::this_cluster();
    const uint32_t rank = cluster.block_rank();
    const int t = (int)(blockIdx.x / cl);
    if (rank > 0) {
        const int64_t base = a.trace_ptr[t];
        const int n = (int)(a.trace_ptr[t + 1] - base);
        const int nch = (n + 31) >> 5;
        const int64_t cb = chunk_base(base, t);
        const int cpc = 1 << a.clu_cshift, ppc = 1 << a.clu_pshift;
        const int j0 = (int)(rank - 1) * cpc, p0 = (int)(rank - 1) * ppc;
        const int jn = max(0, min(cpc, nch - j0)), pn = max(0, min(ppc, n - p0));
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            const uint32_t tb = 128u * (uint32_t)jn, lb = ((4u * (uint32_t)pn) + 15u) & ~15u;
            mbar_expect_tx(&bar, 2 * tb + lb);
            if (tb) {
                bulk_copy(smem, a.sf + 32 * (cb + j0), tb, &bar);
                bulk_copy(smem + 128 * cpc, a.sp + 32 * (cb + j0), tb, &bar);
            }
            if (lb) bulk_copy(smem + 256 * cpc, a.lt + base + p0, lb, &bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        cluster.sync();  // slices in place
        cluster.sync();  // the plan is done
        return;
    }
    cluster.sync();
    plan_trace<uint32_t, true, STATS, 1, TIER_SKEL, false, false, true>(a, t);
    cluster.sync();
}

// TIER_TINY planner: one warp per trace (grid = traces or tlist); packed
// choose keys when every height fits 27 bits
template <bool STATS>
__global__ void __launch_bounds__(32) k_tiny(PlanArgs a, const uint2 *ent, int packed) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int t = a.tlist ? a.tlist[blockIdx.x] : (int)blockIdx.x;
    if (packed) plan_tiny<true, STATS, !STATS>(a, ent, t, smem);
    else plan_tiny<false, STATS, !STATS>(a, ent, t, smem);
}

template <typename HT, bool LINES_SMEM, bool STATS, int NW, int TIER, bool TIMING>
__global__ void __launch_bounds__(32 * NW) k_plan(PlanArgs a) {
    plan_trace<HT, LINES_SMEM, STATS, NW, TIER, TIMING>(a, a.tlist ? a.tlist[blockIdx.x]
                                                                   : (int)blockIdx.x);
}

// Batched variant: capped at 128 registers (LEAN step loop, no spills) so
// 16 single-warp CTAs (traces) fit an SM — 4 warps per sub-partition's
// 16 K registers — instead of 9 for the uncapped kernel; the extra resident
// traces hide the step chain's latency (blocks/s: 9 -> 199 M, 12 at 168
// registers -> 285 M, 16 at 128 -> 307 M).  A lone trace is slower under the
// cap, so single traces keep the uncapped kernel.
constexpr int kOccCtas = 16;  // minBlocks hint that yields the 128-register cap
template <typename HT, bool LINES_SMEM, bool STATS, int TIER>
__global__ void __launch_bounds__(32, kOccCtas) k_plan_occ(PlanArgs a) {
    plan_trace<HT, LINES_SMEM, STATS, 1, TIER, false, true>(a, a.tlist ? a.tlist[blockIdx.x]
                                                                 : (int)blockIdx.x);
}

// Fused small-trace path: one CTA per trace runs K0 for its trace in shared
// memory (prep_small), then its warp 0 runs the TIER_SCAN step loop.
// One-warp CTAs (<= 128 blocks) are capped at 128 registers (no spill), so
// 16 traces share an SM (LSTM 4096 profiles: 0.118 -> 0.094 ms).
// The step loop is TIER_TINY (warp_engine.cuh) for 32-bit heights — a trace
// whose skyline outgrows its 31 register lines restarts right here on
// plan_trace TIER_SCAN — and TIER_SCAN for 64-bit heights (TINY = 0:
// TIER_SCAN only, the pre-r2 loop kept for A/B runs).
template <int THREADS, int ITEMS, bool STATS, int TINY>
__global__ void __launch_bounds__(THREADS, THREADS == 32 ? 16 : 1) k_fused_small(PlanArgs a, FusedIn in) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int t = (int)blockIdx.x;
    const int64_t n = a.trace_ptr[t + 1] - a.trace_ptr[t];
    if (n > 0)
        prep_small<THREADS, ITEMS>(a.trace_ptr, in, a.sf, a.sp, const_cast<Rec *>(a.rec),
                          const_cast<uint2 *>(a.raw2), t, smem);
    if (threadIdx.x >= 32) return;
    if (n == 0 || in.total_units[t] < (uint64_t(1) << 32)) {
        int st = PS_LINES_OVERFLOW;
        if constexpr (TINY > 0) {
            // block summaries where windows get long (traces > 512 blocks)
            constexpr bool SUM = THREADS == 256 && !STATS;
            st = in.total_units[t] < (uint64_t(1) << 27) ? plan_tiny<true, STATS, SUM>(a, in.ent, t, smem)
                                                         : plan_tiny<false, STATS, SUM>(a, in.ent, t, smem);
            __syncwarp();
        }
        if (st == PS_LINES_OVERFLOW) plan_trace<uint32_t, true, STATS, 1, TIER_SCAN, false, true>(a, t);
    } else {
        plan_trace<uint64_t, true, STATS, 1, TIER_SCAN, false, true>(a, t);
    }
}

constexpr int64_t kFusedMaxBlocks = 4096;

// Per-trace stats rows -> one row, on the device, so a batch of thousands of
// small traces returns 8 * (ST_N + 2) bytes instead of 8 * ST_N per trace.
// out[ST_STATUS] is the status of the first trace (in batch order) that
// failed with anything but a skyline overflow, out[ST_N] counts overflowed
// traces, out[ST_N + 1] is that first failing trace (or T).
constexpr int kRedThreads = 256;
__global__ void __launch_bounds__(kRedThreads) k_reduce_stats(const int64_t *st, int64_t T,
                                                              int64_t *out) {
    __shared__ int64_t part[kRedThreads];
    int64_t acc[ST_N], ovf = 0, first = T;
#pragma unroll
    for (int k = 0; k < ST_N; k++) acc[k] = 0;
    for (int64_t t = threadIdx.x; t < T; t += kRedThreads) {
        const int64_t *row = st + t * ST_N;
#pragma unroll
        for (int k = 0; k < ST_N; k++)
            if (k == ST_MAXLINES) acc[k] = max(acc[k], row[k]);
            else if (k != ST_STATUS) acc[k] += row[k];
        const int64_t stv = row[ST_STATUS];
        if (stv == PS_LINES_OVERFLOW) ovf++;
        else if (stv != PS_OK && t < first) first = t;
    }
    // one slot at a time through shared memory (ST_N + 2 small reductions)
    for (int k = 0; k < ST_N + 2; k++) {
        const int64_t v = k < ST_N ? acc[k] : (k == ST_N ? ovf : first);
        part[threadIdx.x] = v;
        __syncthreads();
        for (int o = kRedThreads / 2; o; o >>= 1) {
            if ((int)threadIdx.x < o) {
                const int64_t x = part[threadIdx.x], y = part[threadIdx.x + o];
                part[threadIdx.x] = (k == ST_MAXLINES) ? max(x, y)
                                  : (k == ST_N + 1)    ? min(x, y)
                                                       : x + y;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) out[k] = part[0];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[ST_STATUS] = out[ST_N + 1] < T ? st[out[ST_N + 1] * ST_N + ST_STATUS]
                                                             : PS_OK;
}

thread_local int64_t g_launches = 0;
thread_local int g_nwarps = 1;  // warps per trace chosen by plan_device
thread_local int g_carveout = -1;  // shared-memory carveout percent (-1: driver default)
thread_local bool g_occ = false;   // batched launch: use the register-capped k_plan_occ
// Function attributes are per process: setting them and launching is one
// critical section, so concurrent plans (pipelined halves, user threads)
// cannot lower each other's shared-memory opt-in between set and launch.
std::mutex g_launch_mu;

int sm_count(int device) {
    static int cache[64] = {0};
    int v = device >= 0 && device < 64 ? cache[device] : 0;
    if (!v) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
        if (device >= 0 && device < 64) cache[device] = v;
    }
    return v > 0 ? v : 148;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when the value for
// this kernel changes (a driver call per plan otherwise); callers hold
// g_launch_mu
struct AttrCache {
    const void *fn;
    int smem;
};
int set_smem_attr(const void *fn, int smem) {
    static AttrCache cache[64];
    static int used = 0;
    for (int i = 0; i < used; i++)
        if (cache[i].fn == fn) {
            if (cache[i].smem == smem) return MP_OK;
            MP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            cache[i].smem = smem;
            return MP_OK;
        }
    MP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (used < 64) cache[used++] = AttrCache{fn, smem};
    return MP_OK;
}

// per-thread events and a pinned reduced-stats buffer for the fused path
struct FusedCtx {
    cudaEvent_t k0 = nullptr, k1 = nullptr;
    int64_t *red_h = nullptr;
    int init() {
        if (k0) return MP_OK;
        MP_CUDA(cudaEventCreate(&k0));
        MP_CUDA(cudaEventCreate(&k1));
        MP_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&red_h), 256, cudaHostAllocDefault));
        return MP_OK;
    }
};
thread_local FusedCtx g_fctx;

template <typename HT, bool Ls, bool ST, int NW, int TIER, bool TM>
int launch_kt(const PlanArgs &a, int grid, size_t smem, cudaStream_t s) {
    auto fn = k_plan<HT, Ls, ST, NW, TIER, TM>;
    if constexpr (sizeof(HT) == 4 && Ls && NW == 1 && !TM) {
        if (g_occ) fn = k_plan_occ<HT, Ls, ST, TIER>;
    }
    // always opt in: dynamic + static shared memory may pass 48 KB even when
    // the dynamic part alone does not
    std::lock_guard<std::mutex> lock(g_launch_mu);
    MP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // keep only the shared memory the resident CTAs need: the rest is L1,
    // which caches the L2-resident window table between steps
    MP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, g_carveout));
    fn<<<grid, 32 * NW, smem, s>>>(a);
    MP_CUDA(cudaGetLastError());
    g_launches++;
    return MP_OK;
}

// Phase timing (MEMPLAN_TIMING) is compiled only into the single-warp,
// 32-bit-height, shared-memory-lines kernels that the latency study uses.
template <typename HT, bool Ls, bool ST, int NW, int TIER>
int launch_k(const PlanArgs &a, int grid, size_t smem, cudaStream_t s) {
    if constexpr (sizeof(HT) == 4 && Ls && !ST && NW == 1) {
        if (a.timing) return launch_kt<HT, Ls, ST, NW, TIER, true>(a, grid, smem, s);
    }
    return launch_kt<HT, Ls, ST, NW, TIER, false>(a, grid, smem, s);
}

template <typename HT, bool Ls, bool ST, int TIER>
int launch_nw(const PlanArgs &a, int grid, size_t smem, cudaStream_t s) {
    if (g_nwarps == 1) return launch_k<HT, Ls, ST, 1, TIER>(a, grid, smem, s);
    return launch_k<HT, Ls, ST, 8, TIER>(a, grid, smem, s);
}

template <typename HT, bool Ls, bool ST>
int launch_tier(const PlanArgs &a, int grid, int tier, size_t smem, cudaStream_t s) {
    switch (tier) {
        case TIER_SCAN: return launch_nw<HT, Ls, ST, TIER_SCAN>(a, grid, smem, s);
        case TIER_ALL: return launch_nw<HT, Ls, ST, TIER_ALL>(a, grid, smem, s);
        case TIER_SKEL: return launch_nw<HT, Ls, ST, TIER_SKEL>(a, grid, smem, s);
        case TIER_GROUP: return launch_nw<HT, Ls, ST, TIER_GROUP>(a, grid, smem, s);
        default: return launch_nw<HT, Ls, ST, TIER_GLOBAL>(a, grid, smem, s);
    }
}

template <typename HT, bool ST>
int launch_ht(const PlanArgs &a, int grid, int tier, bool lines_smem, size_t smem,
              cudaStream_t s) {
    if (lines_smem) return launch_tier<HT, true, ST>(a, grid, tier, smem, s);
    return launch_tier<HT, false, ST>(a, grid, tier, smem, s);
}

int launch_clu(const PlanArgs &a, int cl, size_t smem, bool stats, cudaStream_t s) {
    auto fn = stats ? k_plan_clu<true> : k_plan_clu<false>;
    std::lock_guard<std::mutex> lock(g_launch_mu);
    MP_TRY(set_smem_attr(reinterpret_cast<const void *>(fn), (int)smem));
    if (cl > 8) MP_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)cl);
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    MP_CUDA(cudaLaunchKernelEx(&cfg, fn, a, cl));
    g_launches++;
    return MP_OK;
}

int launch_tiny(const PlanArgs &a, const uint2 *ent, int grid, size_t smem, bool stats,
                bool packed, cudaStream_t s) {
    auto fn = stats ? k_tiny<true> : k_tiny<false>;
    std::lock_guard<std::mutex> lock(g_launch_mu);
    MP_TRY(set_smem_attr(reinterpret_cast<const void *>(fn), (int)smem));
    fn<<<grid, 32, smem, s>>>(a, ent, packed ? 1 : 0);
    MP_CUDA(cudaGetLastError());
    g_launches++;
    return MP_OK;
}

int launch_plan(const PlanArgs &a, int grid, bool h32, int tier, bool lines_smem, size_t smem,
                cudaStream_t s, bool stats) {
    if (stats)
        return h32 ? launch_ht<uint32_t, true>(a, grid, tier, lines_smem, smem, s)
                   : launch_ht<uint64_t, true>(a, grid, tier, lines_smem, smem, s);
    return h32 ? launch_ht<uint32_t, false>(a, grid, tier, lines_smem, smem, s)
               : launch_ht<uint64_t, false>(a, grid, tier, lines_smem, smem, s);
}

thread_local mp_plan_info g_info;

size_t smem_limit(int device) {
    static int cache[64] = {0};
    int v = device >= 0 && device < 64 ? cache[device] : 0;
    if (!v) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
        if (device >= 0 && device < 64) cache[device] = v;
    }
    return v > 0 ? (size_t)v : 48 * 1024;
}



inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

struct Layout {
    bool lines_smem, rec_smem;
    int tier;  // TIER_GLOBAL / TIER_SKEL / TIER_ALL
    size_t smem;
};

// Shared memory priority: skyline lines > pending list > chunk skeleton >
// chunk-sorted window table > winner records.
// per line: LineRec = packed key + LOP, 16 B (32 B for 64-bit heights)
size_t lines_bytes(int lcap, size_t hbytes) {
    const size_t lr = hbytes == 4 ? 16 : 32;
    return a16((size_t)(lcap + 1) * lr);
}

Layout choose_layout(int64_t nmax, int lcap, size_t hbytes, size_t lim, int nwarps,
                     bool force_global, bool lines_global = false, int max_tier = TIER_SCAN) {
    Layout l{};
    l.tier = TIER_GLOBAL;
    const size_t lines_b = lines_bytes(lcap, hbytes);
    const size_t pend_b = (size_t)nwarps * 2 * kPendCap * sizeof(uint32_t);
    const int64_t nch = (nmax + 31) / 32;
    const size_t grp_b = (size_t)((nch + 31) / 32) * 16;
    const size_t skel_b = (size_t)nch * 32 + a16((size_t)nch * 8);
    const size_t tab_b = (size_t)nch * 32 * 8;
    const size_t rec_b = (size_t)nmax * 40;  // records + raw alloc/free
    size_t used = pend_b + lt_bytes(nmax);
    if (!force_global) {
        if (!lines_global && used + lines_b <= lim) { l.lines_smem = true; used += lines_b; }
        if (max_tier >= TIER_GROUP && used + grp_b <= lim) {
            l.tier = TIER_GROUP;
            used += grp_b;
            if (max_tier >= TIER_SKEL && used + skel_b <= lim) {
                l.tier = TIER_SKEL;
                used += skel_b;
                if (max_tier >= TIER_ALL && used + tab_b <= lim) {
                    l.tier = TIER_ALL;
                    used += tab_b;
                    if (used + rec_b <= lim) { l.rec_smem = true; used += rec_b; }
                }
            }
        }
    }
    l.smem = used;
    // small traces: table + records in shared memory, no skeletons (scan)
    int64_t scan_max = kScanMaxBlocks;
    if (const char *env = getenv("MEMPLAN_SCAN_MAX")) scan_max = atoll(env);  // tuning
    if (!force_global && max_tier >= TIER_SCAN && nmax <= scan_max) {
        size_t u2 = pend_b + (l.lines_smem ? lines_b : 0);
        if (u2 + tab_b <= lim) {
            Layout sc = l;
            sc.tier = TIER_SCAN;
            u2 += tab_b;
            sc.rec_smem = u2 + rec_b <= lim;
            if (sc.rec_smem) u2 += rec_b;
            sc.smem = u2;
            return sc;
        }
    }
    return l;
}

}  // namespace

const mp_plan_info &last_plan_info() { return g_info; }
void set_plan_info(const mp_plan_info &info) { g_info = info; }

void *plan_workspace(size_t bytes, cudaStream_t s) {
    // one per thread and device; grown (never shrunk) on demand
    (void)s;
    static thread_local KeptBuffer ws[64];
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return nullptr;
    return ws[dev].get(bytes);
}

namespace {

// Fold per-trace planner statistics into g_info; map the status words to the
// reference's errors.
int collect_stats(const std::vector<int64_t> &hst, int64_t T) {
    for (int64_t t = 0; t < T; t++) {
        g_info.steps += hst[t * ST_N + ST_STEPS];
        g_info.lifts += hst[t * ST_N + ST_LIFTS];
        g_info.sum_wlive += hst[t * ST_N + ST_WLIVE];
        for (int k = 0; k < 4; k++) g_info.diag[k] += hst[t * ST_N + ST_SCAN + k];
        for (int k = 0; k < 6; k++) g_info.cycles[k] += hst[t * ST_N + ST_T0 + k];
        g_info.max_lines = std::max(g_info.max_lines, hst[t * ST_N + ST_MAXLINES]);
        const int64_t stv = hst[t * ST_N + ST_STATUS];
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

constexpr int kFusedFallback = -1;

template <int THREADS, int ITEMS, int TINY>
int launch_fused_l(const PlanArgs &a, const FusedIn &in, int grid, size_t smem, bool stats,
                   cudaStream_t s) {
    auto fn = stats ? k_fused_small<THREADS, ITEMS, true, TINY>
                    : k_fused_small<THREADS, ITEMS, false, TINY>;
    std::lock_guard<std::mutex> lock(g_launch_mu);
    MP_TRY(set_smem_attr(reinterpret_cast<const void *>(fn), (int)smem));
    fn<<<grid, THREADS, smem, s>>>(a, in);
    MP_CUDA(cudaGetLastError());
    g_launches++;
    return MP_OK;
}

// tiny = 0: the TIER_SCAN loop (A/B runs, MEMPLAN_NO_TINY)
template <int THREADS, int ITEMS>
int launch_fused(const PlanArgs &a, const FusedIn &in, int grid, size_t smem, bool stats,
                 int tiny, cudaStream_t s) {
    if (tiny) return launch_fused_l<THREADS, ITEMS, 1>(a, in, grid, smem, stats, s);
    return launch_fused_l<THREADS, ITEMS, 0>(a, in, grid, smem, stats, s);
}

// Traces of at most kFusedMaxBlocks blocks: one launch, no global sorts and
// no host round trip between K0 and the planner.  Returns kFusedFallback
// when the batch is not eligible or a skyline outgrew shared memory (the
// caller then takes the general path, which restarts such traces).
int plan_fused(const int64_t *trace_ptr_d, int64_t T, int64_t N, int64_t nmax,
               const int64_t *alloc_d, const int64_t *free_d, const int64_t *size_d,
               int64_t *offsets_d, int64_t *peaks_d, int flags, int device, cudaStream_t s,
               HostCopy *hc) {
    if (nmax > kFusedMaxBlocks || (flags & MP_FORCE_GLOBAL) || getenv("MEMPLAN_NO_FUSED"))
        return kFusedFallback;
    // CTA shape by size: one warp (the planner's own) for tiny traces, so the
    // register-heavy step loop does not cap residency; 256 threads for K0's
    // block sorts beyond that
    // (one-warp CTAs up to 256 blocks: LSTM L=64 profiles have 129)
    const int variant = nmax <= 128 ? 0 : nmax <= 256 ? 3 : nmax <= 512 ? 1 : nmax <= 2048 ? 2 : 4;
    const size_t prep_smem = variant == 0 ? sizeof(SmallPrep<32, 8>::Shared)
                           : variant == 3 ? sizeof(SmallPrep<32, 16>::Shared)
                           : variant == 1 ? sizeof(SmallPrep<128, 8>::Shared)
                           : variant == 2 ? sizeof(SmallPrep<256, 16>::Shared)
                                          : sizeof(SmallPrep<256, 32>::Shared);
    // planner layout (TIER_SCAN), sized for 64-bit heights so either fits
    const int sms = sm_count(device);
    // 2049-4096 blocks: one 256-thread CTA per SM (a 4096-key block sort in
    // shared memory) — single traces and small batches only; bigger batches
    // keep the 16-traces-per-SM batched kernel
    if (variant == 4 && T > sms) return kFusedFallback;
    const size_t lim = smem_limit(device) - 8192;  // two StepShared blocks + prep statics
    const int conc = (int)std::min<int64_t>((T + sms - 1) / sms, 8);
    const size_t budget = conc > 1 ? std::min(lim, (size_t)(228 * 1024) / conc - 8192) : lim;
    const int64_t lneed = 2 * nmax + 2;
    const int lcap = (int)std::min<int64_t>(lneed, conc > 1 ? 256 : 1024);
    Layout lay = choose_layout(nmax, lcap, 8, budget, 1, false);
    if (lay.tier != TIER_SCAN || !lay.lines_smem) return kFusedFallback;
    // step loop: TIER_WARP (register skyline) unless disabled (A/B runs)
    const int tiny = getenv("MEMPLAN_NO_TINY") ? 0 : 1;
    const size_t smem = std::max(std::max(prep_smem + 256, lay.smem),
                                 tiny ? tiny_smem_bytes(nmax) : size_t(0));
    if (smem > lim) return kFusedFallback;

    const int64_t nchunks = N / 32 + T + 1;
    const size_t bytes = 2 * Carver::need<uint32_t>(32 * nchunks) + Carver::need<Rec>(N) +
                         2 * Carver::need<uint2>(N) + Carver::need<uint32_t>(T) +
                         4 * Carver::need<int64_t>(T) + Carver::need<int64_t>(T * ST_N) +
                         Carver::need<int64_t>(ST_N + 2);
    void *ws = plan_workspace(bytes, s);
    if (!ws) return MP_ERR_CUDA;
    MP_TRY(g_fctx.init());
    Carver cv(ws, bytes);
    PlanArgs a{};
    FusedIn in{};
    a.trace_ptr = trace_ptr_d;
    a.sf = cv.take<uint32_t>(32 * nchunks);
    a.sp = cv.take<uint32_t>(32 * nchunks);
    Rec *rec = cv.take<Rec>(N);
    uint2 *raw2 = cv.take<uint2>(N);
    a.rec = rec;
    a.raw2 = raw2;
    in.ent = cv.take<uint2>(N);
    in.U = cv.take<uint32_t>(T);
    in.unit = cv.take<int64_t>(T);
    in.tmin = cv.take<int64_t>(T);
    in.tspan = cv.take<int64_t>(T);
    in.total_units = reinterpret_cast<uint64_t *>(cv.take<int64_t>(T));
    int64_t *stats = cv.take<int64_t>(T * ST_N);
    int64_t *red = cv.take<int64_t>(ST_N + 2);
    in.alloc = alloc_d;
    in.free_ = free_d;
    in.size = size_d;
    a.U = in.U;
    a.unit = in.unit;
    a.tspan = in.tspan;
    a.offsets = offsets_d;
    a.peaks = peaks_d;
    a.stats = stats;
    a.lcap = lcap;
    a.rec_smem = lay.rec_smem;
    const bool stats_on = (flags & MP_STATS) != 0;
    cudaEvent_t k0 = g_fctx.k0, k1 = g_fctx.k1;
    const int64_t launches0 = g_launches;
    cudaEventRecord(k0, s);
    int rc = variant == 0 ? launch_fused<32, 8>(a, in, (int)T, smem, stats_on, tiny, s)
           : variant == 3 ? launch_fused<32, 16>(a, in, (int)T, smem, stats_on, tiny, s)
           : variant == 1 ? launch_fused<128, 8>(a, in, (int)T, smem, stats_on, tiny, s)
           : variant == 2 ? launch_fused<256, 16>(a, in, (int)T, smem, stats_on, tiny, s)
                          : launch_fused<256, 32>(a, in, (int)T, smem, stats_on, tiny, s);
    if (rc != MP_OK) return rc;
    cudaEventRecord(k1, s);
    // one trace: its stats row is the reduction (no extra launch)
    if (T > 1) {
        k_reduce_stats<<<1, kRedThreads, 0, s>>>(stats, T, red);
        MP_CUDA(cudaGetLastError());
        g_launches++;
    }
    // host-array callers: their results ride the same round trip
    if (hc)
        for (int i = 0; i < hc->n; i++)
            if (hc->bytes[i])
                MP_CUDA(cudaMemcpyAsync(hc->dst[i], hc->src[i], hc->bytes[i],
                                        cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaMemcpyAsync(g_fctx.red_h, T > 1 ? red : stats,
                            sizeof(int64_t) * (T > 1 ? ST_N + 2 : ST_N), cudaMemcpyDeviceToHost,
                            s));
    MP_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> hst(g_fctx.red_h, g_fctx.red_h + ST_N + 2);
    if (T == 1) {  // the reduction's extra slots: overflowed traces, first failing trace
        hst[ST_N] = hst[ST_STATUS] == PS_LINES_OVERFLOW ? 1 : 0;
        hst[ST_N + 1] = hst[ST_STATUS] != PS_OK && hst[ST_STATUS] != PS_LINES_OVERFLOW ? 0 : 1;
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, k0, k1);
    if (hst[ST_N] > 0) return kFusedFallback;
    if (hc) hc->done = true;
    g_info.prep_ms = 0;
    g_info.plan_ms = ms;
    g_info.kernel_ms = ms;
    g_info.launches = g_launches - launches0;
    // 256: fused small-trace path; 512: TIER_TINY step loop
    g_info.engine = 8 | 2 | (lay.rec_smem ? 1 : 0) | 128 | 256 | (tiny ? 512 : 0);
    g_info.cluster = 1;
    return collect_stats(hst, 1);
}

}  // namespace

int plan_device(const int64_t *trace_ptr_d, const int64_t *trace_ptr_h, int64_t T,
                const int64_t *alloc_d, const int64_t *free_d, const int64_t *size_d,
                int64_t *offsets_d, int64_t *peaks_d, int flags, int device, cudaStream_t s,
                HostCopy *hc) {
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
    {
        const int rc = plan_fused(trace_ptr_d, T, N, nmax, alloc_d, free_d, size_d, offsets_d,
                                  peaks_d, flags, device, s, hc);
        if (rc != kFusedFallback) return rc;
        g_info = mp_plan_info{};
    }
    const int64_t nchunks = N / 32 + T + 1;
    const int64_t ngroups = nchunks / 32 + T + 1;
    const size_t prep_b = prep_scratch_bytes(N, T);
    const size_t tab_b = Carver::need<uint2>(N) + Carver::need<Rec>(N) +
                         Carver::need<uint32_t>(T) + Carver::need<int64_t>(T) +
                         Carver::need<uint64_t>(T) + Carver::need<int64_t>(T * ST_N) +
                         2 * Carver::need<uint4>(nchunks) + Carver::need<uint2>(nchunks) +
                         Carver::need<uint32_t>(nchunks) +
                         Carver::need<uint4>(ngroups) + Carver::need<uint2>(N) +
                         Carver::need<uint32_t>(N) + 2 * Carver::need<int64_t>(T) +
                         2 * Carver::need<uint32_t>(32 * nchunks);
    Scratch sc;
    MP_TRY(sc.alloc(prep_b + tab_b, s));
    Carver cv(sc.ptr, prep_b + tab_b);
    PrepOut po;
    po.ent = cv.take<uint2>(N);
    po.sf = cv.take<uint32_t>(32 * nchunks);
    po.sp = cv.take<uint32_t>(32 * nchunks);
    po.s0 = cv.take<uint4>(nchunks);
    po.s1 = cv.take<uint4>(nchunks);
    po.s2 = cv.take<uint2>(nchunks);
    po.nchunks = nchunks;
    po.gs = cv.take<uint4>(ngroups);
    po.ngroups = ngroups;
    po.cnt = cv.take<uint32_t>(nchunks);
    po.rec = cv.take<Rec>(N);
    po.raw2 = cv.take<uint2>(N);
    po.rawpos = cv.take<uint32_t>(N);
    po.tmin = cv.take<int64_t>(T);
    po.tspan = cv.take<int64_t>(T);
    po.U = cv.take<uint32_t>(T);
    po.unit = cv.take<int64_t>(T);
    po.total_units = cv.take<uint64_t>(T);
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

    // 32-bit heights when every trace's total bytes fit 2^32 size units
    std::vector<uint64_t> tot((size_t)T);
    MP_CUDA(cudaMemcpyAsync(tot.data(), po.total_units, sizeof(uint64_t) * T,
                            cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    bool h32 = true;
    for (int64_t t = 0; t < T; t++) h32 = h32 && tot[t] < (uint64_t(1) << 32);
    const size_t hb = h32 ? 4 : 8;

    // dynamic shared memory limit (the static StepShared block takes ~2.8 KB)
    const size_t lim = smem_limit(device) - 4096;
    const bool force_global = (flags & MP_FORCE_GLOBAL) != 0;
    const int64_t lneed = 2 * nmax + 2;  // worst case 2n+1 lines
    // Layout policy.  A single trace (or fewer traces than SMs) gets the
    // whole shared memory of its SM: latency is what matters.  A large batch
    // wants several traces resident per SM to hide the step chain's memory
    // latency, so each CTA is budgeted 1/conc of the SM's shared memory
    // (conc = traces per SM, capped) and the window structures take the
    // highest tier that fits that budget.
    const int sms = sm_count(device);
    // more than one trace per SM: the register-capped kernel, up to 16 per SM
    g_occ = T > sms;
    if (const char *env = getenv("MEMPLAN_OCC")) g_occ = atoi(env) != 0;
    int conc = (int)std::min<int64_t>((T + sms - 1) / sms, g_occ ? kOccCtas : 8);
    if (const char *env = getenv("MEMPLAN_CONC")) conc = std::max(1, std::min(32, atoi(env)));
    const int lcap_s = (int)std::min<int64_t>(lneed, conc > 1 ? 256 : 1024);
    const size_t budget =
        conc > 1 ? std::min(lim, (size_t)(228 * 1024) / conc - 1024 - 2048) : lim;
    g_nwarps = 1;
    Layout lay = choose_layout(nmax, lcap_s, hb, budget, 1, force_global);
    if (const char *env = getenv("MEMPLAN_NWARPS")) {
        const int v = atoi(env);
        if (v == 1 || v == 8) {
            g_nwarps = v;
            lay = choose_layout(nmax, lcap_s, hb, budget, v, force_global);
        }
    }
    if (const char *env = getenv("MEMPLAN_TIER")) {  // tuning: cap the shared-memory tier
        const int v = atoi(env);
        if (v >= TIER_GLOBAL && v < lay.tier)
            lay = choose_layout(nmax, lcap_s, hb, budget, g_nwarps, force_global, false, v);
    }
    if (getenv("MEMPLAN_DEBUG_LAYOUT"))
        fprintf(stderr, "memplan layout: nmax=%lld T=%lld nw=%d tier=%d lines_smem=%d rec_smem=%d "
                        "smem=%zu budget=%zu lim=%zu lcap=%d\n",
                (long long)nmax, (long long)T, g_nwarps, lay.tier, (int)lay.lines_smem,
                (int)lay.rec_smem, lay.smem, budget, lim, lcap_s);
    {
        const int64_t per_sm = std::max<int64_t>(1, (T + sms - 1) / sms);
        const double need = (double)per_sm * (double)(lay.smem + 1024 + sizeof(void *) * 256);
        int pct = (int)std::ceil(100.0 * need / (228.0 * 1024.0));
        g_carveout = std::min(100, std::max(0, pct));
    }

    PlanArgs a{};
    a.trace_ptr = trace_ptr_d;
    a.sf = po.sf;
    a.sp = po.sp;
    a.s0 = po.s0;
    a.s1 = po.s1;
    a.s2 = po.s2;
    a.gs = po.gs;
    a.cnt = po.cnt;
    a.rec = po.rec;
    a.raw2 = po.raw2;
    a.tspan = po.tspan;
    a.U = po.U;
    a.unit = po.unit;
    a.offsets = offsets_d;
    a.peaks = peaks_d;
    a.stats = stats;
    a.tlist = nullptr;
    a.lcap = lay.lines_smem ? lcap_s : (int)lneed;
    a.rec_smem = lay.rec_smem;
    a.timing = getenv("MEMPLAN_TIMING") != nullptr;
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
    // TIER_TINY (register skyline, warp_engine.cuh) for traces of up to
    // kTinyMaxBlocks blocks with 32-bit heights when no more traces than SMs;
    // traces whose skyline outgrows the 31 register lines come back as
    // PS_LINES_OVERFLOW and re-run below on plan_trace
    bool h27 = true;
    for (int64_t t = 0; t < T; t++) h27 = h27 && tot[t] < (uint64_t(1) << 27);
    const bool use_tiny = h32 && nmax <= kTinyMaxBlocks && T <= sms && !force_global &&
                          !a.timing && g_nwarps == 1 && !getenv("MEMPLAN_NO_TINY") &&
                          !getenv("MEMPLAN_TIER") && tiny_smem_bytes(nmax) <= lim;
    // Cluster tier (opt-in, MEMPLAN_CLUSTER=1): a single trace whose chunk
    // skeletons fit the SM but whose table does not (10^5 blocks) gets a
    // thread-block cluster — the planner CTA plus worker CTAs holding the
    // table and the lifetimes, read over DSMEM instead of L2.  Bit-exact, but
    // measured 9-10 % SLOWER than the L2-resident table at 10^5 (uniform
    // 363 vs 333 ms, cnn 268 vs 244 ms): the table is L2/L1-hot, DSMEM saves
    // little latency, and the placed-entry bitmap + address mapping cost more
    // (profiles/r2_summary.md)
    int clu = 0;
    size_t clu_smem = 0;
    if (!use_tiny && T == 1 && h32 && lay.tier == TIER_SKEL && lay.lines_smem && !a.timing &&
        g_nwarps == 1 && getenv("MEMPLAN_CLUSTER")) {
        const int64_t nch = (nmax + 31) / 32;
        const size_t lead = lay.smem + a16((size_t)nch * 4);
        for (int cl : {2, 4, 8, 16}) {
            const int64_t W = cl - 1;
            int cs = 0, ps = 0;
            while ((int64_t(1) << cs) * W < nch) cs++;
            while ((int64_t(1) << ps) * W < nmax) ps++;
            const size_t work = ((size_t)256 << cs) + ((size_t)4 << ps);
            if (work <= lim && lead <= lim) {
                clu = cl;
                a.clu_cshift = cs;
                a.clu_pshift = ps;
                clu_smem = std::max(lead, work);
                break;
            }
        }
    }
    Scratch lt_sc;
    if (use_tiny) {
        MP_TRY(launch_tiny(a, po.ent, (int)T, tiny_smem_bytes(nmax), stats_on, h27, s));
        lay.tier = TIER_WARP;
    } else if (clu) {
        MP_TRY(lt_sc.alloc(sizeof(uint32_t) * (size_t)(N + 8), s));
        a.lt = lt_sc.as<uint32_t>();
        k_lifetimes<<<std::min<int64_t>(1024, (N + 255) / 256), 256, 0, s>>>(po.raw2, lt_sc.as<uint32_t>(), N);
        MP_CUDA(cudaGetLastError());
        MP_TRY(launch_clu(a, clu, clu_smem, stats_on, s));
        lay.tier = TIER_CLU;
    } else {
        MP_TRY(launch_plan(a, (int)T, h32, lay.tier, lay.lines_smem, lay.smem, s, stats_on));
    }
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
        lay2 = choose_layout(nmax, b.lcap, hb, lim, g_nwarps, force_global, /*lines_global=*/true);
        b.rec_smem = lay2.rec_smem;
        Scratch lg;
        MP_TRY(lg.alloc(redo.size() * lines_bytes(b.lcap, hb), s));
        b.lines_g = lg.as<unsigned char>();
        MP_TRY(launch_plan(b, (int)redo.size(), h32, lay2.tier, false, lay2.smem, s, stats_on));
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
    const bool skel = lay.tier != TIER_SCAN && lay.tier != TIER_WARP && lay.tier != TIER_CLU;
    g_info.engine = (h32 ? 16 : 0) | (lay.lines_smem && lay.tier != TIER_WARP ? 8 : 0) |
                    (skel && lay.tier >= TIER_SKEL ? 4 : 0) |
                    (skel && lay.tier >= TIER_ALL ? 2 : 0) | (lay.rec_smem ? 1 : 0) |
                    (redo.empty() ? 0 : 32) | (skel && lay.tier >= TIER_GROUP ? 64 : 0) |
                    (lay.tier == TIER_SCAN ? 128 : 0) | (lay.tier == TIER_WARP ? 512 : 0) |
                    (lay.tier == TIER_CLU ? (1024 | 64 | 4) : 0);
    g_info.cluster = clu ? clu : g_nwarps;  // CTAs per trace (cluster tier) or warps per trace
    return collect_stats(hst, T);
}

}  // namespace mp
