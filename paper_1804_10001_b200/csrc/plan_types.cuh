// Device-side data layout shared by the prep (K0) and planner (K1/K2)
// kernels.  See DESIGN.md "Data layout in HBM".
#pragma once
#include <stdint.h>

namespace mp {

// One block as the planner's winner lookup sees it, indexed by its priority
// rank (0 = best key).  Priority order is the reference's selection key
// (lifetime desc, size desc, id asc) — bestfit.py:216, :250-256 — computed
// once from RAW times (rule R4) so the device loop only
// compares 32-bit ranks.
struct __align__(16) Rec {
    uint32_t pos;    // position in (alloc, id) order  (bestfit.py:232)
    uint32_t arank;  // compressed alloc time
    uint32_t frank;  // compressed free time
    uint32_t apos;   // first (alloc,id)-position with alloc >= this alloc
    uint32_t fpos;   // first (alloc,id)-position with alloc >= this free
    uint32_t k;      // block index within its trace (id - 1)
    int64_t size;    // aligned size (core.py:216)
};
static_assert(sizeof(Rec) == 32, "Rec must stay 32 bytes");

// Window entry in (alloc, id) order: .x = compressed free time, .y = priority
// rank.  A placed block is overwritten with DEAD so it neither fits nor wins.
constexpr uint32_t kDead = 0xFFFFFFFFu;

// Chunk-sorted window table.
// Positions in (alloc, id) order are grouped into 32-entry chunks; within a
// chunk the entries are sorted by compressed free rank.  Per slot:
//   SF = (free_rank << 5) | position-within-chunk   (padding: 0xFFFFFFFF)
//   SP = priority rank, kDead once placed / padding
// A block fits a line iff free_rank <= hi, i.e. SF <= (hi << 5 | 31), so
// the fitting entries of a chunk are a PREFIX of its sorted slots.
//
// Chunk skeleton — enough to answer most chunks of a window query without
// touching SF/SP.  Per chunk (36 B, array-of-structs so one LDS.128 serves
// the common case):
//   S0 = {K0, A, P, K15}      (uint4)
//   S1 = {K7, K23, P7, P15}   (uint4)
//   S2 = {P23, RA}            (uint2; RA = raw alloc time of the chunk's
//                             first position relative to the trace origin)
//   K0        key of the first live slot (no live entry fits unless K0 <= thr)
//   A, P      key and priority of the chunk's best live entry: if A <= thr
//             the chunk's answer is exactly P
//   K7/15/23  keys at slots 7/15/23: locate the 8-slot segment where the
//             fitting prefix ends
//   P7/15/23  prefix minima of SP through slots 7/15/23
// Only the segment holding the boundary ever needs SF/SP (one 32-byte
// sector each), and only when its prefix minimum can still improve.
// Chunk index of a trace's chunk j: (trace_base >> 5) + t + j (disjoint per
// trace for any CSR layout).
//
// Group skeleton — the same idea one level up, per group of 32 chunks (1024
// positions): GS = {G0 = min K0, GA = key of the group's best live entry,
// GP = its priority, GR = raw alloc time of the group's first position
// relative to the trace origin}.  A window query first looks at whole groups: none
// fits (G0 > thr) -> skip 32 chunks; the group's best entry fits -> exact
// answer GP; otherwise scan the group's chunks.  Group index of a trace's
// group g: (chunk_base >> 5) + t + g.
constexpr int kRankBits = 27;  // free ranks must stay below 2^27

__host__ __device__ inline int64_t chunk_base(int64_t trace_base, int64_t t) {
    return (trace_base >> 5) + t;
}

__host__ __device__ inline int64_t group_base(int64_t trace_base, int64_t t) {
    return (chunk_base(trace_base, t) >> 5) + t;
}

#ifdef __CUDACC__
// Group skeleton of group g from its chunks' S0 (one warp; lane = chunk
// within the group, q = that chunk's S0 or all-ones past the trace end).
__device__ __forceinline__ void group_reduce(uint4 q, uint4 *gs, int64_t g, int lane) {
    constexpr unsigned full = 0xFFFFFFFFu;
    constexpr uint32_t none = 0xFFFFFFFFu;
    const uint32_t g0 = __reduce_min_sync(full, q.x);
    const uint32_t gp = __reduce_min_sync(full, q.z);
    const unsigned at = __ballot_sync(full, q.z == gp && gp != none);
    const uint32_t ga = at ? __shfl_sync(full, q.y, __ffs(at) - 1) : none;
    if (lane == 0) {  // GS.w (the group's raw alloc origin) is static: keep it
        uint32_t *d = reinterpret_cast<uint32_t *>(gs + g);
        d[0] = g0;
        d[1] = ga;
        d[2] = gp;
    }
}

__device__ __forceinline__ void group_store(const uint4 *s0, int64_t nch, uint4 *gs, int64_t g,
                                            int lane) {
    const int64_t j = 32 * g + lane;
    uint4 q = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0u);
    if (j < nch) q = s0[j];
    group_reduce(q, gs, g, lane);
}

// Rebuild and store the skeleton of chunk j from its sorted row (one warp;
// lane = sorted slot, `key` = SF, `pr` = SP with retired / padding slots at
// kDead).  Returns the live count.
__device__ __forceinline__ uint32_t skel_store(uint32_t key, uint32_t pr, int lane, uint4 *s0,
                                               uint4 *s1, uint2 *s2, int64_t j,
                                               uint4 *s0_out = nullptr) {
    constexpr unsigned full = 0xFFFFFFFFu;
    constexpr uint32_t none = 0xFFFFFFFFu;
    const unsigned live = __ballot_sync(full, pr != kDead);
    const uint32_t p7 = __reduce_min_sync(full, lane <= 7 ? pr : none);
    const uint32_t p15 = __reduce_min_sync(full, lane <= 15 ? pr : none);
    const uint32_t p23 = __reduce_min_sync(full, lane <= 23 ? pr : none);
    const uint32_t p = __reduce_min_sync(full, pr);
    const uint32_t k0 = live ? __shfl_sync(full, key, __ffs(live) - 1) : none;
    const unsigned at = __ballot_sync(full, pr == p && pr != kDead);
    const uint32_t a = at ? __shfl_sync(full, key, __ffs(at) - 1) : none;
    const uint32_t k7 = __shfl_sync(full, key, 7), k15 = __shfl_sync(full, key, 15),
                   k23 = __shfl_sync(full, key, 23);
    if (lane == 0) {
        s0[j] = make_uint4(k0, a, p, k15);
        s1[j] = make_uint4(k7, k23, p7, p15);
        s2[j].x = p23;  // S2.y (the chunk's raw alloc origin) is static
    }
    if (s0_out) *s0_out = make_uint4(k0, a, p, k15);
    return (uint32_t)__popc(live);
}
#endif

// Per-trace planner statistics slots.
// ST_SCAN..ST_EDGE are diagnostics counted only with MP_STATS: choose scans,
// skeleton passes, table segments read, edge rows read.
enum {
    ST_STEPS = 0, ST_LIFTS = 1, ST_MAXLINES = 2, ST_STATUS = 3, ST_WLIVE = 4,
    ST_SCAN = 5, ST_PASS = 6, ST_SEG = 7, ST_EDGE = 8,
    ST_T0 = 9,  // 6 slots: clock64() sums per phase / step kind with MEMPLAN_TIMING
    ST_N = 15
};

// Planner status values written to stats[ST_STATUS].
enum { PS_OK = 0, PS_LOOP_BOUND = 2, PS_ILLEGAL_LIFT = 3, PS_LINES_OVERFLOW = 100 };

}  // namespace mp
