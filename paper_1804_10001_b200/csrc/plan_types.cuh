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

// Chunk-sorted window table (replaces a flat (alloc,id)-ordered table).
// Positions in (alloc, id) order are grouped into 32-entry chunks; within a
// chunk the entries are sorted by compressed free rank.  Per slot:
//   SF = (free_rank << 5) | position-within-chunk   (padding: 0xFFFFFFFF)
//   SP = priority rank, kDead once placed / padding
//   PM = inclusive prefix min of SP over the chunk's sorted slots
// A block fits a line iff free_rank <= hi, i.e. SF <= (hi << 5 | 31), so
// the fitting entries of a chunk are a prefix and their best priority is
// PM[count - 1].  Per chunk summary (uint4): min / max live free rank,
// best live priority (= PM[31]), live count.
// Chunk index of a trace's chunk j: (trace_base >> 5) + t + j (disjoint per
// trace for any CSR layout).
constexpr int kRankBits = 27;  // free ranks must stay below 2^27

__host__ __device__ inline int64_t chunk_base(int64_t trace_base, int64_t t) {
    return (trace_base >> 5) + t;
}

// Per-trace planner statistics slots.
enum { ST_STEPS = 0, ST_LIFTS = 1, ST_MAXLINES = 2, ST_STATUS = 3, ST_WLIVE = 4, ST_N = 5 };

// Planner status values written to stats[ST_STATUS].
enum { PS_OK = 0, PS_LOOP_BOUND = 2, PS_ILLEGAL_LIFT = 3, PS_LINES_OVERFLOW = 100 };

// Bytes of skyline storage per line slot: lo, hi, lop, hip (u32), prv, nxt
// (i32), height (i64).
constexpr int kLineBytes = 32;

}  // namespace mp
