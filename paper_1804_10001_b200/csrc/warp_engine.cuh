// TIER_TINY — lean single-warp step loop for traces of at most
// kTinyMaxBlocks blocks (the per-network traces, the LSTM profiles).  Same
// rules as plan_trace (R1-R9, bestfit.py:276-309), different machine
// mapping: the skyline lives in REGISTERS (lane i = line i, the sentinel
// (t_hi, n) in lane nl), the window entries and winner records in shared
// memory, and every step is a short chain of warp collectives.
//
// Requirements: 32-bit heights (total units < 2^32), n <= kTinyMaxBlocks
// (priorities and positions < 2^12, time ranks < 2^16), at most 31 lines
// (more -> PS_LINES_OVERFLOW; the caller restarts the trace on plan_trace).
#pragma once

namespace mp {
namespace {

struct __align__(16) WRec {
    uint32_t ar, fr;  // alloc / free time rank
    uint32_t pp;      // LOP(alloc) | LOP(free) << 16
    uint32_t sz;      // size in units of the trace's gcd
};

// The loop, cut to its dependent chain:
//  * choose (R3) is ONE REDUX: lane i holds key (height << 5 | i) (heights
//    < 2^27 units; PACKED = false: the height relative to the last chosen
//    one, saturated, with a REDUX + ballot fallback);
//  * each line is (height, lo | LOP << 16): two SHFL fetch a line;
//  * window entries are (free rank << 12 | priority); a fitting entry at
//    position P bids (priority << 12 | P), so ONE REDUX names the winner AND
//    its position (retire without a ballot);
//  * offsets are kept per priority rank in shared memory and written out
//    once at the end (no global memory operation inside the loop).
// Chain per step: REDUX, SHFL, LDS (window), REDUX, LDS (record), SHFL
// (splice) — about 240 cycles plus the window's extra rounds.
// Beyond ~4096 blocks the windows (positions between LOP(lo) and LOP(hi),
// placed entries included) get long enough that the skeleton engine's
// pruning wins (a first register-skyline loop measured 1.6 vs 0.92 us per
// step at 10^4 uniform blocks).
constexpr int64_t kTinyMaxBlocks = 4096;
constexpr int kTinyBits = 12;
constexpr uint32_t kTinyMask = (1u << kTinyBits) - 1;

__host__ __device__ inline size_t tiny_smem_bytes(int64_t n) {
    // entries + offsets per priority (4 B each) + 16-B records
    return ((size_t)n * 8 + 15) / 16 * 16 + (size_t)n * sizeof(WRec);
}

// Block summaries (SUM): windows longer than 128 positions are mostly
// made of whole 64-position blocks, and nearly every live entry inside a
// long window fits it (Inception-ResNet-v2: 136 of 136 on average).  Lane i
// keeps, for blocks i and i + 32, the block's best live bid (priority << 12
// | position) ignoring fit, and that entry's free rank.  A long query then
// scans only its two partial edge blocks (one round of 4 loads per lane)
// and takes one summary per lane for the interior; a summary whose entry
// does not fit sends its block to a full scan (rare).  Summaries go stale
// when an entry of the block is retired: a 64-bit dirty mask marks the
// block and the next long query that covers it recomputes it (lazily, so
// short-window steps pay one OR).  Cuts the window rounds of IRv2 from
// 27 k to 10.5 k (tools/tiny_scan_sim.py).
constexpr int kSumBlk = 64;

template <bool PACKED, bool STATS, bool SUM = false>
__device__ __forceinline__ int plan_tiny(const PlanArgs &a, const uint2 *ent, const int t,
                                          unsigned char *smem) {
    constexpr unsigned full = 0xFFFFFFFFu;
    constexpr uint32_t NONE = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const int64_t base = a.trace_ptr[t];
    const int n = (int)(a.trace_ptr[t + 1] - base);
    int64_t *st = a.stats + (int64_t)t * ST_N;
    if (n == 0) {  // R1 (bestfit.py:285-286)
        if (lane == 0) {
            a.peaks[t] = 0;
            for (int k = 0; k < ST_N; k++) st[k] = 0;
            st[ST_STATUS] = PS_OK;
        }
        return PS_OK;
    }
    const int64_t unit = a.unit[t];
    uint32_t *went = reinterpret_cast<uint32_t *>(smem);
    uint32_t *offp = went + n;
    WRec *wrec = reinterpret_cast<WRec *>(smem + ((size_t)n * 8 + 15) / 16 * 16);
    const Rec *R = a.rec + base;
    for (int i = lane; i < n; i += 32) {
        const uint2 e = ent[base + i];
        went[i] = e.y == kDead ? NONE : ((e.x << kTinyBits) | e.y);
    }
    for (int p = lane; p < n; p += 32) {
        const uint4 *r4 = reinterpret_cast<const uint4 *>(R + p);
        const uint4 q0 = r4[0], q1 = r4[1];  // {pos, arank, frank, apos}, {fpos, k, size}
        wrec[p] = WRec{q0.y, q0.z, q0.w | (q1.x << 16), q1.z};
    }
    __syncwarp();

    // R2 (bestfit.py:287-289): line 0 = [t_lo, t_hi) at height 0; lane 1
    // holds the sentinel (t_hi, LOP n)
    uint32_t Lh = 0, Lq = lane == 1 ? ((a.U[t] - 1) | ((uint32_t)n << 16)) : 0u;
    int nl = 1, maxl = 1, placed = 0, status = PS_OK, steps = 0, lifts = 0;
    const int bound = 3 * n + 4;
    uint32_t peak = 0, hbase = 0;
    unsigned long long wlive = 0;
    // block summaries (SUM): all stale until first needed
    uint32_t sk0 = NONE, sf0 = 0, sk1 = NONE, sf1 = 0;
    unsigned long long dirty = ~0ull;

    bool illegal = false;
    while (placed < n && steps < bound && !illegal) {  // R8 (bestfit.py:297): checked below
        ++steps;
        // ---- choose (R3): lowest, then leftmost line ----
        int c;
        uint32_t ch;
        if (PACKED) {
            const uint32_t k = __reduce_min_sync(full, lane < nl ? (Lh << 5) | (uint32_t)lane : NONE);
            c = (int)(k & 31u);
            ch = k >> 5;
        } else {
            // heights relative to the last chosen height (the lowest height
            // never decreases), saturated at 2^27 - 1: one REDUX unless the
            // lowest line sits >= 2^27 units above the last one
            constexpr uint32_t SAT = (1u << 27) - 1u;
            const uint32_t k = __reduce_min_sync(full, lane < nl ? (min(Lh - hbase, SAT) << 5) | (uint32_t)lane : NONE);
            if ((k >> 5) < SAT) {
                c = (int)(k & 31u);
                ch = hbase + (k >> 5);
            } else {
                ch = __reduce_min_sync(full, lane < nl ? Lh : NONE);
                c = __ffs(__ballot_sync(full, lane < nl && Lh == ch)) - 1;
            }
            hbase = ch;
        }
        const uint32_t cq = __shfl_sync(full, Lq, c);
        const uint32_t nq = __shfl_sync(full, Lq, c + 1);
        const uint32_t hN = __shfl_sync(full, Lh, c + 1);
        const uint32_t hP = __shfl_sync(full, Lh, c > 0 ? c - 1 : 0);
        const bool hasP = c > 0, hasN = c + 1 < nl;
        const uint32_t clo = cq & 0xFFFFu, clop = cq >> 16, chi = nq & 0xFFFFu, chip = nq >> 16;

        // ---- query (R4): bids (priority << 12 | position) of fitting entries ----
        const uint32_t thr = (chi << kTinyBits) | kTinyMask;
        uint32_t bid = NONE;
        if (SUM && chip - clop > 128) {
            const uint32_t b0 = (clop + kSumBlk - 1) / kSumBlk, b1 = chip / kSumBlk;  // interior [b0, b1)
            // edges: [clop, b0 * 64) and [b1 * 64, chip), each < 64 positions
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint32_t p = u < 2 ? clop + 32 * u + lane : b1 * kSumBlk + 32 * (u - 2) + lane;
                const bool in = u < 2 ? p < b0 * kSumBlk : p < chip;
                const uint32_t ev = in ? went[p] : NONE;
                bid = ev <= thr ? min(bid, ((ev & kTinyMask) << kTinyBits) | p) : bid;
            }
            const unsigned long long imask = ((b1 >= 64 ? 0ull : (1ull << b1)) - 1ull) & ~((1ull << b0) - 1ull);
            unsigned long long need = dirty & imask;
            dirty &= ~need;
            while (need) {  // recompute stale summaries
                const int b = __ffsll((long long)need) - 1;
                need &= need - 1;
                uint32_t k = NONE;
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    const uint32_t p = (uint32_t)b * kSumBlk + 32 * u + lane;
                    const uint32_t ev = p < (uint32_t)n ? went[p] : NONE;
                    k = ev != NONE ? min(k, ((ev & kTinyMask) << kTinyBits) | p) : k;
                }
                k = __reduce_min_sync(full, k);
                const uint32_t fr = k == NONE ? 0u : went[k & kTinyMask] >> kTinyBits;
                if (lane == (b & 31)) {
                    if (b < 32) { sk0 = k; sf0 = fr; }
                    else { sk1 = k; sf1 = fr; }
                }
            }
            const bool i0 = (uint32_t)lane >= b0 && (uint32_t)lane < b1;
            const bool i1 = (uint32_t)lane + 32 >= b0 && (uint32_t)lane + 32 < b1;
            bid = i0 && sk0 != NONE && sf0 <= chi ? min(bid, sk0) : bid;
            bid = i1 && sk1 != NONE && sf1 <= chi ? min(bid, sk1) : bid;
            // a block whose best entry does not fit: scan it
            unsigned long long slow = 0;
            {
                const unsigned m0 = __ballot_sync(full, i0 && sk0 != NONE && sf0 > chi);
                const unsigned m1 = __ballot_sync(full, i1 && sk1 != NONE && sf1 > chi);
                slow = (unsigned long long)m0 | ((unsigned long long)m1 << 32);
            }
            while (slow) {
                const int b = __ffsll((long long)slow) - 1;
                slow &= slow - 1;
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    const uint32_t p = (uint32_t)b * kSumBlk + 32 * u + lane;
                    const uint32_t ev = went[p];
                    bid = ev <= thr ? min(bid, ((ev & kTinyMask) << kTinyBits) | p) : bid;
                }
            }
        } else
        for (uint32_t p0 = clop; p0 < chip; p0 += 128) {
            uint32_t e[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint32_t p = p0 + 32 * u + lane;
                e[u] = p < chip ? went[p] : NONE;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint32_t p = p0 + 32 * u + lane;
                bid = e[u] <= thr ? min(bid, ((e[u] & kTinyMask) << kTinyBits) | p) : bid;
                if (STATS) wlive += __popc(__ballot_sync(full, e[u] != NONE));
            }
        }
        const uint32_t wb = __reduce_min_sync(full, bid);

        // ---- update: lines [c, c+e] -> m new lines (h, lo | LOP << 16) ----
        uint32_t h0, h1 = 0, h2 = 0, q0, q1 = 0, q2 = 0;
        int m, e;
        if (wb == NONE) {
            // lift_up (R5, bestfit.py:180-201)
            ++lifts;
            // lifting the only line (bestfit.py:185-186) ends the loop at
            // its condition; this step's splice is discarded with the plan
            illegal = !hasP && !hasN;
            const bool intoN = !hasP || (hasN && hP > hN);
            const bool intoP = !intoN && (!hasN || hP < hN);
            e = intoP ? 0 : 1;
            m = intoN ? 1 : 0;
            h0 = hN;
            q0 = cq;
        } else {
            // place (R6, bestfit.py:149-178)
            const uint32_t pr = wb >> kTinyBits;
            const WRec r = wrec[pr];
            if (lane == 0) {
                went[wb & kTinyMask] = NONE;  // retire
                offp[pr] = ch;
            }
            if (SUM) dirty |= 1ull << ((wb & kTinyMask) / kSumBlk);
            const uint32_t newh = ch + r.sz;
            const uint32_t qa = r.ar | (r.pp << 16);                  // raised: lo = alloc
            const uint32_t qf = r.fr | ((r.pp >> 16) << 16);          // right shoulder: lo = free
            peak = max(peak, newh);
            ++placed;
            const bool hasL = clo < r.ar, hasR = r.fr < chi;
            const bool mP = !hasL && hasP && hP == newh;  // flush re-merge (:171-174)
            const bool mN = !hasR && hasN && hN == newh;  // (:175-177)
            e = mN ? 1 : 0;
            // sequence: [L?] [raised unless merged into P] [R?]
            h0 = hasL ? ch : (!mP ? newh : ch);
            q0 = hasL ? cq : (!mP ? qa : qf);
            h1 = hasL ? (!mP ? newh : ch) : ch;
            q1 = hasL ? (!mP ? qa : qf) : qf;
            h2 = ch;
            q2 = qf;
            m = (hasL ? 1 : 0) + (mP ? 0 : 1) + (hasR ? 1 : 0);
            // only a place can grow the skyline (a lift has d <= 0)
            if (nl + m - e > 32) {
                status = PS_LINES_OVERFLOW;
                break;
            }
        }
        const int d = m - 1 - e;
        // splice: lane i keeps its line (i < c), takes new line i - c
        // (i < c + m), or its old line i - d
        const uint32_t sh = __shfl_sync(full, Lh, (lane - d) & 31);
        const uint32_t sq = __shfl_sync(full, Lq, (lane - d) & 31);
        const int r = lane - c;
        const uint32_t nh = r == 0 ? h0 : (r == 1 ? h1 : h2);
        const uint32_t nq2 = r == 0 ? q0 : (r == 1 ? q1 : q2);
        if (r >= 0) {
            Lh = r < m ? nh : sh;
            Lq = r < m ? nq2 : sq;
        }
        nl += d;
        maxl = max(maxl, nl);
        __syncwarp();  // the retired entry is visible to the next scan
    }
    if (illegal) {
        status = PS_ILLEGAL_LIFT;
    } else if (status == PS_OK && placed < n) {  // R8: the bound ran out
        status = PS_LOOP_BOUND;
        steps = bound + 1;
    }
    __syncwarp();
    // offsets per block index (id order), one pass: offset = height * unit
    if (status == PS_OK)
        for (int p = lane; p < n; p += 32) a.offsets[base + R[p].k] = (int64_t)offp[p] * unit;
    if (lane == 0) {
        a.peaks[t] = (int64_t)peak * unit;  // R7: max(offset + size)
        st[ST_STEPS] = steps;
        st[ST_LIFTS] = lifts;
        st[ST_MAXLINES] = maxl;
        st[ST_STATUS] = status;
        st[ST_WLIVE] = (int64_t)wlive;
        for (int k = ST_SCAN; k < ST_N; k++) st[k] = 0;
    }
    return status;
}

}  // namespace
}  // namespace mp
