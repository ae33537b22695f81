"""ORACLE — TEST/BASELINE INFRASTRUCTURE ONLY (never imported by the product).

Python + numpy restatement of the reference ``solve_bestfit``
(/root/reference/pkg/src/memplan/bestfit.py:276-309) with the same algorithm
and the same vectorisation: a lazy min-heap over skyline lines keyed by
(height, time_lo) (bestfit.py:101-122), and the unplaced blocks sorted by
(alloc, id) queried with two searchsorted calls, a fit mask and the
three-stage (lifetime, size, -id) argmax (bestfit.py:243-262), compacted when
dead entries exceed half (bestfit.py:264-273).

Used as the ``--impl reference`` / ``cpu_baseline`` timing arm of bench.py:
it runs at the reference's own speed class (CPython + numpy, one thread per
trace), which is what BASELINE.md's CPU numbers were measured on.  Parity with
the C oracle and the golden vectors is checked in tests/test_oracle.py.
"""

from __future__ import annotations

import heapq

import numpy as np


def solve_bestfit_np(alloc, free, size):
    """(offsets int64[n] in id order, peak) — reference semantics R1-R8."""
    alloc = np.asarray(alloc, dtype=np.int64)
    free = np.asarray(free, dtype=np.int64)
    size = np.asarray(size, dtype=np.int64)
    n = len(alloc)
    offsets = np.zeros(n, dtype=np.int64)
    if n == 0:
        return offsets, 0
    # ---- skyline (parallel lists; a line is an index) ----
    lo_l = [int(alloc.min())]
    hi_l = [int(free.max())]
    h_l = [0]
    prv = [-1]
    nxt = [-1]
    alive = [True]
    heap = [(0, lo_l[0], 0, 0)]
    seq = 1

    def new_line(lo, hi, h):
        lo_l.append(lo); hi_l.append(hi); h_l.append(h)
        prv.append(-1); nxt.append(-1); alive.append(True)
        return len(lo_l) - 1

    def splice(first, last, repl):
        nonlocal seq
        before, after = prv[first], nxt[last]
        k = first
        while True:
            alive[k] = False
            if k == last:
                break
            k = nxt[k]
        for x, y in zip(repl, repl[1:]):
            nxt[x] = y
            prv[y] = x
        prv[repl[0]] = before
        nxt[repl[-1]] = after
        if before >= 0:
            nxt[before] = repl[0]
        if after >= 0:
            prv[after] = repl[-1]
        for r in repl:
            heapq.heappush(heap, (h_l[r], lo_l[r], seq, r))
            seq += 1

    # ---- remaining blocks (bestfit.py:231-241) ----
    order = np.lexsort((np.arange(n), alloc))
    r_alloc = alloc[order]
    r_free = free[order]
    r_life = r_free - r_alloc
    r_size = size[order]
    r_id = order.astype(np.int64)
    r_live = np.ones(n, dtype=bool)
    dead = 0
    sentinel = n + 1

    placed = steps = peak = 0
    while placed < n:
        steps += 1
        assert steps <= 3 * n + 4, "best-fit loop exceeded its iteration bound"
        while not alive[heap[0][3]]:
            heapq.heappop(heap)
        line = heap[0][3]
        lo, hi, h = lo_l[line], hi_l[line], h_l[line]
        # take_best
        i0 = int(np.searchsorted(r_alloc, lo, side="left"))
        i1 = int(np.searchsorted(r_alloc, hi, side="left"))
        pick = -1
        if i0 < i1:
            fits = r_live[i0:i1] & (r_free[i0:i1] <= hi)
            if fits.any():
                life = np.where(fits, r_life[i0:i1], -1)
                sz = np.where(life == life.max(), r_size[i0:i1], -1)
                ids = np.where(sz == sz.max(), r_id[i0:i1], sentinel)
                pick = i0 + int(ids.argmin())
        if pick < 0:
            p, q = prv[line], nxt[line]
            if p < 0 and q < 0:
                raise RuntimeError("IllegalLift")
            if p < 0:
                splice(line, q, [new_line(lo, hi_l[q], h_l[q])])
            elif q < 0:
                splice(p, line, [new_line(lo_l[p], hi, h_l[p])])
            elif h_l[p] == h_l[q]:
                splice(p, q, [new_line(lo_l[p], hi_l[q], h_l[p])])
            elif h_l[p] < h_l[q]:
                splice(p, line, [new_line(lo_l[p], hi, h_l[p])])
            else:
                splice(line, q, [new_line(lo, hi_l[q], h_l[q])])
            continue
        k = int(r_id[pick])
        r_live[pick] = False
        dead += 1
        a, f, s = int(alloc[k]), int(free[k]), int(size[k])
        repl = []
        if lo < a:
            repl.append(new_line(lo, a, h))
        raised = new_line(a, f, h + s)
        repl.append(raised)
        if f < hi:
            repl.append(new_line(f, hi, h))
        splice(line, line, repl)
        p = prv[raised]
        if p >= 0 and h_l[p] == h_l[raised]:
            merged = new_line(lo_l[p], hi_l[raised], h_l[raised])
            splice(p, raised, [merged])
            raised = merged
        q = nxt[raised]
        if q >= 0 and h_l[q] == h_l[raised]:
            splice(raised, q, [new_line(lo_l[raised], hi_l[q], h_l[raised])])
        offsets[k] = h
        peak = max(peak, h + s)
        placed += 1
        if dead * 2 > len(r_live):
            keep = r_live
            r_alloc, r_free, r_life = r_alloc[keep], r_free[keep], r_life[keep]
            r_size, r_id = r_size[keep], r_id[keep]
            r_live = np.ones(len(r_alloc), dtype=bool)
            dead = 0
    return offsets, peak
