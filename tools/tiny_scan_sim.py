"""Window-scan cost model of the TIER_TINY query (csrc/warp_engine.cuh) on a
per-network trace: replays the best-fit heuristic on the host (rules R3-R6,
bestfit.py:276-309) and counts query rounds of 128 positions for

  * the plain position scan over [LOP(lo), LOP(hi)), and
  * block summaries of B positions (the edges scanned, one summary per
    interior block, stale summaries recomputed lazily on demand).

    python tools/tiny_scan_sim.py inception_resnet_v2 128
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_10001_b200 as mp  # noqa: E402


def simulate(a, f, s, B):
    n = len(a)
    key = sorted(range(n), key=lambda i: (-(f[i] - a[i]), -s[i], i))
    prio = np.empty(n, int)
    prio[key] = np.arange(n)
    order = np.argsort(a, kind="stable")  # positions: alloc order
    A, F, P, S = a[order], f[order], prio[order], s[order]
    live = np.ones(n, bool)
    dirty = set(range((n + B - 1) // B))
    lines = [[int(a.min()), int(f.max()), 0]]
    placed = steps = lifts = fallbacks = 0
    old = new = 0.0
    while placed < n:
        steps += 1
        c = min(range(len(lines)), key=lambda i: (lines[i][2], i))
        lo, hi, h = lines[c]
        p0, p1 = np.searchsorted(A, lo), np.searchsorted(A, hi)
        w = p1 - p0
        old += max(1, -(-w // 128))
        if w <= 128:
            new += 1
        else:
            b0, b1 = -(-p0 // B), p1 // B
            new += 2  # edge round + summary read
            d = [x for x in dirty if b0 <= x < b1]
            new += len(d) * B / 128
            dirty.difference_update(d)
            for b in range(b0, b1):
                lv = live[b * B:(b + 1) * B]
                if lv.any():
                    cand = b * B + np.nonzero(lv)[0][np.argmin(P[b * B:(b + 1) * B][lv])]
                    if F[cand] > hi:
                        fallbacks += 1
                        new += B / 128
        fit = live[p0:p1] & (F[p0:p1] <= hi)
        if fit.any():
            idx = np.nonzero(fit)[0]
            best = p0 + idx[np.argmin(P[p0:p1][idx])]
            live[best] = False
            dirty.add(best // B)
            placed += 1
            al, fr = int(A[best]), int(F[best])
            seg = ([[lo, al, h]] if lo < al else []) + [[al, fr, h + int(S[best])]] + \
                  ([[fr, hi, h]] if fr < hi else [])
            lines[c:c + 1] = seg
            r = c + (1 if lo < al else 0)
            if r > 0 and lines[r - 1][2] == lines[r][2]:
                lines[r - 1:r + 1] = [[lines[r - 1][0], lines[r][1], lines[r][2]]]
                r -= 1
            if r + 1 < len(lines) and lines[r + 1][2] == lines[r][2]:
                lines[r:r + 2] = [[lines[r][0], lines[r + 1][1], lines[r][2]]]
        else:
            lifts += 1
            hp = lines[c - 1][2] if c > 0 else None
            hn = lines[c + 1][2] if c + 1 < len(lines) else None
            if hp is not None and hn is not None and hp == hn:
                lines[c - 1:c + 2] = [[lines[c - 1][0], lines[c + 1][1], hp]]
            elif hn is not None and (hp is None or hn < hp):
                lines[c:c + 2] = [[lo, lines[c + 1][1], hn]]
            else:
                lines[c - 1:c + 1] = [[lines[c - 1][0], hi, hp]]
    return dict(n=n, steps=steps, lifts=lifts, rounds_scan=old, rounds_summary=new,
                fallbacks=fallbacks)


if __name__ == "__main__":
    net, batch = sys.argv[1], int(sys.argv[2])
    a, f, s = mp.profile_to_instance(mp.record(mp.parse_trace(mp.net_trace(net, batch))),
                                     alignment=512).arrays()
    for B in (128, 64, 32):
        print(net, batch, "B", B, simulate(a, f, s, B))
