"""Long randomised parity campaign (GPU): thousands of single traces and
batches across every planner path and tuning switch, each plan compared
with the C oracle (tests/ runs a shorter version of the same sweep).

    python tools/fuzz_campaign.py [seconds]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1804_10001_b200.bestfit import (PlanPipe, plan_info, solve_bestfit_arrays,  # noqa: E402
                                           solve_bestfit_batched_arrays)
from test_fuzz_gpu import KINDS, _trace  # noqa: E402

SWITCHES = [{}, {}, {}, {"MEMPLAN_NO_FUSED": "1"}, {"MEMPLAN_NO_TINY": "1"},
            {"MEMPLAN_TIER": "0"}, {"MEMPLAN_TIER": "2"}, {"MEMPLAN_DENSE_RANKS": "1"},
            {"MEMPLAN_NO_LOP": "1"}]
SIZES = [1, 2, 3, 13, 31, 32, 33, 64, 128, 129, 255, 256, 257, 511, 512, 513, 1000, 2047,
         2048, 2049, 3000, 4095, 4096, 4097, 6000, 12000]


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 240.0
    rng = np.random.default_rng(int(time.time()) & 0xFFFF)
    t_end = time.time() + budget
    singles = batches = piped = blocks = 0
    engines = set()
    while time.time() < t_end:
        sw = SWITCHES[rng.integers(len(SWITCHES))]
        for k, v in sw.items():
            os.environ[k] = v
        try:
            if rng.random() < 0.7:
                n = int(rng.choice(SIZES))
                kind = KINDS[rng.integers(len(KINDS))]
                a, f, s = _trace(rng, n, kind)
                off, pk = solve_bestfit_arrays(a, f, s)
                engines.add(plan_info()["engine"])
                ooff, opk = oracle.solve_bestfit(a, f, s)
                assert pk == opk and np.array_equal(off, ooff), ("single", n, kind, sw)
                singles += 1
                blocks += n
            else:
                T = int(rng.choice([2, 7, 60, 149, 300, 1000]))
                cap = int(rng.choice([20, 200, 2000, 5000]))
                sizes = rng.integers(0, cap, T)
                cols = [_trace(rng, int(m), KINDS[i % len(KINDS)]) if m else
                        (np.zeros(0, np.int64),) * 3 for i, m in enumerate(sizes)]
                tp = np.zeros(T + 1, np.int64)
                np.cumsum([len(c[0]) for c in cols], out=tp[1:])
                A, F, S = (np.concatenate([c[i] for c in cols]) for i in range(3))
                if rng.random() < 0.3:
                    with PlanPipe() as pipe:
                        off, pks = pipe.wait(pipe.submit(tp, A, F, S))
                    piped += 1
                else:
                    off, pks = solve_bestfit_batched_arrays(tp, A, F, S)
                engines.add(plan_info()["engine"])
                for t in rng.choice(T, size=min(T, 24), replace=False):
                    lo, hi = tp[t], tp[t + 1]
                    ooff, opk = oracle.solve_bestfit(A[lo:hi], F[lo:hi], S[lo:hi])
                    assert pks[t] == opk and np.array_equal(off[lo:hi], ooff), ("batch", T, t, sw)
                batches += 1
                blocks += int(tp[-1])
        finally:
            for k in sw:
                del os.environ[k]
    print(f"fuzz campaign ok: {singles} single traces, {batches} batches ({piped} through "
          f"PlanPipe), {blocks} blocks planned, engines seen {sorted(engines)}")


if __name__ == "__main__":
    main()
