"""Plan latency of the per-network traces (configs[0..2]), 10^4-block single
traces and the LSTM profile batches (configs[3]), host to host and device,
bit-exact against the C oracle, next to the C oracle's own time on one core.

    python tools/small_lat.py            # current default engines
    MEMPLAN_NO_WARP=1 python tools/small_lat.py   # the pre-TIER_WARP loops
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_1804_10001_b200 as mp  # noqa: E402
from paper_1804_10001_b200.bestfit import (plan_info, solve_bestfit_arrays,  # noqa: E402
                                           solve_bestfit_batched_arrays)


def best_of(fn, reps):
    b = float("inf")
    r = None
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        b = min(b, time.perf_counter() - t0)
    return b, r


def main():
    from conftest import family_instance, lstm_instances
    cases = [(net, mp.profile_to_instance(mp.record(mp.parse_trace(mp.net_trace(net, b))),
                                          alignment=512).arrays())
             for net, b in [("alexnet", 32), ("googlenet", 64), ("resnet50", 64),
                            ("inception_resnet_v2", 128)]]
    for name in ("uniform_1e4_s0", "cnn_1e4_s0", "walk_1e4_s0"):
        cases.append((name, family_instance(name)))
    for name, (a, f, s) in cases:
        solve_bestfit_arrays(a, f, s)
        wall, (off, pk) = best_of(lambda: solve_bestfit_arrays(a, f, s), 7)
        info = plan_info()
        ow, (ooff, opk) = best_of(lambda: oracle.solve_bestfit(a, f, s), 3)
        ok = bool(np.array_equal(off, ooff) and pk == opk)
        print(f"{name:22s} n={len(a):6d} h2h={1e3 * wall:8.3f} ms dev={info['plan_ms'] + info['prep_ms']:8.3f} ms "
              f"steps={info['steps']:6d} ns/step={1e6 * info['plan_ms'] / max(1, info['steps']):6.1f} "
              f"engine={info['engine']} maxl={info['max_lines']} oracle={1e3 * ow:8.3f} ms "
              f"x_oracle={ow / wall:5.2f} exact={ok}", flush=True)
    for layers in (6, 64):
        tp, a, f, s = lstm_instances(layers)
        solve_bestfit_batched_arrays(tp, a, f, s)
        wall, (off, pks) = best_of(lambda: solve_bestfit_batched_arrays(tp, a, f, s), 7)
        info = plan_info()
        ok = True
        for t in range(0, len(tp) - 1, 37):
            o, p = oracle.solve_bestfit(a[tp[t]:tp[t + 1]], f[tp[t]:tp[t + 1]], s[tp[t]:tp[t + 1]])
            ok = ok and p == pks[t] and np.array_equal(o, off[tp[t]:tp[t + 1]])
        print(f"lstm_L{layers:<17d} T=4096 h2h={1e3 * wall:8.3f} ms dev={info['plan_ms'] + info['prep_ms']:8.3f} ms "
              f"engine={info['engine']} exact_sampled={ok}", flush=True)


if __name__ == "__main__":
    main()
