"""Single-trace plan latency per family/size and warps-per-trace (MEMPLAN_NWARPS),
bit-exact against the first run of each family (and the C oracle at n <= 2e4)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1804_10001_b200 as mp
from paper_1804_10001_b200.bestfit import solve_bestfit_arrays, plan_info
from paper_1804_10001_b200.workloads import uniform_arrays

sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "10000,100000").split(",")]
nws = (sys.argv[2] if len(sys.argv) > 2 else "1,8").split(",")
fams = sys.argv[3].split(",") if len(sys.argv) > 3 else ["uniform", "cnn"]
for n in sizes:
    for fam in fams:
        if fam == "uniform":
            a, f, s = uniform_arrays(n, 0); s = ((s + 511) // 512) * 512
        elif fam in ("alexnet", "googlenet", "resnet50", "inception_resnet_v2"):
            a, f, s = mp.profile_to_instance(mp.record(mp.parse_trace(mp.net_trace(fam, n))),
                                             alignment=512).arrays()
            n = len(a)
        else:
            a, f, s = mp.profile_to_instance(mp.record(mp.parse_trace(mp.cnn_like_trace(
                mp.GenSpec(model="cnn", layers=n // 2, seed=0)))), alignment=512).arrays()
        ref = None
        if n <= 20000:
            import oracle
            ref = oracle.solve_bestfit(a, f, s)
        for nw in nws:
            os.environ["MEMPLAN_NWARPS"] = nw
            best = 1e9
            for rep in range(3):
                off, pk = solve_bestfit_arrays(a, f, s)
                i = plan_info()
                best = min(best, i["kernel_ms"])
            if ref is None:
                ref = (off, pk)
            ok = np.array_equal(off, ref[0]) and pk == ref[1]
            solve_bestfit_arrays(a, f, s, flags=8)  # MP_STATS pass: diagnostics
            d = plan_info()
            os.environ["MEMPLAN_TIMING"] = "1"
            solve_bestfit_arrays(a, f, s)
            cyc = plan_info()["cycles"]
            del os.environ["MEMPLAN_TIMING"]
            print(f"{fam:8s} n={n:7d} nw={nw} kernel_ms={best:9.2f} steps={i['steps']} "
                  f"ns/step={1e6 * best / i['steps']:7.1f} engine={i['engine']} "
                  f"maxl={i['max_lines']} exact={ok} lifts={d['lifts']} "
                  f"wlive/step={d['sum_wlive'] / d['steps']:.0f} diag/step="
                  + " ".join(f"{k}={v / d['steps']:.2f}" for k, v in d['diag'].items())
                  + " cyc/step " + " ".join(f"{k}={v / d['steps']:.0f}" for k, v in cyc.items()
                                            if not k.endswith("_steps"))
                  + f" cyc/lift={cyc['lift_steps'] / max(1, d['lifts']):.0f}"
                  + f" cyc/place={cyc['place_steps'] / max(1, d['steps'] - d['lifts']):.0f}",
                  flush=True)
