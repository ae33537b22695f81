"""Single-trace latency vs warps-per-trace (MEMPLAN_NWARPS) at large n."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1804_10001_b200 as mp
from paper_1804_10001_b200.bestfit import solve_bestfit_arrays, plan_info
from paper_1804_10001_b200.workloads import uniform_arrays

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
fams = {}
a, f, s = uniform_arrays(n, 0); fams["uniform"] = (a, f, ((s + 511) // 512) * 512)
inst = mp.profile_to_instance(mp.record(mp.parse_trace(mp.cnn_like_trace(
    mp.GenSpec(model="cnn", layers=n // 2, seed=0)))), alignment=512)
fams["cnn"] = inst.arrays()
ref = {}
for name, (a, f, s) in fams.items():
    for nw in sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "4", "8", "16"]:
        os.environ["MEMPLAN_NWARPS"] = nw
        off, pk = solve_bestfit_arrays(a, f, s)
        if name in ref:
            assert np.array_equal(off, ref[name][0]) and pk == ref[name][1], (name, nw)
        else:
            ref[name] = (off, pk)
        i = plan_info()
        print(f"{name} n={n} nw={nw} kernel_ms={i['kernel_ms']:.1f} steps={i['steps']} "
              f"us/step={1e3 * i['kernel_ms'] / i['steps']:.3f} engine={i['engine']}", flush=True)
