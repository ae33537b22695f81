"""Plan one golden 10^4 trace a few times (for ncu / timing)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1804_10001_b200.bestfit import solve_bestfit_arrays, plan_info
name = sys.argv[1] if len(sys.argv) > 1 else "cnn_1e4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
d = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "plans_large.npz"))
b = d[name + "_blocks"]
for r in range(reps):
    off, peak = solve_bestfit_arrays(b[:, 1], b[:, 2], b[:, 0], flags=flags)
    assert peak == int(d[name + "_peak"][0])
    print(name, plan_info(), flush=True)
