"""One large single-trace plan (for ncu): family n nwarps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_10001_b200 as mp
from paper_1804_10001_b200.bestfit import solve_bestfit_arrays, plan_info
from paper_1804_10001_b200.workloads import uniform_arrays
fam, n = sys.argv[1], int(sys.argv[2])
os.environ["MEMPLAN_NWARPS"] = sys.argv[3] if len(sys.argv) > 3 else "8"
if fam == "uniform":
    a, f, s = uniform_arrays(n, 0); s = ((s + 511) // 512) * 512
else:
    a, f, s = mp.profile_to_instance(mp.record(mp.parse_trace(mp.cnn_like_trace(
        mp.GenSpec(model="cnn", layers=n // 2, seed=0)))), alignment=512).arrays()
solve_bestfit_arrays(a, f, s)
print(fam, n, plan_info())
