"""Plan one layer-shape net trace a few times (for ncu): net batch reps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_10001_b200 as mp
from paper_1804_10001_b200.bestfit import solve_bestfit_arrays, plan_info
net, b = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
a, f, s = mp.profile_to_instance(mp.record(mp.parse_trace(mp.net_trace(net, b))), alignment=512).arrays()
for _ in range(reps):
    solve_bestfit_arrays(a, f, s)
print(net, b, len(a), plan_info())
