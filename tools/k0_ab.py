"""K0 (prep) device time of the bench batch, median of several plans (A/B aid)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1804_10001_b200 import _native as N
from paper_1804_10001_b200.bestfit import check, plan_info
T = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
tp, A, F, S = bench.make_batch("uniform", 100000, T, 0, 16)
dev = torch.device("cuda")
d = [torch.from_numpy(x).to(dev) for x in (tp, A, F, S)]
off = torch.empty(len(A), dtype=torch.int64, device=dev); pk = torch.empty(T, dtype=torch.int64, device=dev)
lib = N.lib()
sh = torch.cuda.current_stream().cuda_stream
prep, plan = [], []
for i in range(8):
    check(lib.mp_plan_bestfit_batched(d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), d[3].data_ptr(), T,
                                      off.data_ptr(), pk.data_ptr(), N.MP_DEVICE_PTRS, 0, sh))
    if i >= 2:
        info = plan_info(); prep.append(info["prep_ms"]); plan.append(info["plan_ms"])
print("prep_ms median", statistics.median(prep), "min", min(prep), "plan_ms median", statistics.median(plan))
