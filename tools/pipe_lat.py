import sys, time, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo")); sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests"))
import numpy as np, torch
from conftest import lstm_instances
from paper_1804_10001_b200.bestfit import PlanPipe, solve_bestfit_batched_arrays
tp, a, f, s = lstm_instances(6)
pin = [torch.from_numpy(x).pin_memory().numpy() for x in (a, f, s)]
outs = [(torch.empty(len(a), dtype=torch.int64).pin_memory().numpy(), torch.empty(len(tp)-1, dtype=torch.int64).pin_memory().numpy()) for _ in range(2)]
with PlanPipe() as pipe:
    for rep in range(3):
        t0 = time.perf_counter(); pend = []
        for k in range(50):
            if len(pend) == 2: pipe.wait(pend.pop(0))
            o, p = outs[k % 2]
            pend.append(pipe.submit(tp, *pin, offsets_out=o, peaks_out=p))
        for t in pend: pipe.wait(t)
        print("pipe ms/batch", (time.perf_counter() - t0) * 1e3 / 50)
    t0 = time.perf_counter()
    for k in range(50): pipe.wait(pipe.submit(tp, *pin, offsets_out=outs[0][0], peaks_out=outs[0][1]))
    print("pipe serial ms/batch", (time.perf_counter() - t0) * 1e3 / 50)
for rep in range(2):
    t0 = time.perf_counter()
    for k in range(50): solve_bestfit_batched_arrays(tp, *pin)
    print("sync ms/batch", (time.perf_counter() - t0) * 1e3 / 50)
