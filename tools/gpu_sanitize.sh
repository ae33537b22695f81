# compute-sanitizer memcheck / racecheck / synccheck on the planner, validator
# and prep kernels over small traces (single and batched): TIER_TINY (single
# and fused — one-warp 128 / 256-block, 4 / 8-warp, 4096-block — incl. the
# staircase restart; k_tiny with block summaries), the LEAN batched kernel, and the
# cluster tier (DSMEM table, bulk-copy fills).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/san_case.py <<'PY'
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import numpy as np
import paper_1804_10001_b200 as mp
from paper_1804_10001_b200.bestfit import solve_bestfit_arrays, solve_bestfit_batched_arrays
from paper_1804_10001_b200.verifier import verify_arrays
from paper_1804_10001_b200.workloads import uniform_arrays
a, f, s = uniform_arrays(3000, 1); s = ((s + 511) // 512) * 512
off, pk = solve_bestfit_arrays(a, f, s)
solve_bestfit_arrays(a, f, s, flags=4)
r = verify_arrays(a, f, s, off)
assert r["n_violations"] == 0
inst = mp.profile_to_instance(mp.record(mp.parse_trace(mp.cnn_like_trace(mp.GenSpec(model="cnn", layers=500, seed=0)))), alignment=512)
solve_bestfit_arrays(*inst.arrays())
tp = np.array([0, 1000, 1500, 3000]); solve_bestfit_batched_arrays(tp, a, f, s)
k = np.arange(1200, dtype=np.int64); solve_bestfit_arrays(2 * k, 2 * k + 1, k + 1)
def batch(sizes, seed):
    cols = [uniform_arrays(n, seed + i) for i, n in enumerate(sizes)]
    cols = [(x, y, ((z + 511) // 512) * 512) for x, y, z in cols]
    tp = np.zeros(len(cols) + 1, np.int64); np.cumsum([len(c[0]) for c in cols], out=tp[1:])
    return tp, [np.concatenate([c[j] for c in cols]) for j in range(3)]
# fused path: one-warp (<= 128 blocks) and 4-warp CTAs, more traces than SMs
for sizes in ([13] * 300, [200] * 300, [400] * 200, [3500] * 8):
    tp, cat = batch(sizes, 7)
    solve_bestfit_batched_arrays(tp, *cat)
# register-capped LEAN batched kernel + composite / raw-rank K0 (N >= 2^16)
tp, cat = batch([2100] * 160, 11)
solve_bestfit_batched_arrays(tp, *cat)
# cluster tier (opt-in): planner CTA + worker CTAs, table over DSMEM, bulk-copy fills
os.environ["MEMPLAN_CLUSTER"] = "1"
a2, f2, s2 = uniform_arrays(40000, 3); s2 = ((s2 + 511) // 512) * 512
from paper_1804_10001_b200.bestfit import plan_info
off2, pk2 = solve_bestfit_arrays(a2, f2, s2)
assert plan_info()["engine"] & 1024, plan_info()
del os.environ["MEMPLAN_CLUSTER"]
off3, pk3 = solve_bestfit_arrays(a2, f2, s2)
assert pk2 == pk3 and (off2 == off3).all()
# k_tiny after the global K0 (block summaries for long windows)
os.environ["MEMPLAN_NO_FUSED"] = "1"
off4, pk4 = solve_bestfit_arrays(a, f, s)
assert pk4 == pk and (off4 == off).all()
del os.environ["MEMPLAN_NO_FUSED"]
print("case ok", pk, pk2)
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 3 python /tmp/san_case.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; tail -n 3 gpurun_out/san_$tool.log
done
