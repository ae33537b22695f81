"""Single-trace latency of the 10^5 reference families (device time of the
planner, best of 3), bit-exact against the reference digests (A/B aid)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import family_instance, sha64  # noqa: E402
from paper_1804_10001_b200.bestfit import plan_info, solve_bestfit_arrays  # noqa: E402
gold = {}
for fn in ("huge.json",):
    with open(os.path.join(ROOT, "tests", "golden", fn)) as fh:
        gold.update({c["name"]: c for c in json.load(fh)["cases"]})
for name in sys.argv[1:] or ["uniform_1e5_s0", "cnn_1e5_s0", "walk_1e5_s0"]:
    a, f, s = family_instance(name)
    best = None
    for _ in range(3):
        off, pk = solve_bestfit_arrays(a, f, s)
        ms = plan_info()["plan_ms"]
        best = ms if best is None else min(best, ms)
    g = gold.get(name, {})
    ok = g.get("peak") == pk and g.get("offsets_sha256") == sha64(off) if g else None
    print(f"{name:16s} plan {best:8.2f} ms  peak {pk}  matches_reference {ok}", flush=True)
