"""The reference's OWN test suite (`memplan`'s tests: bestfit, verifier,
arena, core, profiler, workloads, acceptance) run against this package
through the import alias tests/refsuite/memplan.

The test files travel with the reference install (baseline/install_ref.sh
copies them to baseline/_ref/reftests; git-ignored, shipped to the GPU box).
Out of scope and not collected: test_cli.py, test_exact.py, test_svg.py
(CLI, exact solver, SVG — DESIGN.md §7).  Tests that call the exact solver
are SKIPPED by the alias's stubs; everything else — including the
step-by-step skyline tests against the host types in skyline.py — must
pass."""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REFTESTS = os.path.join(ROOT, "baseline", "_ref", "reftests")
OUT_OF_SCOPE = ("test_cli.py", "test_exact.py", "test_svg.py")
# the stubs' skip reasons: the only skips allowed
ALLOWED_SKIPS = ("solve_exact", "brute_force_peak")


def test_reference_suite_passes_against_the_dropin(tmp_path):
    if not os.path.isdir(REFTESTS):
        pytest.skip("baseline/_ref/reftests missing (run baseline/install_ref.sh)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join(
        [os.path.join(ROOT, "tests", "refsuite"), ROOT, env_path()]))
    cmd = [sys.executable, "-m", "pytest", REFTESTS, "-q", "-rs", "-p", "no:cacheprovider",
           "-o", "addopts="] + [f"--ignore={os.path.join(REFTESTS, f)}" for f in OUT_OF_SCOPE]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=str(tmp_path),
                       env=env)
    out = r.stdout + r.stderr
    summary = out.strip().splitlines()[-1] if out.strip() else ""
    print(summary)
    assert r.returncode == 0, out[-6000:]
    passed = int(re.search(r"(\d+) passed", summary).group(1))
    assert passed >= 100, summary
    for line in out.splitlines():
        if line.startswith("SKIPPED"):
            assert any(k in line for k in ALLOWED_SKIPS), line


def env_path():
    return os.environ.get("PYTHONPATH", "")
