"""Replay through PyTorch: memplan's CUDAPluggableAllocator hooks serve every
planned request at base + offset[lambda] inside ONE cudaMalloc'd region
(north_star), checked against the plan; the hook cost is measured next to
PyTorch's caching allocator (tools/replay_bench.py)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(alloc, layers=400, reps=3):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "replay_bench.py"), "--alloc",
                        alloc, "--layers", str(layers), "--reps", str(reps)],
                       capture_output=True, text=True, timeout=600)
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert lines, r.stderr[-2000:]
    return json.loads(lines[-1])


def test_pluggable_allocator_replays_the_plan():
    out = _run("memplan")
    assert out["addresses_match_plan"] is True
    assert out["outside_region"] == 0
    assert out["plan_peak_bytes"] < out["pool_peak_bytes"]
    assert out["hook_ns_per_alloc"] < 200


def test_caching_allocator_baseline_runs():
    out = _run("caching")
    assert out["ns_per_alloc"] > 0


def test_training_iteration_record_plan_replay():
    """Paper §4 end to end on a real PyTorch forward+backward: record one
    iteration through the hooks, plan it on the GPU, replay later iterations
    out of one region; results bit-identical to a cudaMalloc-per-tensor run."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "torch_model_replay.py"),
                        "--alloc", "memplan", "--batch", "8", "--width", "16", "--iters", "3"],
                       capture_output=True, text=True, timeout=900)
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert lines, r.stderr[-2000:]
    out = json.loads(lines[-1])
    assert out["replay_bit_identical"] is True
    assert out["requests_from_plan"] > 0
    # only the two checking epochs (which allocate comparison temporaries
    # after the profiled iteration) may leave the profile
    assert out["epochs_off_profile"] <= 2
    assert out["clique_lower_bound_bytes"] <= out["plan_peak_bytes"] <= out["pool_peak_bytes"]
