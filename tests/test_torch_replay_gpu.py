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


def test_replay_safety_cases():
    """Real-memory rules of csrc/torch_alloc.cpp: a tensor held across an
    epoch boundary keeps its bytes; growth is side-served then re-planned on
    the GPU at the next boundary into a larger region; a reordered free of a
    grown block stops planned placement before it can alias; another stream
    is side-served; tensors outlive replay_end and release the region last."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "torch_replay_cases.py")],
                       capture_output=True, text=True, timeout=600)
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert lines, r.stderr[-3000:]
    out = json.loads(lines[-1])
    bad = [k for k, v in out.items() if isinstance(v, bool) and not v]
    assert not bad, (bad, out)


def test_floor_allocator_runs():
    """torch's pluggable front end alone (trivial hooks): the floor under
    the memplan hooks' through-torch cost."""
    out = _run("floor")
    assert out["ns_per_alloc"] > 0


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
