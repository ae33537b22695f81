"""bench.py contract checks on a small workload: the one-line JSON schema at
N=1, and the N>1 code path (torchrun, rank 0 prints, max-over-ranks timing,
trace sharding and the rank-0 gather) run as two ranks on one GPU over gloo."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = ["--steps", "2", "--warmup", "3", "--blocks", "3000", "--traces", "64"]


def _last_json(out):
    lines = [x for x in out.splitlines() if x.startswith("{")]
    assert lines, out[-3000:]
    return json.loads(lines[-1])


def test_bench_json_contract_single_gpu():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *SMALL, "--no-cpu",
                        "--no-replay", "--no-suite"], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    d = _last_json(r.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["parity_vs_oracle"]["bit_exact"] is True
    assert d["parity_vs_oracle"]["traces_checked"] >= 16
    assert d["roofline"]["bound"] == "latency" and 0 < d["roofline"]["frac"] <= 1.2
    assert set(d["e2e"]) >= {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}
    assert set(d["roofline"]) >= {"bound", "achieved", "peak", "unit", "frac", "traffic"}


def test_bench_two_ranks_one_gpu():
    env = dict(os.environ, MEMPLAN_BENCH_BACKEND="gloo", MEMPLAN_BENCH_DEVICE="0")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29531", os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        *SMALL], capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["global_batch_traces"] == 128
    assert d["parity_vs_oracle"]["gathered_bit_exact"] is True


def test_bench_lstm_two_ranks_one_gpu():
    """configs[3] through dist.lpt_shards + gather_device with the GPU
    planner on every rank; rank 0 checks all 4096 gathered profiles against
    the C oracle."""
    env = dict(os.environ, MEMPLAN_BENCH_BACKEND="gloo", MEMPLAN_BENCH_DEVICE="0")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                        "--master-port", "29533", os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--workload", "lstm", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    d = _last_json(r.stdout)
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["parity_vs_oracle"]["bit_exact"] is True
    assert d["parity_vs_oracle"]["gathered_bit_exact"] is True


def test_bench_reference_arm_times_the_reference():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1", "--blocks", "2000"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    d = _last_json(r.stdout)
    assert d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "reference" and d["value"] > 0
