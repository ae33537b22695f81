"""Benchmark: best-fit planning throughput on B200 (blocks planned / s).

Workloads (`--workload`):
  uniform  (default; BASELINE.json configs[4], "synthetic random-lifetime
           traces ... vs host-CPU reference") every GPU plans --traces
           (default 2368 = 16 per SM) uniform-random-lifetime traces of
           --blocks (default 10^5) blocks (alloc ~ U[0,2n), free ~ U(alloc,2n],
           size ~ U[1,2^20] rounded to 512 B), seeded per rank -> weak scaling;
  cnn/walk the other two families of configs[4] (reference cli.py:208-224
           cnn-like generator; alloc/free random walk), --traces per GPU;
  lstm     BASELINE.json configs[3]: the 4096 variable-length LSTM seq2seq
           profiles (workloads.py:74-126, --lstm-layers 6 -> 13 blocks,
           64 -> 129 blocks per profile), ONE global batch sharded over the
           ranks by LPT (dist.py) -> strong scaling.
One step = one batched plan of the rank's traces (+ the rank-0 gather of
offsets and peaks when N > 1, the only collective).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload uniform|cnn|walk|lstm]

`value` is device-timed with inputs resident in HBM (inputs > L2 per step
for the 10^5 families, so no flush is needed; the LSTM batch is L2-resident
and says so in `config`); `e2e` goes through the public pipelined C ABI
(`mp_pipe_submit` / `mp_pipe_wait`) with pinned host buffers — K batches,
each with its H2D and D2H inside the timed region, two in flight — and
`e2e.sync_call` through one `mp_plan_bestfit_batched` call per batch.  Parity: >= 16 traces
spread over the batch (all 4096 for lstm) against the C oracle, and after
N > 1 runs the GATHERED results on rank 0.  The reference arm
(`--impl reference`) times the unmodified reference `memplan.solve_bestfit`
installed in baseline/_ref (baseline/install_ref.sh) on the host cores.
"""

from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "blocks planned/sec and plan latency (bit-exact peak bytes); replay ns/alloc"
UNIT = "blocks/s"
ALIGN = 512
N_SMS = 148


# ---------------------------------------------------------------------------
# workloads (the product's own generators; the same code makes the reference
# fixtures' instances, see tests/golden/make_huge_golden.py)
# ---------------------------------------------------------------------------
def _align(s):
    return ((s + ALIGN - 1) // ALIGN) * ALIGN


def gen_trace(fam: str, n: int, seed: int):
    """(alloc, free, size) int64 columns in id order, sizes aligned to 512."""
    from paper_1804_10001_b200.workloads import uniform_arrays, uniform_blocks, walk_trace
    from paper_1804_10001_b200.profiler import ingest_arrays
    import paper_1804_10001_b200 as mp
    if fam == "uniform":  # numpy draw (large batches)
        a, f, s = uniform_arrays(n, seed)
        return a, f, _align(s)
    if fam == "uniform_rr":  # random.Random draw (reference fixtures)
        b = np.asarray(uniform_blocks(n, seed), np.int64)
        return b[:, 1].copy(), b[:, 2].copy(), _align(b[:, 0])
    if fam == "cnn":
        txt = mp.cnn_like_trace(mp.GenSpec(model="cnn", layers=n // 2, seed=seed))
    elif fam == "walk":
        txt = walk_trace(n, seed)
    else:
        raise ValueError(fam)
    a, f, s = ingest_arrays(txt, alignment=ALIGN)[:3]
    return a, f, s


def _gen_one(args):
    return gen_trace(*args)


def csr(cols):
    tp = np.zeros(len(cols) + 1, np.int64)
    np.cumsum([len(c[0]) for c in cols], out=tp[1:])
    cat = lambda i: np.concatenate([c[i] for c in cols])  # noqa: E731
    return tp, cat(0), cat(1), cat(2)


def trace_seed(rank: int, t: int) -> int:
    return (rank + 1) * 100003 + t


def make_batch(fam: str, n: int, traces: int, rank: int, procs: int):
    """CSR batch of `traces` traces of family `fam` for `rank` (weak scaling)."""
    jobs = [(fam, n, trace_seed(rank, t)) for t in range(traces)]
    if fam == "uniform" or traces <= 2:
        return csr([gen_trace(*j) for j in jobs])
    import multiprocessing as mpc
    with mpc.get_context("fork").Pool(procs) as pool:
        return csr(pool.map(_gen_one, jobs, chunksize=4))


def lstm_batch(layers: int):
    """configs[3]: the 4096 profiles as one CSR batch (id order per profile)."""
    from paper_1804_10001_b200.workloads import lstm_profiles
    from paper_1804_10001_b200.profiler import ingest_arrays
    return csr([ingest_arrays(t, alignment=ALIGN)[:3]
                for t in lstm_profiles(4096, layers=layers, batch=64)])


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.int64).tobytes()).hexdigest()


def golden_huge() -> dict:
    out = {}
    for name in ("huge.json", "huge_lstm.json"):
        try:
            with open(os.path.join(ROOT, "tests", "golden", name)) as fh:
                out.update({c["name"]: c for c in json.load(fh)["cases"]})
        except (OSError, ValueError, KeyError):
            pass
    return out


# ---------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md "clocks DURING the timed region")
# ---------------------------------------------------------------------------
class Clocks:
    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        q = self.q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.thread.join(timeout=2)
        if not self.rows:  # a timed region shorter than one sampling period
            try:
                r = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.q}",
                                    "--format=csv,noheader,nounits"], capture_output=True,
                                   text=True, timeout=30)
                self.rows = [[x.strip() for x in line.split(",")]
                             for line in r.stdout.splitlines() if line.strip()]
            except (OSError, subprocess.SubprocessError):
                pass
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, name in enumerate(names):
                if len(r) > 3 + k and r[3 + k].lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# CPU arms: the reference itself (baseline/_ref) and the numpy port (oracle/)
# ---------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _ref_module():
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import memplan  # the unmodified reference package
    return memplan


def _ref_solve(cols):
    """Time memplan.solve_bestfit (bestfit.py:276) on each (a, f, s)."""
    M = _ref_module()
    t_solve = 0.0
    for a, f, s in cols:
        inst = M.build_instance(list(zip(s.tolist(), a.tolist(), f.tolist())), alignment=ALIGN)
        t0 = time.perf_counter()
        M.solve_bestfit(inst)
        t_solve += time.perf_counter() - t0
    return t_solve


def _port_solve(cols):
    from oracle.bestfit_np import solve_bestfit_np
    t = 0.0
    for a, f, s in cols:
        t0 = time.perf_counter()
        solve_bestfit_np(a, f, s)
        t += time.perf_counter() - t0
    return t


def cpu_sample(kind: str, groups: list) -> tuple[float, float]:
    """Plan every group of traces in its own process, all in parallel;
    returns (wall seconds, mean per-process solve seconds)."""
    import multiprocessing as mpc
    fn = _ref_solve if kind == "reference" else _port_solve
    with mpc.get_context("fork").Pool(len(groups)) as pool:
        t0 = time.perf_counter()
        per = pool.map(fn, groups)
        wall = time.perf_counter() - t0
    return wall, statistics.mean(per)


def cpu_groups(args, procs: int, k: int):
    """One bounded sample of the workload: `procs` traces (one per core), or
    the whole LSTM profile batch split over the cores."""
    if args.workload == "lstm":
        tp, A, F, S = lstm_batch(args.lstm_layers)
        cols = [(A[tp[t]:tp[t + 1]], F[tp[t]:tp[t + 1]], S[tp[t]:tp[t + 1]])
                for t in range(len(tp) - 1)]
        return [cols[i::procs] for i in range(procs)], int(len(A))
    cols = [gen_trace(args.workload, args.n, 7_000_000 + 1000 * k + i) for i in range(procs)]
    return [[c] for c in cols], procs * args.n


def run_reference(args, rank: int, world: int):
    """`--impl reference`: the unmodified reference memplan.solve_bestfit on
    the host cores, rank 0 only; each step one bounded sample of the same
    workload (steps stop early at --ref-budget seconds, >= 1 step)."""
    if rank != 0:
        return
    try:
        _ref_module()
    except ImportError as exc:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"baseline/_ref missing ({exc}); run baseline/install_ref.sh"}))
        return
    procs = min(host_cores(), args.cpu_procs)
    small = [[gen_trace("uniform", 300, i)] for i in range(procs)]
    for _ in range(min(args.warmup, 3)):
        cpu_sample("reference", small)
    vals, walls, t_start, blocks = [], [], time.perf_counter(), 0
    for k in range(args.steps):
        groups, blocks = cpu_groups(args, procs, k)
        wall, _ = cpu_sample("reference", groups)
        vals.append(blocks / wall)
        walls.append(wall)
        if time.perf_counter() - t_start > args.ref_budget:
            break
    value = float(np.median(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": len(vals), "steps_requested": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.median(walls)), "higher_is_better": True,
        "scaling": "strong" if args.workload == "lstm" else "weak", "vs_baseline": None,
        "dtype": "int64", "data": "synthetic", "config": bench_config(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs, "kind": "reference",
                         "cpu": cpu_model(),
                         "sample": (f"{blocks} blocks per step: " +
                                    ("the 4096 LSTM profiles split over the cores"
                                     if args.workload == "lstm" else
                                     f"{procs} {args.workload} traces x {args.n} blocks, one "
                                     f"per process") +
                                    "; unmodified memplan.solve_bestfit from baseline/_ref "
                                    "(build_instance outside the timed solve)")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# parity (outside the timed region): the C oracle, one trace per process
# ---------------------------------------------------------------------------
def _oracle_one(job):
    import oracle
    a, f, s, off, pk = job
    o, p = oracle.solve_bestfit(a, f, s)
    return bool(np.array_equal(o, off) and p == pk)


def oracle_check(tp, A, F, S, off, pks, traces, procs) -> bool:
    jobs = [(A[tp[t]:tp[t + 1]], F[tp[t]:tp[t + 1]], S[tp[t]:tp[t + 1]],
             off[tp[t]:tp[t + 1]], int(pks[t])) for t in traces]
    if len(jobs) <= 1:
        return all(_oracle_one(j) for j in jobs)
    import multiprocessing as mpc
    with mpc.get_context("fork").Pool(min(procs, len(jobs))) as pool:
        return all(pool.map(_oracle_one, jobs))


def spread(T: int, k: int) -> list:
    """k trace indices spread evenly over [0, T) (first and last included)."""
    if T <= k:
        return list(range(T))
    return sorted({int(round(i * (T - 1) / (k - 1))) for i in range(k)})


# ---------------------------------------------------------------------------
# step-latency floor (tools/ubench/step_floor.cu), measured live
# ---------------------------------------------------------------------------
def step_floor(variant: int, ctas: int, iters: int = 20000):
    path = os.path.join(ROOT, "tools", "ubench", "libstepfloor.so")
    try:
        lib = ctypes.CDLL(path)
    except OSError:
        return None
    cyc, sps = ctypes.c_double(), ctypes.c_double()
    rc = lib.step_floor(variant, ctas, iters, ctypes.byref(cyc), ctypes.byref(sps))
    if rc != 0:
        return None
    return {"cycles_per_step": cyc.value, "steps_per_s": sps.value}


# ---------------------------------------------------------------------------
# BASELINE.json configs[0..3] + the single-trace sweep of configs[4]
# ---------------------------------------------------------------------------
def _best_wall(fn, reps):
    best = float("inf")
    r = None
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        best = min(best, time.perf_counter() - t0)
    return best, r


def _lstm_cpu_one(traces):
    from oracle.bestfit_np import solve_bestfit_np
    for a, f, s in traces:
        solve_bestfit_np(a, f, s)
    return len(traces)


def config_suite(cpu_procs: int, sweep_1e6: bool) -> dict:
    """Plan latency host-to-host and device-side for the per-network traces
    (configs[0..2]), the LSTM profile batches (configs[3], L=6 and L=64, all
    4096 checked in full against the C oracle and against the reference's
    own digest) and single traces of configs[4] at 10^5 / 10^6 (checked
    against the reference's sha256 digests, tests/golden/huge.json)."""
    import oracle
    import paper_1804_10001_b200 as mp
    from paper_1804_10001_b200.bestfit import (solve_bestfit_arrays, plan_info,
                                               solve_bestfit_batched_arrays)
    from oracle.bestfit_np import solve_bestfit_np
    out = {}
    gold = golden_huge()
    cases = [("alexnet_mb32", "alexnet", 32), ("googlenet_mb64", "googlenet", 64),
             ("resnet50_mb64", "resnet50", 64), ("inception_resnet_v2_mb128",
                                                 "inception_resnet_v2", 128)]
    insts = [(k, mp.profile_to_instance(mp.record(mp.parse_trace(mp.net_trace(net, b))),
                                        alignment=ALIGN).arrays()) for k, net, b in cases]
    for name, n in (("cnn_1e4", 10000), ("uniform_1e4", 10000)):
        fam = name.split("_")[0]
        insts.append((name, gen_trace(fam, n, 0)))
    for key, (a, f, s) in insts:
        solve_bestfit_arrays(a, f, s)  # warm-up (module load, pools)
        wall, (off, pk) = _best_wall(lambda: solve_bestfit_arrays(a, f, s), 5)
        info = plan_info()
        ref_off, ref_pk = oracle.solve_bestfit(a, f, s)
        cw, _ = _best_wall(lambda: oracle.solve_bestfit(a, f, s), 5 if len(a) < 5000 else 1)
        cpu_wall, _ = _best_wall(lambda: solve_bestfit_np(a, f, s), 3 if len(a) < 5000 else 1)
        out[key] = {"blocks": int(len(a)), "peak_bytes": int(pk),
                    "gpu_host_to_host_ms": 1e3 * wall,
                    "gpu_device_ms": float(info["prep_ms"] + info["plan_ms"]),
                    "cpu_port_1core_ms": 1e3 * cpu_wall,
                    "cpu_c_oracle_1core_ms": 1e3 * cw,
                    "speedup_vs_1core": cpu_wall / wall,
                    "bit_exact_vs_oracle": bool(np.array_equal(off, ref_off) and pk == ref_pk)}
    # K3 validator (verify_plan, verifier.py:44-81) at 10^4 / 10^5
    from paper_1804_10001_b200.verifier import verify_arrays
    for n in (10000, 100000):
        a, f, s = gen_trace("uniform", n, 0)
        off, pk = solve_bestfit_arrays(a, f, s)
        verify_arrays(a, f, s, off)
        wall, r = _best_wall(lambda: verify_arrays(a, f, s, off), 3)
        rec = {"blocks": n, "gpu_host_to_host_ms": 1e3 * wall,
               "valid": r["n_violations"] == 0 and r["offsets_ok"] and r["peak_recomputed"] == pk}
        if n <= 10000:
            cw, cr = _best_wall(lambda: oracle.verify(a, f, s, off), 1)
            rec["cpu_c_oracle_1core_ms"] = 1e3 * cw
            rec["agrees_with_oracle"] = (cr["n_violations"] == r["n_violations"] and
                                         cr["peak_recomputed"] == r["peak_recomputed"] and
                                         cr["used"] == r["used"])
        out[f"verify_uniform_{n}"] = rec
    # configs[3]: 4096 LSTM profiles, L=6 (13 blocks) and L=64 (129 blocks)
    import multiprocessing as mpc
    for layers in (6, 64):
        tp, A, F, S = lstm_batch(layers)
        solve_bestfit_batched_arrays(tp, A, F, S)
        wall, (off, pks) = _best_wall(lambda: solve_bestfit_batched_arrays(tp, A, F, S), 5)
        info = plan_info()
        exact = oracle_check(tp, A, F, S, off, pks, range(len(tp) - 1), cpu_procs)
        g = gold.get(f"lstm_L{layers}_a{ALIGN}")
        cols = [(A[tp[t]:tp[t + 1]], F[tp[t]:tp[t + 1]], S[tp[t]:tp[t + 1]])
                for t in range(len(tp) - 1)]
        chunks = [cols[i::cpu_procs] for i in range(cpu_procs)]
        with mpc.get_context("fork").Pool(cpu_procs) as pool:
            pool.map(_lstm_cpu_one, [c[:4] for c in chunks])
            t0 = time.perf_counter()
            pool.map(_lstm_cpu_one, chunks)
            cpu_wall = time.perf_counter() - t0
        out[f"lstm_4096_profiles_L{layers}_b64"] = {
            "blocks": int(len(A)), "traces": 4096, "gpu_host_to_host_ms": 1e3 * wall,
            "gpu_device_ms": float(info["prep_ms"] + info["plan_ms"]),
            "cpu_port_ms": 1e3 * cpu_wall, "cpu_cores": cpu_procs,
            "speedup_vs_cpu": cpu_wall / wall,
            "all_offsets_bit_exact_vs_oracle": bool(exact),
            "matches_reference_digest": (None if g is None else
                                         _sha(off) == g["offsets_sha256"] and
                                         _sha(pks) == g["peaks_sha256"])}
    # configs[4] single traces: uniform / cnn / walk at 10^5, uniform / cnn
    # at 10^6, bit-exact against the reference's own digests
    sweep = [("uniform_1e5_s0", "uniform_rr", 100000), ("cnn_1e5_s0", "cnn", 100000),
             ("walk_1e5_s0", "walk", 100000)]
    if sweep_1e6:
        sweep += [("uniform_1e6_s0", "uniform_rr", 1000000), ("cnn_1e6_s0", "cnn", 1000000),
                  ("walk_1e6_s0", "walk", 1000000)]
    for key, fam, n in sweep:
        a, f, s = gen_trace(fam, n, 0)
        g = gold.get(key)
        solve_bestfit_arrays(a[:1000], f[:1000], s[:1000])
        t0 = time.perf_counter()
        off, pk = solve_bestfit_arrays(a, f, s)
        wall = time.perf_counter() - t0
        info = plan_info()
        rec = {"blocks": n, "gpu_host_to_host_ms": 1e3 * wall,
               "gpu_device_ms": float(info["prep_ms"] + info["plan_ms"]),
               "steps": info["steps"],
               "ns_per_step": 1e6 * float(info["plan_ms"]) / max(1, info["steps"]),
               "peak_bytes": int(pk)}
        if g is not None:
            rec["instance_matches_reference"] = _sha(np.stack([s, a, f], 1)) == g["blocks_sha256"]
            rec["bit_exact_vs_reference"] = (_sha(off) == g["offsets_sha256"] and
                                             pk == g["peak"])
            rec["reference_1core_s_build_container"] = g["ref_s"]
        out[f"single_{key}"] = rec
    return out


def nccl_version():
    import torch
    v = torch.cuda.nccl.version()
    return ".".join(map(str, v)) if isinstance(v, tuple) else str(v)


def bench_config(args, world):
    if args.workload == "lstm":
        return {"workload": f"4096 variable-length LSTM seq2seq profiles (L={args.lstm_layers}, "
                            f"batch 64, BASELINE.json configs[3]) as one batch, sharded over "
                            f"{world} GPU(s) by LPT",
                "global_batch_traces": 4096, "lstm_layers": args.lstm_layers,
                "alignment": ALIGN,
                "parallelism": f"traces sharded over {world} GPU(s), gather to rank 0",
                "l2": "batch is L2-resident (a few MB); each step re-plans it from scratch"}
    return {"workload": f"{args.workload} random-lifetime traces, n={args.n} blocks each, "
                        f"{args.traces} traces per GPU per step (BASELINE.json configs[4])",
            "family": args.workload, "n_blocks_per_trace": args.n,
            "traces_per_gpu": args.traces, "global_batch_traces": args.traces * world,
            "alignment": ALIGN,
            "parallelism": f"traces sharded over {world} GPU(s), gather to rank 0",
            "l2": "inputs larger than L2 per step (no flush needed)"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist
    from paper_1804_10001_b200 import _native as N
    from paper_1804_10001_b200.bestfit import check, plan_info
    from paper_1804_10001_b200 import dist as D

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        backend = os.environ.get("MEMPLAN_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            # NCCL's init lines (rank count, transport) on stderr, for the record
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # stdout: the JSON line
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream
    lib = N.lib()
    procs = min(host_cores(), args.cpu_procs)

    if args.workload == "lstm":
        g_tp, g_A, g_F, g_S = lstm_batch(args.lstm_layers)
        gb = D.Batch(g_tp, g_A, g_F, g_S)
        shards = D.lpt_shards([D.trace_cost(int(n)) for n in gb.sizes()], world)
        my_ids = shards[rank]
        sub = gb.subset(my_ids)
        tp, A, F, S = sub.trace_ptr, sub.alloc, sub.free, sub.size
        total_blocks = len(g_A)
    else:
        tp, A, F, S = make_batch(args.workload, args.n, args.traces, rank, procs)
        my_ids = list(range(rank * args.traces, (rank + 1) * args.traces))
        total_blocks = world * len(A)
    T, NB = len(tp) - 1, len(A)
    d_tp = torch.from_numpy(tp).to(dev)
    d_a, d_f, d_s = (torch.from_numpy(x).to(dev) for x in (A, F, S))
    d_off = torch.empty(max(NB, 1), dtype=torch.int64, device=dev)
    d_pk = torch.empty(max(T, 1), dtype=torch.int64, device=dev)

    def step_device(flags=0):
        rc = lib.mp_plan_bestfit_batched(d_tp.data_ptr(), d_a.data_ptr(), d_f.data_ptr(),
                                         d_s.data_ptr(), T, d_off.data_ptr(), d_pk.data_ptr(),
                                         N.MP_DEVICE_PTRS | flags, local_rank, sh)
        check(rc)

    # diagnostics pass (outside the timed region): steps per trace, sum(W_live)
    step_device(N.MP_STATS)
    info_stats = plan_info()

    # parity: >= 16 traces spread over this rank's batch vs the C oracle
    # (every profile of the LSTM batch)
    torch.cuda.synchronize(dev)
    parity = None
    if args.check:
        off_h = d_off[:NB].cpu().numpy()
        pk_h = d_pk[:T].cpu().numpy()
        sample = range(T) if args.workload == "lstm" else spread(T, args.check_traces)
        parity = oracle_check(tp, A, F, S, off_h, pk_h, sample, procs)

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()

    clocks = Clocks(local_rank)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kern_ms, launches = [], 0
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(args.steps):
        step_device()
        info = plan_info()
        kern_ms.append(info["kernel_ms"])
        launches += int(info["launches"])
        if world > 1:  # the only collective: gather results to rank 0 (NCCL)
            D.gather_device(my_ids, d_off[:NB], d_pk[:T])
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = max_over_ranks(ms)
    value = total_blocks / (ms / 1e3)

    # parity of the GATHERED results (N > 1): rank 0 checks sampled traces of
    # every rank against the C oracle (all profiles of the LSTM batch)
    gathered_parity = None
    if world > 1 and args.check:
        bufs = D.gather_device(my_ids, d_off[:NB], d_pk[:T])
        if rank == 0:
            gathered_parity = check_gathered(args, bufs, world, procs)

    # e2e: public C ABI with pinned host buffers (H2D + D2H inside the region)
    h_tp = torch.from_numpy(tp).pin_memory()
    h_a, h_f, h_s = (torch.from_numpy(x).pin_memory() for x in (A, F, S))
    h_off = torch.empty(max(NB, 1), dtype=torch.int64).pin_memory()
    h_pk = torch.empty(max(T, 1), dtype=torch.int64).pin_memory()
    # short steps (the LSTM batch: ~0.2 ms) take the median over all K steps
    # after one untimed warm-up call; long ones over at most 5
    e2e_steps = max(1, args.steps if ms < 50 else min(args.steps, 5))
    check(lib.mp_plan_bestfit_batched(h_tp.data_ptr(), h_a.data_ptr(), h_f.data_ptr(),
                                      h_s.data_ptr(), T, h_off.data_ptr(), h_pk.data_ptr(),
                                      0, local_rank, sh))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e2e_each = []
    for _ in range(e2e_steps):  # median of per-step times (robust to one slow copy)
        e0.record(stream)
        check(lib.mp_plan_bestfit_batched(h_tp.data_ptr(), h_a.data_ptr(), h_f.data_ptr(),
                                          h_s.data_ptr(), T, h_off.data_ptr(), h_pk.data_ptr(),
                                          0, local_rank, sh))
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_each.append(e0.elapsed_time(e1))
    e2e_sync_ms = max_over_ranks(float(np.median(e2e_each)))
    e2e_exact = bool(np.array_equal(h_off[:NB].numpy(), d_off[:NB].cpu().numpy()) and
                     np.array_equal(h_pk[:T].numpy(), d_pk[:T].cpu().numpy()))

    # e2e through the pipelined C ABI (mp_pipe_*, PlanPipe): K batches from
    # the same pinned host arrays, two in flight, each with its own upload
    # and download inside the timed region (two output buffer sets); the
    # copies of batch k overlap the planning of batches k -/+ 1
    from paper_1804_10001_b200.bestfit import PlanPipe
    pipe_out = [(h_off, h_pk), (torch.empty(max(NB, 1), dtype=torch.int64).pin_memory(),
                                torch.empty(max(T, 1), dtype=torch.int64).pin_memory())]
    np_in = [x.numpy() for x in (h_a, h_f, h_s)]
    with PlanPipe(local_rank) as pipe:
        pipe.wait(pipe.submit(tp, *np_in, offsets_out=pipe_out[1][0].numpy(),
                              peaks_out=pipe_out[1][1].numpy()))  # warm-up (slot buffers)
        pipe.wait(pipe.submit(tp, *np_in, offsets_out=pipe_out[0][0].numpy(),
                              peaks_out=pipe_out[0][1].numpy()))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        pending = []
        for k in range(args.steps):
            if len(pending) == 2:
                pipe.wait(pending.pop(0))
            o, p = pipe_out[k % 2]
            pending.append(pipe.submit(tp, *np_in, offsets_out=o.numpy(), peaks_out=p.numpy()))
        for tk in pending:
            pipe.wait(tk)
        pipe_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    pipe_ms = max_over_ranks(pipe_ms)
    pipe_exact = all(bool(np.array_equal(o[:NB].numpy(), d_off[:NB].cpu().numpy()) and
                          np.array_equal(p[:T].numpy(), d_pk[:T].cpu().numpy()))
                     for o, p in pipe_out)
    e2e_ms = pipe_ms
    e2e_value = total_blocks / (e2e_ms / 1e3)

    # single-trace latency (trace 0 of the batch, device pointers)
    lat_ms, single_info = None, None
    if rank == 0 and args.workload != "lstm":
        n = int(tp[1])
        o1 = torch.empty(n, dtype=torch.int64, device=dev)
        p1 = torch.empty(1, dtype=torch.int64, device=dev)
        for _ in range(2):
            check(lib.mp_plan_bestfit(d_a.data_ptr(), d_f.data_ptr(), d_s.data_ptr(), n,
                                      o1.data_ptr(), p1.data_ptr(), N.MP_DEVICE_PTRS,
                                      local_rank, sh))
        torch.cuda.synchronize(dev)
        e0.record(stream)
        check(lib.mp_plan_bestfit(d_a.data_ptr(), d_f.data_ptr(), d_s.data_ptr(), n,
                                  o1.data_ptr(), p1.data_ptr(), N.MP_DEVICE_PTRS, local_rank, sh))
        e1.record(stream)
        torch.cuda.synchronize(dev)
        lat_ms = e0.elapsed_time(e1)
        single_info = plan_info()

    if rank == 0:
        kms = float(np.median(kern_ms))
        roof = roofline(args, T, NB, info_stats, kms, lat_ms, single_info)
        cpu = None
        if world == 1 and not args.no_cpu:
            groups, blocks = cpu_groups(args, procs, 0)
            wall, per = cpu_sample("port", groups)
            cpu = {"value": blocks / wall, "unit": UNIT, "cores": procs, "kind": "port",
                   "cpu": cpu_model(),
                   "sample": (f"{blocks} blocks: " +
                              ("the 4096 LSTM profiles split over the cores"
                               if args.workload == "lstm" else
                               f"{procs} {args.workload} traces x {args.n} blocks, one per "
                               f"process ({per:.1f} s/trace)") +
                              "; oracle/bestfit_np.py, the numpy restatement of "
                              "memplan.bestfit (the reference itself: --impl reference)")}
        suite = None
        if world == 1 and not args.no_suite:
            try:
                suite = config_suite(procs, not args.no_1e6)
            except Exception as exc:  # noqa: BLE001  (reported, not fatal)
                suite = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        replay = None
        if world == 1 and not args.no_replay:
            replay = replay_numbers()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True,
            "scaling": "strong" if args.workload == "lstm" else "weak", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic", "config": bench_config(args, world),
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": int(8 * (3 * NB + T + 1)),
                    "d2h_bytes_per_step": int(8 * (NB + T)),
                    "api": "mp_pipe_submit / mp_pipe_wait (PlanPipe), pinned host arrays, "
                           "K batches two in flight, host wall clock over all K",
                    "results_equal_device_path": pipe_exact,
                    "sync_call": {"value": total_blocks / (e2e_sync_ms / 1e3),
                                  "api": "mp_plan_bestfit_batched, median per call",
                                  "results_equal_device_path": e2e_exact}},
            "gpu_launches": launches,
            "collective": ({"backend": dist.get_backend(), "nranks": dist.get_world_size(),
                            "nccl_version": nccl_version() if dist.get_backend() == "nccl"
                            else None,
                            "op": "grouped send/recv gather of offsets and peaks to rank 0 "
                                  "(paper_1804_10001_b200.dist.gather_device)"}
                           if world > 1 else None),
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clk,
            "single_trace": ({"n": int(tp[1]), "latency_ms": lat_ms,
                              "blocks_per_s": int(tp[1]) / (lat_ms / 1e3),
                              "steps": single_info["steps"]} if lat_ms else None),
            "plan_info": {k: info_stats[k] for k in ("steps", "lifts", "max_lines", "engine",
                                                     "sum_wlive")},
            "parity_vs_oracle": {"traces_checked": (T if args.workload == "lstm"
                                                    else len(spread(T, args.check_traces))),
                                 "bit_exact": parity, "gathered_bit_exact": gathered_parity},
            "replay": replay,
            "configs": suite,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def check_gathered(args, bufs, world: int, procs: int) -> bool:
    """Rank 0: the gathered payloads [ids | peaks | offsets] of every rank
    against the C oracle (sampled traces per rank; all LSTM profiles)."""
    if args.workload == "lstm":
        g_tp, g_A, g_F, g_S = lstm_batch(args.lstm_layers)
        from paper_1804_10001_b200 import dist as D
        shards = D.lpt_shards([D.trace_cost(int(n)) for n in np.diff(g_tp)], world)
        off = np.zeros(len(g_A), np.int64)
        pks = np.zeros(len(g_tp) - 1, np.int64)
        seen = 0
        for r, b in enumerate(bufs):
            v = b.cpu().numpy()
            nt = len(shards[r])
            ids, pk, offs = v[:nt], v[nt:2 * nt], v[2 * nt:]
            if not np.array_equal(ids, shards[r]):
                return False
            pos = 0
            for i, t in enumerate(ids):
                a, b2 = int(g_tp[t]), int(g_tp[t + 1])
                off[a:b2] = offs[pos:pos + b2 - a]
                pks[t] = pk[i]
                pos += b2 - a
            seen += nt
        return seen == len(pks) and oracle_check(g_tp, g_A, g_F, g_S, off, pks,
                                                 range(len(pks)), procs)
    ok = True
    per = max(2, args.check_traces // world)
    for r, b in enumerate(bufs):
        v = b.cpu().numpy()
        T = args.traces
        ids, pk, offs = v[:T], v[T:2 * T], v[2 * T:]
        if not np.array_equal(ids, np.arange(r * T, (r + 1) * T)):
            return False
        sample = spread(T, per)
        cols = [gen_trace(args.workload, args.n, trace_seed(r, t)) for t in sample]
        tp, A, F, S = csr(cols)
        # rank r's traces are all n blocks: trace t starts at t * n
        got = np.concatenate([offs[t * args.n:(t + 1) * args.n] for t in sample])
        ok = ok and oracle_check(tp, A, F, S, got, pk[sample], range(len(sample)), procs)
    return bool(ok)


def roofline(args, T: int, NB: int, info_stats: dict, kms: float, lat_ms, single_info) -> dict:
    """Latency roofline (SURVEY §8(d) "step-latency floor"): the planner is
    a dependent chain of S ~ 3n steps per trace, each needing at least one
    shared-memory argmin, one dependent table read and one line update.
    `peak` = the step rate of that minimal chain (tools/ubench/step_floor.cu,
    measured now, same GPU) at the batch's residency; `achieved` = the
    planner's trace-steps per second.  DRAM traffic (ncu) and the survey's
    algorithmic bytes are reported beside it."""
    steps_total = float(info_stats["steps"])
    achieved = steps_total / (kms / 1e3)
    resident = max(1, min(16, -(-T // N_SMS)))
    # the window table is in shared memory for TIER_TINY / TIER_SCAN / TIER_ALL
    # (engine bits 512 / 128 / 2): the floor's table read is an LDS there
    eng = int(info_stats.get("engine", 0))
    smem_table = bool(eng & (512 | 128 | 2))
    fl_batch = step_floor(1 if smem_table else 0, N_SMS * resident)
    fl_one = step_floor(0, 1)
    fl_one_smem = step_floor(1, 1)
    peak = fl_batch["steps_per_s"] if fl_batch else None
    hbm_peak, peak_kind = measured_peak()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            rec = json.load(fh).get(f"{args.workload} n={args.n} traces={args.traces}")
        traffic = int(rec["dram_bytes"]) if rec else None
    except (OSError, ValueError, KeyError, TypeError):
        traffic = None
    b_alg = 24 * info_stats["sum_wlive"] + 32 * NB
    out = {
        "bound": "latency", "unit": "trace-steps/s", "achieved": achieved, "peak": peak,
        "frac": (achieved / peak) if peak else None, "traffic": traffic,
        "kernel": ("k_plan_occ (K2 batched planner)" if resident > 1 else
                   "planner (K1/K2, engine %d)" % eng), "kernel_ms": kms,
        "steps_per_launch": steps_total, "steps_per_trace": steps_total / max(T, 1),
        "traces_resident_per_sm": resident,
        "peak_def": (f"measured step rate of the minimal dependent step (LDS argmin + REDUX + "
                     f"VOTE/SHFL, one dependent {'shared-memory' if smem_table else 'L2'} "
                     f"table read + REDUX, STS update) with "
                     f"{resident} one-warp traces per SM on {N_SMS} SMs "
                     f"(tools/ubench/step_floor.cu)"),
        "floor_batch": fl_batch,
        "floor_single_l2": fl_one, "floor_single_smem": fl_one_smem,
        "hbm": {"peak_gbs": hbm_peak, "peak_source": peak_kind,
                "achieved_gbs": (traffic / (kms / 1e3) / 1e9) if traffic else None,
                "frac": (traffic / (kms / 1e3) / 1e9 / hbm_peak) if traffic else None,
                "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram bytes)"},
        "alg_bytes_per_launch": b_alg if info_stats.get("sum_wlive") else None,
    }
    if lat_ms and single_info and fl_one:
        s = float(single_info["steps"])
        floor_ms = s * fl_one["cycles_per_step"] / 1.965e9 * 1e3
        out["single_trace"] = {"steps": s, "latency_ms": lat_ms,
                               "floor_ms": floor_ms, "frac": floor_ms / lat_ms,
                               "floor_def": "S x t_step,min (one warp, L2 table read per step, "
                                            "at 1965 MHz)"}
    return out


def replay_numbers():
    try:
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "replay_bench.py"),
                            "--alloc", "all", "--reps", "10"], capture_output=True,
                           text=True, timeout=900)
        rl = [x for x in r.stdout.splitlines() if x.startswith("{")]
        rr = json.loads(rl[-1]) if rl else {}
        g = lambda a, k: rr.get(a, {}).get(k)  # noqa: E731
        return {"unit": "ns/alloc",
                "trace": "cnn-like L=5000 (10^4 allocs/epoch), best of 10 epochs",
                "memplan_c_abi_arena": g("carena", "ns_per_alloc"),
                "memplan_torch_hooks": g("memplan", "hook_ns_per_alloc"),
                "memplan_via_torch_pluggable": g("memplan", "ns_per_alloc"),
                "torch_pluggable_floor": g("floor", "ns_per_alloc"),
                "torch_caching_allocator": g("caching", "ns_per_alloc"),
                "torch_cudaMallocAsync": g("async", "ns_per_alloc"),
                "torch_empty": {a: g(a, "torch_empty_ns_per_alloc")
                                for a in ("memplan", "floor", "caching", "async")},
                "addresses_match_plan": g("memplan", "addresses_match_plan"),
                "plan_peak_bytes": g("memplan", "plan_peak_bytes"),
                "pool_peak_bytes": g("memplan", "pool_peak_bytes")}
    except (OSError, ValueError, subprocess.SubprocessError) as exc:
        return {"error": str(exc)[:200]}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", choices=["uniform", "cnn", "walk", "lstm"], default="uniform")
    p.add_argument("--lstm-layers", type=int, default=6)
    p.add_argument("--blocks", dest="n", type=int, default=100_000,
                   help="blocks per trace (not --n: torchrun would take it as its own flag)")
    p.add_argument("--traces", type=int, default=None,
                   help="traces per GPU (default 2368: 16 per SM)")
    p.add_argument("--cpu-procs", type=int, default=32)
    p.add_argument("--check-traces", type=int, default=16)
    p.add_argument("--ref-budget", type=float, default=150.0,
                   help="reference arm: stop measured steps after this many seconds")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-replay", action="store_true")
    p.add_argument("--no-suite", action="store_true")
    p.add_argument("--no-1e6", action="store_true")
    p.add_argument("--check", action="store_true", default=True)
    p.add_argument("--no-check", dest="check", action="store_false")
    args = p.parse_args()
    if args.traces is None:
        # 16 one-warp traces per SM for every family (cnn / walk: 592 -> 2368
        # traces raised 196 -> 553 / 116 -> 348 M blocks/s; 4736 adds nothing)
        args.traces = 2368
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    # test hook: run every rank on one device (functional check of the N > 1
    # path on a single GPU, with MEMPLAN_BENCH_BACKEND=gloo)
    if os.environ.get("MEMPLAN_BENCH_DEVICE") is not None:
        local_rank = int(os.environ["MEMPLAN_BENCH_DEVICE"])
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
