#!/usr/bin/env python
"""Benchmark: signals/s of zero-tree OMP (headline) and full OMP on B200.

Workload: BASELINE.json configs[4] ("large": N=4096 fine / 512 coarse,
T_high=16384, T_low=2048, Q=8, K=64, 1,000,000 signals, sigma=0.01, fp32
inputs, stop at K or |r| <= 1e-3 |y|) -- the config the 1/2/4/8-GPU sweep
is quoted on; its 16.4 GB of signals fit one B200.  Synthetic and seeded:
the signals are drawn on the device (paper_1511_05174_b200.workloads.
signals_device, the BASELINE generator in 65,536-signal blocks), so every
rank generates just its own shard.

A step = one pass of the hot path over all 1,000,000 signals.  With N GPUs
the signals are partitioned into N contiguous shards (strong scaling; the
dictionary is replicated; no collective on the data path).  `value` times the
step through the C ABI with inputs resident in HBM (CUDA events on the
launching stream, L2 flushed between steps, max over ranks); `e2e` times the
same C-ABI call with pinned HOST buffers (H2D of the signals and D2H of every
output inside the timed region) plus, for N > 1, the NCCL gather of all
outputs to rank 0; `e2e_api` times the Python drop-in
(crossscale.zero_tree_many_arrays) on a pageable N x P fp64 column batch.
`--impl reference` times the reference itself (crossdict's numba kernel from
baseline/_ref, forked processes on all host cores) on a bounded sample.

Run:  python bench.py [--gpus N --steps K --warmup W]
      (N > 1 without torchrun: the script launches torchrun itself)
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_1511_05174_b200 import workloads as W  # noqa: E402

METRIC = "signals/sec for zero-tree OMP and full OMP at 1/2/4/8 B200; % of roofline"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
REF_PATH = os.path.join(REPO, "baseline", "_ref")


def load_traffic():
    """ncu DRAM traffic of each profiled kernel: round 2 (profiles/r2_ncu_traffic.json,
    configs[4] captures) as bytes per unit (signal) of a captured launch; round-1
    entries (bytes per configs[1] launch) only for kernels round 2 did not capture."""
    out = {}
    for name in ("r1_ncu_traffic.json", "r2_ncu_traffic.json"):
        try:
            with open(os.path.join(REPO, "profiles", name)) as f:
                out.update({k: v for k, v in json.load(f).items() if not k.startswith("_")})
        except (OSError, ValueError):
            pass
    return out


def traffic_per_launch(entry, units_per_launch):
    """DRAM bytes of one launch: a round-2 per-unit figure times the units the
    launch processes, or a round-1 per-launch figure as is."""
    if isinstance(entry, dict):
        return entry["bytes_per_unit"] * units_per_launch
    return entry


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return dict(PEAKS_FALLBACK), "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and throttle reasons sampled during a region: NVML polled
    every 5 ms from a thread (the data nvidia-smi reports), or nvidia-smi
    -lms 100 when pynvml is unavailable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []  # (sm_mhz, max_mhz, set(reasons))
        self.proc = None
        self.thread = None
        self.stop_flag = threading.Event()
        self.source = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = self.gpu
            if vis and vis.split(",")[self.gpu].strip().isdigit():
                idx = int(vis.split(",")[self.gpu])
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.source = "nvml"
            self.thread = threading.Thread(target=self._poll_nvml, args=(pynvml, h), daemon=True)
            self.thread.start()
            return
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        self.source = "nvidia-smi"
        self.thread = threading.Thread(target=self._read_smi, daemon=True)
        self.thread.start()

    def _poll_nvml(self, nv, h):
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                "sw_power_cap": 0x4}
        smax = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        while not self.stop_flag.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, smax, {k for k, b in bits.items() if r & b}))
            except Exception:
                pass
            time.sleep(0.005)

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                rs = {nm for i, nm in enumerate(self.NAMES) if parts[2 + i].lower().startswith("active")}
                self.samples.append((float(parts[0]), float(parts[1]), rs))
            except ValueError:
                continue

    def stop(self):
        self.stop_flag.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [x[0] for x in self.samples]
        reasons = set().union(*[x[2] for x in self.samples]) if self.samples else set()
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": self.samples[-1][1] if self.samples else None,
                "reasons": sorted(reasons), "samples": len(sm), "source": self.source}


# ------------------------------------------------------------------ helpers
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def flops_ls(n, counts):
    """MGS/Cholesky least-squares flops of the reference cost model,
    4N k(k-1) + 11 N k per signal, summed over signals."""
    k = counts.astype(np.float64)
    return float(np.sum(4.0 * n * k * (k - 1.0) + 11.0 * n * k))


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def model_arrays(ci):
    """(low_t, high_t, k1, fine_shape, factors, phi) of a config's zero-tree model."""
    w = W.CONFIGS[ci]
    d = W.dictionaries(ci)
    if w.measurements:
        return d.e_low_t, d.e_high_t, min(w.k, w.n_signal, w.t_low), None, None, True
    return d.low_t, d.high_t, w.k, w.fine_shape, w.factors, False


# ---- the reference itself: crossdict (baseline/_ref) in forked processes
_REF = {}


def reference_available():
    """crossdict importable from baseline/_ref (its numba kernel needs numba)."""
    if "mod" in _REF:
        return _REF["mod"] is not None
    try:
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/cdb_numba_cache")
        if os.path.isdir(REF_PATH) and REF_PATH not in sys.path:
            sys.path.insert(0, REF_PATH)
        import crossdict.crossscale as cs
        import crossdict.pursuit as cp
        import crossdict.scaling as sc
        import crossdict.tensor as ct
        _REF["mod"] = (cs, cp, sc, ct)
    except Exception as e:  # noqa: BLE001 -- reported in the JSON line
        _REF["mod"] = None
        _REF["why"] = f"{type(e).__name__}: {e}"
    return _REF["mod"] is not None


def _ref_model(ci):
    cs, cp, sc, ct = _REF["mod"]
    w = W.CONFIGS[ci]
    d = W.dictionaries(ci)
    cp.REL_RESIDUAL_TOL = W.REL_TOL  # BASELINE stopping rule
    if w.measurements:  # cfg 3: batched OMP on the effective dictionaries
        return ("phi", np.ascontiguousarray(d.e_low_t.T), np.ascontiguousarray(d.e_high_t.T),
                min(w.k, w.n_signal, w.t_low), w.k, w.q)
    return ("zt", cs.CrossScaleModel(ct.Dictionary(np.ascontiguousarray(d.low_t.T)),
                                     ct.Dictionary(np.ascontiguousarray(d.high_t.T)),
                                     sc.ScaleSpec(w.fine_shape, w.factors), w.k, w.k))


def _ref_solve(model, cols):
    """crossdict's zero-tree solve of the N x P column batch (its public API)."""
    cs, cp, _, _ = _REF["mod"]
    if model[0] == "zt":
        return cs.zero_tree_many_arrays(model[1], cols)
    _, e_low, e_high, k1, k2, q = model
    low = cp.omp_many_arrays(e_low, cols, cp.PursuitConfig(k1))
    blocks = np.sort(low.sel, axis=1)
    return low, cp.omp_many_arrays(e_high, cols, cp.PursuitConfig(k2), allowed_blocks=blocks,
                                   block_q=q), {}


_FORK = {}


def _ref_worker(bounds):
    from threadpoolctl import threadpool_limits
    lo, hi = bounds
    with threadpool_limits(1):
        t0 = time.perf_counter()
        _ref_solve(_FORK["model"], _FORK["cols"][:, lo:hi])
        return time.perf_counter() - t0


def reference_rate(ci, cols, procs):
    """crossdict on `procs` forked processes, signals split contiguously;
    returns (signals/s, seconds) with the time = max over processes of the
    solver-call wall time."""
    import multiprocessing as mp
    p = cols.shape[1]
    procs = max(1, min(procs, p))
    _FORK["cols"] = cols
    if "model" not in _FORK or _FORK.get("ci") != ci:
        _FORK["model"] = _ref_model(ci)
        _FORK["ci"] = ci
    cuts = np.linspace(0, p, procs + 1).astype(int)
    bounds = [(int(cuts[i]), int(cuts[i + 1])) for i in range(procs)]
    if procs == 1:
        dt = _ref_worker(bounds[0])
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            dt = max(pool.map(_ref_worker, bounds))
    return p / dt, dt


def reference_warm(ci, cols):
    """JIT-compile crossdict's kernel in this process (forked children inherit it)."""
    _FORK["model"] = _ref_model(ci)
    _FORK["ci"] = ci
    _ref_solve(_FORK["model"], cols[:, :1])


def reference_cpu_baseline(ci, cols, threads, budget_s):
    """Single-core rate, then a multi-process sample of about budget_s."""
    reference_warm(ci, cols)
    r1, _ = reference_rate(ci, cols[:, : min(2, cols.shape[1])], 1)
    per_proc = int(max(1, min(cols.shape[1] // threads, round(r1 * budget_s))))
    m = min(cols.shape[1], per_proc * threads)
    rate, dt = reference_rate(ci, cols[:, :m], threads)
    return {"value": rate, "unit": "signals/s", "cores": threads, "kind": "reference",
            "single_core_value": r1,
            "sample": f"{m} signals of configs[{ci}] zero-tree OMP in {dt:.1f} s: crossdict "
                      f"(baseline/_ref, numba omp_batch_kernel) zero_tree_many_arrays on "
                      f"{threads} forked processes, time = max over processes; single-core "
                      f"rate from 2 signals on one process"}


# ---- the C restatement of the reference kernel (oracle/), secondary figure
def run_oracle_zero_tree(ci, ys_rows, threads):
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as O
    low_t, high_t, k1, fs, fa, phi = model_arrays(ci)
    w = W.CONFIGS[ci]
    if phi:
        return O.zero_tree_phi_many(low_t, high_t, k1, w.k, ys_rows, rel_tol=W.REL_TOL,
                                    nthreads=threads)
    return O.zero_tree_many_arrays(low_t, high_t, fs, fa, w.k, w.k, ys_rows, rel_tol=W.REL_TOL,
                                   nthreads=threads)


def port_rate(ci, ys_rows, threads, budget_s):
    """oracle/omp_oracle.c on `threads` host threads over a bounded sample."""
    probe = ys_rows[: min(len(ys_rows), max(threads, 16))]
    t0 = time.perf_counter()
    run_oracle_zero_tree(ci, probe, threads)
    rate = len(probe) / max(time.perf_counter() - t0, 1e-6)
    m = int(min(len(ys_rows), max(len(probe), rate * budget_s)))
    t0 = time.perf_counter()
    run_oracle_zero_tree(ci, ys_rows[:m], threads)
    dt = time.perf_counter() - t0
    return {"value": m / dt, "unit": "signals/s", "cores": threads, "kind": "port",
            "sample": f"{m} signals in {dt:.1f} s (oracle/omp_oracle.c restating crossdict's "
                      f"kernel, {threads} threads)"}


def cpu_baseline(ci, ys_host):
    """The reference (crossdict, forked processes) on the benchmark's own
    signals, with the C port as a secondary figure; the port alone when
    crossdict cannot be imported."""
    threads = cpu_threads()
    if reference_available():
        cpu = reference_cpu_baseline(ci, np.ascontiguousarray(ys_host.T), threads, 15.0)
        cpu["port"] = port_rate(ci, ys_host, threads, 10.0)
    else:
        cpu = port_rate(ci, ys_host, threads, 15.0)
        cpu["note"] = f"crossdict unavailable: {_REF.get('why')}"
    return cpu


def cpu_baseline_subprocess(ci, ys_host):
    """Run cpu_baseline in a fresh interpreter (its worker processes fork from
    a parent without CUDA or torch threads)."""
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "ys.npy")
        np.save(path, ys_host)
        out = subprocess.run([sys.executable, os.path.abspath(__file__), "--config", str(ci),
                              "--cpu-sample", path], capture_output=True, text=True)
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    if out.returncode != 0 or not lines:
        return {"error": (out.stderr or out.stdout)[-500:]}
    return json.loads(lines[-1])


# ------------------------------------------------------------------ reference arm
def workload_config(ci, total, world):
    """The `config` object of both arms' lines: the same workload, named once."""
    w = W.CONFIGS[ci]
    per = -(-total // world)
    return {"workload": f"{w.name} (BASELINE configs[{ci}]) zero-tree OMP: "
                        f"N={w.n_high}, N_low={w.n_low}, T_high={w.t_high}, "
                        f"T_low={w.t_low}, Q={w.q}, K={w.k}, {total:,} signals "
                        f"split over {world} GPU(s), stop K or |r|<=1e-3|y|",
            "signals": total, "signals_per_gpu": per,
            "parallelism": f"signal shards x{world}, dictionary replicated",
            "l2": f"flushed between steps (256 MiB write); inputs {total * w.n_high * 4 / 1e9:.1f} GB"
                  " > L2" if total * w.n_high * 4 > (126 << 20) else
                  "flushed between steps (256 MiB write)"}


def bench_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    ci = args.config
    w = W.CONFIGS[ci]
    threads = cpu_threads()
    budget = min(8.0, 150.0 / max(1, args.steps + args.warmup))
    use_ref = reference_available()
    # a pool of seeded signals of the workload (host stream, same distribution
    # as the GPU arm's device stream)
    pool_n = min(w.signals, max(4 * threads, 64))
    ys = W.signals(ci, 0, pool_n)
    cols = np.ascontiguousarray(ys.T)
    if use_ref:
        reference_warm(ci, cols)
        r1, _ = reference_rate(ci, cols[:, :2], 1)
        per_proc = max(1, int(round(r1 * budget)))
        sample = per_proc * threads
        if sample > pool_n:
            ys = W.signals(ci, 0, sample)
            cols = np.ascontiguousarray(ys.T)
        for _ in range(args.warmup):  # untimed: one signal per process
            reference_rate(ci, cols[:, :threads], threads)
        times = [reference_rate(ci, cols[:, :sample], threads)[1] for _ in range(args.steps)]
        kind = "reference"
        desc = (f"{sample} signals of configs[{ci}] per step: crossdict (baseline/_ref) "
                f"zero_tree_many_arrays, numba kernel, {threads} forked processes, time = max "
                f"over processes; single-core {r1:.2f} signals/s")
    else:
        t0 = time.perf_counter()
        run_oracle_zero_tree(ci, ys[:threads], threads)
        rate = threads / max(time.perf_counter() - t0, 1e-6)
        sample = int(min(len(ys), max(threads, rate * budget)))
        for _ in range(args.warmup):
            run_oracle_zero_tree(ci, ys[:threads], threads)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            run_oracle_zero_tree(ci, ys[:sample], threads)
            times.append(time.perf_counter() - t0)
        kind = "port"
        desc = (f"{sample} signals of configs[{ci}] per step (oracle/omp_oracle.c, {threads} "
                f"threads; crossdict unavailable: {_REF.get('why')})")
    value = sample * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "signals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator, fp32-exact inputs)",
        # the workload of our arm's line; each reference step codes a bounded
        # sample of it (cpu_baseline.sample)
        "config": workload_config(ci, args.num_signals or w.signals, world),
        "signals_per_step": sample,
        "cpu_baseline": {"value": value, "unit": "signals/s", "cores": threads, "kind": kind,
                         "sample": desc},
        "e2e": {"value": value, "unit": "signals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def _outs(torch, p, k, dev="cuda", pin=False):
    mk = (lambda shape, dt: torch.empty(shape, dtype=dt, device=dev, pin_memory=pin))
    return dict(sel=mk((p, k), torch.int64), alpha=mk((p, k), torch.float64),
                counts=mk((p,), torch.int64), rnorm=mk((p,), torch.float64),
                scans=mk((p,), torch.int64), flag=mk((p,), torch.uint8))


def _nbytes(o):
    return sum(v.numel() * v.element_size() for v in o.values())


def bench_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1511_05174_b200 import _native as N
    from paper_1511_05174_b200 import device as D
    from paper_1511_05174_b200 import sharding as SH

    rank, world, local = dist_env()
    # CDB_BENCH_SMOKE=1: launcher smoke test on a box with fewer GPUs than ranks
    # (ranks share devices round-robin, gloo process group; timings meaningless)
    smoke = os.environ.get("CDB_BENCH_SMOKE") == "1"
    if smoke:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if smoke:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ci = args.config
    w = W.CONFIGS[ci]
    total = args.num_signals or w.signals
    s0, s1 = SH.shard_range(total, rank, world)
    P = s1 - s0
    low_t, high_t, k1, fs, fa, phi = model_arrays(ci)

    t_gen = time.perf_counter()
    yd = W.signals_device(ci, s0, s1)  # fp32 rows in HBM
    eps_full = (W.REL_TOL * torch.linalg.vector_norm(yd.double(), dim=1)).contiguous()
    lo = D.device_dictionary(low_t)
    hi = D.device_dictionary(high_t)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen

    olo, ohi, ofull = _outs(torch, P, k1), _outs(torch, P, w.k), _outs(torch, P, w.k)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    stream = torch.cuda.current_stream()

    def zt_step():
        D.zero_tree_raw(lo, hi, fs, fa, yd, P, k1, w.k, W.REL_TOL, phi, "auto", olo, ohi)

    def full_step():
        D.omp_batch_raw(hi, yd, P, w.k, eps_full, None, "auto", ofull)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(step, k_steps):
        total_ms = 0.0
        for _ in range(k_steps):
            flush.zero_()
            torch.cuda.synchronize()
            barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b.record(stream)
            torch.cuda.synchronize()
            total_ms += a.elapsed_time(b)
        return max_over_ranks(total_ms)

    for _ in range(args.warmup):
        zt_step()
    # full OMP warm-up on a slice (allocations, one-time attributes)
    wm = min(P, 16384)
    D.omp_batch_raw(hi, yd[:wm], wm, w.k, eps_full[:wm], None, "auto",
                    {k: v[:wm] for k, v in ofull.items()})
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    launches0 = N.launch_count()
    N.profile_enable(True)
    zt_ms = timed(zt_step, args.steps)
    prof_zt = N.profile_read()
    N.profile_enable(True)
    full_ms = timed(full_step, args.full_steps)
    prof_full = N.profile_read()
    N.profile_enable(False)
    launches = N.launch_count() - launches0
    clk = clocks.stop()
    engine_full = N.last_run_info()
    zt_value = total * args.steps / (zt_ms * 1e-3)
    full_value = total * args.full_steps / (full_ms * 1e-3)

    # ---- e2e through the C ABI: pinned host signals in, host outputs out,
    # plus the NCCL gather of every output to rank 0 when N > 1
    yh = torch.empty((P, w.n_signal), dtype=torch.float32, pin_memory=True)
    yh.copy_(yd)
    hlo, hhi = _outs(torch, P, k1, "cpu", True), _outs(torch, P, w.k, "cpu", True)

    def npv(o):
        return {k: v.numpy() for k, v in o.items()}

    hlo_n, hhi_n, yh_n = npv(hlo), npv(hhi), yh.numpy()

    gdev = None if smoke else "cuda"  # NCCL gathers device tensors; gloo host ones

    def e2e_step():
        D.zero_tree_raw(lo, hi, fs, fa, yh_n, P, k1, w.k, W.REL_TOL, phi, "auto", hlo_n, hhi_n)
        if world > 1:
            SH.gather_solutions(hlo_n, total, device=gdev)
            SH.gather_solutions(hhi_n, total, device=gdev)

    e2e_step()  # warm (pinned staging, pipeline buffers)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    e2e_total = 0.0
    for _ in range(e2e_steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        e2e_step()
        e2e_total += time.perf_counter() - t0
    e2e_total = max_over_ranks(e2e_total)
    h2d = total * w.n_signal * 4
    d2h = (_nbytes(hlo) + _nbytes(hhi)) * world
    del yh

    # ---- e2e through the Python drop-in on the reference's layout (rank 0, N = 1)
    e2e_api = e2e_api_full = None
    if rank == 0 and world == 1 and not args.no_api:
        e2e_api = bench_dropin(torch, ci, yd, args.api_signals)
        e2e_api_full = bench_dropin_full(torch, ci, yd, args.api_full_signals)

    # ---- roofline of the dominant kernel and of the whole step
    peaks, peaks_kind = load_peaks()
    traffic_tab = load_traffic()
    n_low = w.n_signal if phi else w.n_low
    c_low = olo["counts"].cpu().numpy()
    c_high = ohi["counts"].cpu().numpy()
    low_scans = olo["scans"].double().sum().item()
    high_scans = ohi["scans"].double().sum().item()
    f_step1 = 2.0 * n_low * low_scans + flops_ls(n_low, c_low)
    f_step2 = 2.0 * w.n_signal * high_scans + flops_ls(w.n_signal, c_high)
    p_emu = peaks["bf16_tflops"] / 6.0
    dom_name, (dom_total, dom_launches) = max(prof_zt.items(), key=lambda kv: kv[1][0])
    dom_ms = dom_total / max(dom_launches, 1)
    # algorithmic flops of one launch of the dominant kernel (SURVEY §8(d) cost
    # model on this rank's actual scan counts)
    step_kernels = {"gram_step2": f_step2, "resident_step2": f_step2, "exact_step2": f_step2,
                    "gram_step1": f_step1, "resident_step1": f_step1, "exact_step1": f_step1,
                    "corr_topk": 2.0 * n_low * low_scans}
    dom_flops = step_kernels.get(dom_name, 0.0) * args.steps / max(dom_launches, 1)
    achieved = dom_flops / (dom_ms * 1e-3) / 1e12 if dom_ms > 0 else 0.0
    step_tf = (f_step1 + f_step2) * world / (zt_ms / args.steps * 1e-3) / 1e12
    roofline = {
        "bound": "tensor", "kernel": dom_name, "achieved": achieved, "peak": p_emu,
        "unit": "TFLOP/s", "frac": achieved / p_emu,
        "traffic": (traffic_per_launch(traffic_tab[dom_name], P * args.steps / max(dom_launches, 1))
                    if dom_name in traffic_tab else None),
        "launch_ms": dom_ms, "share_of_step": dom_total / max(sum(v[0] for v in prof_zt.values()),
                                                              1e-9),
        "step": {"achieved": step_tf, "frac": step_tf / p_emu,
                 "flops_per_signal": (f_step1 + f_step2) / P},
        "basis": "SURVEY §8.0/§8(d) algorithmic flops 2*N*scans + 4Nk(k-1) + 11Nk per signal of "
                 "the kernel's step (actual scan counts) / its mean launch time; peak = "
                 f"{peaks_kind} bf16 {peaks['bf16_tflops']} TF/s / 6 (P_emu, 3xTF32-emulated "
                 "fp32); the Gram formulation of step 2 does ~1/128 of the scan flops, so frac "
                 "can exceed 1; traffic = ncu DRAM bytes per launch (profiles/r2_ncu_traffic.json: "
                 "bytes per signal of a 65,536-signal capture x the signals of this launch)"}
    corr = prof_full.get("corr_topk")
    full_roof = None
    if corr:
        full_scans = ofull["scans"].double().sum().item()
        c_ms = corr[0] / max(corr[1], 1)
        c_flops = 2.0 * w.n_signal * full_scans * args.full_steps / max(corr[1], 1)
        full_roof = {"bound": "tensor", "kernel": "corr_topk",
                     "achieved": c_flops / (c_ms * 1e-3) / 1e12, "peak": peaks["bf16_tflops"],
                     "unit": "TFLOP/s",
                     "frac": c_flops / (c_ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
                     "traffic": (traffic_per_launch(traffic_tab["corr_topk_full"],
                                                    P * args.full_steps * w.k / max(corr[1], 1))
                                 if "corr_topk_full" in traffic_tab else None), "launch_ms": c_ms,
                     "basis": "2*N*scans of the full-OMP batch (actual scan counts) / corr_topk "
                              "time, against the measured bf16 peak it runs on (burst figure; "
                              "frac_sustained: against the sustained one, the kernel being timed "
                              "inside a long power-capped pass)"}
        sus = peaks.get("bf16_tflops_sustained")
        if sus:
            full_roof["peak_sustained"] = sus
            full_roof["frac_sustained"] = full_roof["achieved"] / sus

    # ---- the HBM-bound stage of the step (block-mean downsample, scaling.py:99-116)
    hbm_stages = None
    ds = prof_zt.get("downsample")
    if ds and not phi and ds[0] > 0:
        ds_ms = ds[0] / max(ds[1], 1)
        ds_bytes = (P * args.steps / max(ds[1], 1)) * (4.0 * w.n_high + 8.0 * w.n_low + 16.0)
        hbm_stages = {"downsample": {
            "ms": ds_ms, "achieved": ds_bytes / (ds_ms * 1e-3) / 1e9, "peak": peaks["hbm_gbs"],
            "unit": "GB/s", "frac": ds_bytes / (ds_ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
            "basis": "per signal: N fp32 in + N_low fp64 out + two fp64 tolerances; "
                     "extract_patches / reconstruct_aggregate are in pipeline_ends.roofline"}}

    def resid_stage(prof, counts, n_row, y_bytes, steps):
        """The scan-operand gather r~ = y - D32_S x (_kernels.py:132-137): per
        signal-iteration at support size k, k fp32 atom rows + y in + fp16 operand out."""
        rs = prof.get("ls_resid")
        if not rs or rs[0] <= 0:
            return None
        c = counts.astype(np.float64)
        rows = float((c * (c - 1) / 2).sum())
        iters = float(np.maximum(c - 1, 0).sum())
        b = (rows * n_row * 4.0 + iters * n_row * (y_bytes + 2.0)) * steps
        gbs = b / (rs[0] * 1e-3) / 1e9
        return {"ms_per_step": rs[0] / steps, "achieved": gbs, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"],
                "basis": "algorithmic bytes (k fp32 atom rows per signal-iteration + y in + fp16 "
                         "operand out, actual support sizes) / kernel time; the gathered rows "
                         "hit L2 (the whole fp32 dictionary when it fits), so the figure can "
                         "exceed the HBM peak"}
    if hbm_stages is not None:
        hbm_stages["ls_resid"] = resid_stage(prof_zt, c_low, n_low, 8.0, args.steps)
        hbm_stages["ls_resid_full"] = resid_stage(prof_full, ofull["counts"].cpu().numpy(),
                                                  w.n_signal, 4.0, args.full_steps)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_subprocess(ci, yd[: min(P, 8192)].double().cpu().numpy())

    extras = {}
    if rank == 0 and world == 1 and not args.no_extras:
        extras["pipeline_ends"] = bench_pipeline_ends(peaks)
        extras["ksvd_update"] = bench_ksvd_update(args.no_cpu)
        extras["operator_recovery"] = bench_operator_recovery(args.no_cpu)

    if rank == 0:
        line = {
            "metric": METRIC, "value": zt_value, "unit": "signals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": zt_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE generator drawn on the device, fp32 inputs, "
                    "fp64 dictionaries)",
            "config": workload_config(ci, total, world),
            "full_omp": {"value": full_value, "unit": "signals/s", "steps": args.full_steps,
                         "ms_per_step": full_ms / args.full_steps, "engine": engine_full[0],
                         "exact_rescans": engine_full[2], "roofline": full_roof,
                         "note": f"{args.full_steps} timed pass(es) over all {total:,} signals "
                                 "(one pass is ~10x a zero-tree step)"},
            "roofline": roofline,
            "kernels_ms_per_step": {k: v[0] / args.steps for k, v in prof_zt.items()},
            "kernels_full_ms_per_step": {k: v[0] / args.full_steps for k, v in prof_full.items()},
            "hbm_stages": hbm_stages,
            "cpu_baseline": cpu,
            "e2e": {"value": total * e2e_steps / e2e_total, "unit": "signals/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    "what": "C-ABI cdb_zero_tree_batch on pinned host rows (chunked H2D / "
                            "compute / D2H pipeline) + NCCL gather of all outputs to rank 0 "
                            "when N > 1; wall clock, max over ranks; byte counts whole-job"},
            "e2e_api": e2e_api,
            "e2e_api_full": e2e_api_full,
            "gen_s": t_gen,
            "clocks": clk,
            "gpu_launches": launches,
            **extras,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def bench_dropin(torch, ci, yd, count):
    """zero_tree_many_arrays through the Python drop-in (the call a crossdict
    user makes) on an N x P fp64 column batch in pageable host memory -- the
    reference's layout -- over the first `count` benchmark signals."""
    from paper_1511_05174_b200 import crossscale as C
    from paper_1511_05174_b200 import pursuit as PU
    from paper_1511_05174_b200.scaling import ScaleSpec
    from paper_1511_05174_b200.tensor import Dictionary
    w = W.CONFIGS[ci]
    if w.measurements:
        return None
    d = W.dictionaries(ci)
    m = int(min(count, yd.shape[0]))
    cols = yd[:m].T.contiguous().double().cpu().numpy()  # N x P fp64, pageable
    model = C.CrossScaleModel(Dictionary(np.ascontiguousarray(d.low_t.T)),
                              Dictionary(np.ascontiguousarray(d.high_t.T)),
                              ScaleSpec(w.fine_shape, w.factors), w.k, w.k)
    old = PU.REL_RESIDUAL_TOL
    PU.REL_RESIDUAL_TOL = W.REL_TOL
    try:
        # warm call (dictionary staging, pinned staging buffers), then the timed call
        t0 = time.perf_counter()
        C.zero_tree_many_arrays(model, cols)
        first = time.perf_counter() - t0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        low, high, tim = C.zero_tree_many_arrays(model, cols)
        dt = time.perf_counter() - t0
    finally:
        PU.REL_RESIDUAL_TOL = old
    # the column ABI stages fp32 over PCIe when every value is fp32-exact
    h2d_es = 4 if np.array_equal(cols.astype(np.float32), cols) else 8
    return {"value": m / dt, "unit": "signals/s", "signals": m, "seconds": dt,
            "first_call_s": first, "device_s": tim, "h2d_bytes_per_step": m * w.n_high * h2d_es,
            "d2h_bytes_per_step": int(sum(a.nbytes for a in (low.sel, low.alpha, low.counts,
                                                             low.rnorm, low.scans, high.sel,
                                                             high.alpha, high.counts,
                                                             high.rnorm, high.scans))),
            "what": "paper_1511_05174_b200.crossscale.zero_tree_many_arrays(model, ys) with ys "
                    "an N x P fp64 pageable numpy array, returning BatchSolve objects; the batch "
                    "crosses the C ABI as columns (cdb_zero_tree_batch_cols: host threads stage "
                    "column slabs into pinned memory, fp32 when exact, the device transposes, "
                    "chunks pipelined); includes every copy and the output allocation"}


def bench_dropin_full(torch, ci, yd, count):
    """omp_many_arrays (full OMP) through the Python drop-in on an N x P fp64
    pageable column batch over the first `count` benchmark signals -- the
    full-dictionary twin of bench_dropin (cdb_omp_batch_cols underneath)."""
    from paper_1511_05174_b200 import pursuit as PU
    w = W.CONFIGS[ci]
    if w.measurements or count <= 0:
        return None
    d = W.dictionaries(ci)
    m = int(min(count, yd.shape[0]))
    cols = yd[:m].T.contiguous().double().cpu().numpy()  # N x P fp64, pageable
    mat = np.ascontiguousarray(d.high_t.T)
    old = PU.REL_RESIDUAL_TOL
    PU.REL_RESIDUAL_TOL = W.REL_TOL
    try:
        t0 = time.perf_counter()
        PU.omp_many_arrays(mat, cols, PU.PursuitConfig(w.k))
        first = time.perf_counter() - t0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = PU.omp_many_arrays(mat, cols, PU.PursuitConfig(w.k))
        dt = time.perf_counter() - t0
    finally:
        PU.REL_RESIDUAL_TOL = old
    h2d_es = 4 if np.array_equal(cols.astype(np.float32), cols) else 8
    return {"value": m / dt, "unit": "signals/s", "signals": m, "seconds": dt,
            "first_call_s": first, "h2d_bytes_per_step": m * w.n_high * h2d_es,
            "d2h_bytes_per_step": int(sum(a.nbytes for a in (s.sel, s.alpha, s.counts, s.rnorm,
                                                             s.scans))),
            "what": "paper_1511_05174_b200.pursuit.omp_many_arrays(columns, ys, config) with ys an "
                    "N x P fp64 pageable numpy array (cdb_omp_batch_cols: column slabs staged, "
                    "transposed on the device, tolerances on the device)"}


def bench_operator_recovery(no_cpu=False):
    """per-patch operator recovery (pipelines._recover_operator)
    through the public recover_operator -- a 512 x 512 x 3 image behind a
    random channel mosaic, 8 x 8 x 3 patches at stride 2 (64 009 patches),
    single-scale OMP with K = 6 over 384 atoms -- beside the oracle's
    restatement of the reference (per-patch numpy + the C kernel, 1 thread)
    on a 96 x 96 crop of the same problem."""
    import time as _t
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle"))
    from paper_1511_05174_b200 import sensing as S
    from paper_1511_05174_b200.pipelines import recover_operator
    rng = np.random.default_rng(3)
    h = w = 512
    c = 3
    img = np.cumsum(rng.standard_normal((h, w, c)), axis=0) / 8
    a = rng.integers(1, c + 1, size=h * w)
    op = S.make_channel_mosaic(h * w, c, a)
    coded = op.apply(img.ravel()).reshape(h, w)
    patch, stride = (8, 8, 3), (2, 2, 1)
    d = rng.standard_normal((192, 384))
    d /= np.linalg.norm(d, axis=0)
    recover_operator(coded, op, patch, stride, dictionary=d, sparsity=6)  # warm-up
    t0 = _t.perf_counter()
    _, met, _ = recover_operator(coded, op, patch, stride, dictionary=d, sparsity=6)
    el = _t.perf_counter() - t0
    out = {"workload": "512x512x3 image, random channel mosaic, 8x8x3 patches stride 2, "
                       "K=6 over 384 atoms (exact engine, coded rows)",
           "patches": met.patch_count, "ms": el * 1e3, "patches_per_s": met.patch_count / el}
    if not no_cpu:
        import operator_oracle as OO
        hs = 96
        g = dict(kind="channel-mosaic", assignment=a.reshape(h, w)[:hs, :hs].ravel(), channels=c,
                 sig_shape=np.array((hs, hs, c)), patch=np.array(patch), stride=np.array(stride),
                 meas=coded[:hs, :hs], method="omp-single", atoms=d, k=6)
        t1 = _t.perf_counter()
        OO.recover(g)
        pc = ((hs - 8) // 2 + 1) ** 2
        out["cpu_reference_patches_per_s"] = pc / (_t.perf_counter() - t1)
        out["cpu_kind"] = ("port (oracle/operator_oracle.py: the reference's per-patch "
                           "slicing + the C kernel restatement, 1 thread, 96x96 crop)")
    return out


def bench_ksvd_update(no_cpu=False):
    """SURVEY §8 row f1 follow-on: K-SVD's dictionary-update stage
    (learn._update_stage) on the device -- one call through the public
    learn.update_stage (host E = Y - D X, transfers, the device atom loop) --
    beside the oracle's restatement of the reference stage (numpy + LAPACK,
    the box's host) on the same seeded problem: N=64, T=256, M=20000, K=8,
    two dead atoms."""
    import time as _t
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle"))
    import ksvd_oracle as KO
    from paper_1511_05174_b200 import _native as NN
    from paper_1511_05174_b200.learn import update_stage
    y, d, x = KO.problem(64, 256, 20000, 8, 7, (3, 4))
    update_stage(y, d.copy(), x.copy(), 2)  # warm-up
    d1, x1 = d.copy(), x.copy()
    NN.profile_enable(True)
    t0 = _t.perf_counter()
    rep = update_stage(y, d1, x1, 2)[0]
    t1 = _t.perf_counter()
    prof = NN.profile_read()
    NN.profile_enable(False)
    out = {"workload": "N=64, T=256, M=20000 signals, K=8, 2 dead atoms (seeded)",
           "replaced": rep, "call_ms": (t1 - t0) * 1e3,
           "kernel_ms": prof.get("ksvd_update", (0.0,))[0]}
    if not no_cpu:
        d2, x2 = d.copy(), x.copy()
        t2 = _t.perf_counter()
        KO.update_stage(y, d2, x2, 2)
        out["cpu_reference_ms"] = (_t.perf_counter() - t2) * 1e3
        out["cpu_kind"] = "port (oracle/ksvd_oracle.py: the reference stage's numpy/LAPACK calls)"
    # whole training iterations (row f1): learn.ksvd, codes / residual / refits on the device
    from paper_1511_05174_b200 import learn as LL
    cfg = LL.TrainConfig(256, 8, iterations=3, seed=0)
    LL.ksvd(y[:, :2000], LL.TrainConfig(256, 8, iterations=1, seed=0))  # warm-up
    t3 = _t.perf_counter()
    _, _, rep_d = LL.ksvd(y, cfg)
    train = {"workload": "K-SVD, N=64, T=256, M=20000, K=8, 3 iterations (seeded data)",
             "device_s": _t.perf_counter() - t3,
             "objective_per_iteration": [float(v) for v in rep_d.objective_per_iteration]}
    if not no_cpu:
        thr = len(os.sched_getaffinity(0))
        t4 = _t.perf_counter()
        _, _, _, post, _ = KO.train(y, 256, 8, 3, seed=0, nthreads=thr)
        train["cpu_reference_s"] = _t.perf_counter() - t4
        train["cpu_kind"] = (f"port (oracle: C coding kernel on {thr} threads + the reference "
                             "update stage's numpy/LAPACK calls)")
        train["cpu_objective_per_iteration"] = [float(v) for v in post]
    out["training"] = train
    return out


def bench_pipeline_ends(peaks, reps=3):
    """SURVEY §8 row f2 measurement: the device-resident image recovery chain
    extract_patches -> zero-tree OMP -> reconstruct + overlap-add on a
    1024 x 1024 image with configs[0]'s 8 x 8 patches (stride 1, ~1.03 M
    patches) and model; device times by CUDA events, HBM roofline of the two
    memory-bound ends (algorithmic bytes: patch rows written/read once, the
    image read/written once)."""
    import torch
    from paper_1511_05174_b200 import device as D
    from paper_1511_05174_b200 import patchwork as PW
    w = W.CONFIGS[0]
    d = W.dictionaries(0)
    rng = np.random.default_rng(7)
    img = torch.from_numpy(np.cumsum(rng.standard_normal((1024, 1024)), axis=1) / 32.0).cuda()
    patch, stride = w.fine_shape, (1, 1)
    p = PW.patch_count(img.shape, patch, stride)
    n = w.n_high
    rows = torch.empty((p, n), dtype=torch.float64, device="cuda")
    dc = torch.empty(p, dtype=torch.float64, device="cuda")
    est = torch.empty_like(img)
    lo, hi = D.device_dictionary(d.low_t), D.device_dictionary(d.high_t)

    def outs(k):
        return dict(sel=torch.empty((p, k), dtype=torch.int64, device="cuda"),
                    alpha=torch.empty((p, k), dtype=torch.float64, device="cuda"),
                    counts=torch.empty(p, dtype=torch.int64, device="cuda"),
                    rnorm=torch.empty(p, dtype=torch.float64, device="cuda"),
                    scans=torch.empty(p, dtype=torch.int64, device="cuda"),
                    flag=torch.empty(p, dtype=torch.uint8, device="cuda"))
    ol, oh = outs(w.k), outs(w.k)
    stream = torch.cuda.current_stream()

    def run(ev):
        ev[0].record(stream)
        D.extract_patches_raw(img, patch, stride, True, rows, dc)
        ev[1].record(stream)
        D.zero_tree_raw(lo, hi, w.fine_shape, w.factors, rows, p, w.k, w.k, W.REL_TOL, False,
                        "auto", ol, oh)
        ev[2].record(stream)
        D.reconstruct_aggregate_raw(hi, oh["sel"], oh["alpha"], p, dc, tuple(img.shape), patch,
                                    stride, est)
        ev[3].record(stream)

    evs = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    run(evs)
    torch.cuda.synchronize()
    t = np.zeros(3)
    for _ in range(reps):
        run(evs)
        torch.cuda.synchronize()
        t += [evs[i].elapsed_time(evs[i + 1]) for i in range(3)]
    t /= reps
    cells = img.numel()
    b_extract = 8.0 * (cells + p * n + p)           # image in, rows + dc out
    b_recon = 8.0 * (p * n + p + 2 * p * w.k + cells)  # est rows (+dc), codes, image out
    hbm = peaks["hbm_gbs"]
    ach = b_extract / (t[0] * 1e-3) / 1e9
    return {"workload": f"1024x1024 fp64 image, {patch[0]}x{patch[1]} patches stride 1 "
                        f"({p} patches), configs[0] zero-tree model, K={w.k}, remove_dc",
            "patches_per_s": p / (t.sum() * 1e-3), "unit": "patches/s",
            "ms": {"extract_patches": t[0], "zero_tree": t[1], "reconstruct_aggregate": t[2]},
            "roofline": {"bound": "hbm", "kernel": "extract_patches", "achieved": ach,
                         "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": None,
                         "reconstruct_aggregate_gbs": b_recon / (t[2] * 1e-3) / 1e9}}


def self_launch(args):
    """`--gpus N` without torchrun: run this script under torchrun, N ranks."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # communicator init (nranks) on stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--num-signals", type=int, default=0,
                    help="total signals over all GPUs (default: the config's)")
    ap.add_argument("--full-steps", type=int, default=1, help="timed full-OMP passes")
    ap.add_argument("--e2e-steps", type=int, default=3, help="timed e2e passes (<= steps)")
    ap.add_argument("--api-signals", type=int, default=131072, help="signals of the e2e_api leg")
    ap.add_argument("--api-full-signals", type=int, default=32768,
                    help="signals of the full-OMP e2e_api_full leg")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-api", action="store_true", help="skip the e2e_api leg")
    ap.add_argument("--no-extras", action="store_true", help="skip the f-row legs")
    ap.add_argument("--cpu-sample", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.cpu_sample:  # internal: the cpu_baseline leg in a clean process
        print(json.dumps(cpu_baseline(args.config, np.load(args.cpu_sample))), flush=True)
        return 0
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    if args.impl == "reference":
        return bench_reference(args)
    return bench_ours(args)


if __name__ == "__main__":
    sys.exit(main())
