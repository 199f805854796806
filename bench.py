#!/usr/bin/env python
"""Benchmark: signals/s of zero-tree OMP (headline) and full OMP on B200.

Workload: BASELINE.json configs[1] ("video": N=256 fine / 32 coarse, T_high=2048,
T_low=256, Q=8, K=16, 100,000 signals, sigma=0.01, fp32 inputs, stop at K or
|r| <= 1e-3 |y|) -- the largest config whose metric fits one GPU comfortably.
Synthetic, seeded (paper_1511_05174_b200.workloads); each rank codes its
own 100,000-signal shard of the deterministic stream (weak scaling, no
data-path collective: signals are independent).

A step = one pass of the hot path over the whole batch.  `value` times the
step through the C ABI with the inputs resident in HBM (CUDA events on the
launching stream, L2 flushed between steps); `e2e` times the same C-ABI call
with pinned HOST buffers (H2D of the inputs and D2H of every output inside
the timed region).  `--impl reference` times the reference algorithm on the
host cores (oracle/, the C restatement of crossdict's kernel, all threads)
on a bounded sample of the same workload.

Run:  python bench.py [--gpus N --steps K --warmup W]   (torchrun for N > 1)
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


def load_traffic():
    """DRAM bytes per launch of each profiled kernel (tools/ncu_summary.py output)."""
    try:
        with open(os.path.join(REPO, "profiles", "r1_ncu_traffic.json")) as f:
            return {k: v for k, v in json.load(f).items() if not k.startswith("_")}
    except (OSError, ValueError):
        return {}


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


def run_oracle_zero_tree(ci, ys_rows, threads):
    sys.path.insert(0, os.path.join(REPO, "oracle"))
    import oracle as O
    w = W.CONFIGS[ci]
    d = W.dictionaries(ci)
    if w.measurements:
        return O.zero_tree_phi_many(d.e_low_t, d.e_high_t, w.k, w.k, ys_rows, rel_tol=W.REL_TOL,
                                    nthreads=threads)
    return O.zero_tree_many_arrays(d.low_t, d.high_t, w.fine_shape, w.factors, w.k, w.k, ys_rows,
                                   rel_tol=W.REL_TOL, nthreads=threads)


def cpu_rate(ci, threads, ys, budget_s=24.0):
    """Oracle zero-tree sig/s on a bounded sample: whole passes over the
    config's signals `ys` (the GPU batch) until ~budget_s of CPU time."""
    probe = ys[:256]
    t0 = time.perf_counter()
    run_oracle_zero_tree(ci, probe, threads)
    rate = 256 / max(time.perf_counter() - t0, 1e-6)
    target = int(max(256, rate * budget_s))
    done, dt = 0, 0.0
    while done < target:
        m = min(len(ys), target - done)
        t0 = time.perf_counter()
        run_oracle_zero_tree(ci, ys[:m], threads)
        dt += time.perf_counter() - t0
        done += m
    return done / dt, done, dt


# ------------------------------------------------------------------ reference arm
def bench_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    ci = args.config
    threads = cpu_threads()
    w = W.CONFIGS[ci]
    # bounded per-step sample so that warmup + steps finish within minutes
    probe = W.signals(ci, 0, 256)
    t0 = time.perf_counter()
    run_oracle_zero_tree(ci, probe, threads)
    rate = 256 / max(time.perf_counter() - t0, 1e-6)
    sample = int(min(w.signals, max(256, rate * 4.0)))
    ys = W.signals(ci, 0, sample)
    for _ in range(args.warmup):
        run_oracle_zero_tree(ci, ys[: min(sample, 512)], threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run_oracle_zero_tree(ci, ys, threads)
        times.append(time.perf_counter() - t0)
    value = sample * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "signals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator, fp32-exact inputs)",
        "config": {"workload": f"{w.name} (BASELINE configs[{ci}]) zero-tree OMP",
                   "signals_per_step": sample},
        "cpu_baseline": {"value": value, "unit": "signals/s", "cores": threads, "kind": "port",
                         "sample": f"{sample} signals of configs[{ci}] per step "
                                   f"(oracle/omp_oracle.c, {threads} threads)"},
        "e2e": {"value": value, "unit": "signals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def bench_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1511_05174_b200 import _native as N
    from paper_1511_05174_b200 import device as D

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
    P = args.signals or w.signals
    phi = bool(w.measurements)
    d = W.dictionaries(ci)
    low_t = d.e_low_t if phi else d.low_t
    high_t = d.e_high_t if phi else d.high_t
    k1 = min(w.k, w.n_signal, w.t_low) if phi else w.k
    fs = None if phi else w.fine_shape
    fa = None if phi else w.factors

    ys_host = W.signals(ci, rank * P, (rank + 1) * P).astype(np.float32)
    yd = torch.from_numpy(ys_host).cuda()
    eps_full = torch.from_numpy(
        W.REL_TOL * np.linalg.norm(ys_host.astype(np.float64), axis=1)).cuda()
    lo = D.device_dictionary(low_t)
    hi = D.device_dictionary(high_t)

    def outs(k, dev="cuda", pin=False):
        mk = (lambda shape, dt: torch.empty(shape, dtype=dt, device=dev, pin_memory=pin))
        return dict(sel=mk((P, k), torch.int64), alpha=mk((P, k), torch.float64),
                    counts=mk((P,), torch.int64), rnorm=mk((P,), torch.float64),
                    scans=mk((P,), torch.int64), flag=mk((P,), torch.uint8))

    olo, ohi, ofull = outs(k1), outs(w.k), outs(w.k)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    stream = torch.cuda.current_stream()

    def zt_step():
        D.zero_tree_raw(lo, hi, fs, fa, yd, P, k1, w.k, W.REL_TOL, phi, "auto", olo, ohi)

    def full_step():
        D.omp_batch_raw(hi, yd, P, w.k, eps_full, None, "auto", ofull)

    def timed(step, k_steps):
        total = 0.0
        for _ in range(k_steps):
            flush.zero_()
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b.record(stream)
            torch.cuda.synchronize()
            total += a.elapsed_time(b)
        t = torch.tensor([total], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        zt_step()
        full_step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    launches0 = N.launch_count()
    N.profile_enable(True)
    zt_ms = timed(zt_step, args.steps)
    prof_zt = N.profile_read()
    N.profile_enable(True)
    full_ms = timed(full_step, args.steps)
    prof_full = N.profile_read()
    N.profile_enable(False)
    launches = N.launch_count() - launches0
    clk = clocks.stop()
    engine_full = N.last_run_info()
    full_scans = ofull["scans"].double().sum().item()

    # ---- e2e through the C ABI with pinned host buffers
    yh = torch.from_numpy(ys_host).pin_memory()
    hlo, hhi = outs(k1, "cpu", True), outs(w.k, "cpu", True)
    # numpy views so the library sees host pointers
    def npv(o):
        return {k: v.numpy() for k, v in o.items()}
    hlo_n, hhi_n, yh_n = npv(hlo), npv(hhi), yh.numpy()
    D.zero_tree_raw(lo, hi, fs, fa, yh_n, P, k1, w.k, W.REL_TOL, phi, "auto", hlo_n, hhi_n)
    e2e_total = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        D.zero_tree_raw(lo, hi, fs, fa, yh_n, P, k1, w.k, W.REL_TOL, phi, "auto", hlo_n, hhi_n)
        e2e_total += time.perf_counter() - t0
    t = torch.tensor([e2e_total], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_total = float(t.item())
    h2d = P * w.n_signal * 4
    d2h = sum(v.numel() * v.element_size() for o in (hlo, hhi) for v in o.values())
    # full OMP end to end: the same C-ABI call with pinned host signals,
    # tolerances and outputs (the library pipelines chunked H2D / compute / D2H)
    hfull = outs(w.k, "cpu", True)
    hfull_n = npv(hfull)
    eps_h = eps_full.cpu().numpy()
    D.omp_batch_raw(hi, yh_n, P, w.k, eps_h, None, "auto", hfull_n)
    e2e_full_total = 0.0
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        D.omp_batch_raw(hi, yh_n, P, w.k, eps_h, None, "auto", hfull_n)
        e2e_full_total += time.perf_counter() - t0
    t = torch.tensor([e2e_full_total], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_full_total = float(t.item())
    d2h_full = sum(v.numel() * v.element_size() for v in hfull.values())

    # ---- roofline of the dominant kernel (zero-tree step), algorithmic flops
    peaks, peaks_kind = load_peaks()
    traffic_tab = load_traffic()
    low_scans = olo["scans"].double().sum().item()
    high_scans = ohi["scans"].double().sum().item()
    n_low = w.n_signal if phi else w.n_low
    f_step1 = 2.0 * n_low * low_scans + flops_ls(n_low, olo["counts"].cpu().numpy())
    f_step2 = 2.0 * w.n_signal * high_scans + flops_ls(w.n_signal, ohi["counts"].cpu().numpy())
    # algorithmic flops per launch of each OMP kernel (one launch per step per call)
    flops = {"gram_step1": f_step1, "resident_step1": f_step1, "exact_step1": f_step1,
             "gram_step2": f_step2, "resident_step2": f_step2, "exact_step2": f_step2}
    dom = max(prof_zt.items(), key=lambda kv: kv[1][0]) if prof_zt else ("none", (1.0, 1))
    dom_name, (dom_ms_total, dom_launches) = dom
    dom_ms = dom_ms_total / max(dom_launches, 1)
    p_emu = peaks["bf16_tflops"] / 6.0
    dom_flops = flops.get(dom_name, 0.0) * args.steps / max(dom_launches, 1)
    achieved = dom_flops / (dom_ms * 1e-3) / 1e12 if dom_ms > 0 else 0.0
    roofline = {"bound": "tensor", "kernel": dom_name, "achieved": achieved, "peak": p_emu,
                "unit": "TFLOP/s", "frac": achieved / p_emu if p_emu else None,
                "traffic": traffic_tab.get(dom_name),
                "basis": "SURVEY §8.0 algorithmic flops 2*N*scans + 4Nk(k-1) + 11Nk per signal "
                         f"(actual scan counts) / mean launch time; peak = {peaks_kind} bf16 "
                         f"{peaks['bf16_tflops']} TF/s / 6 (3xTF32-emulated fp32, SURVEY §8(d)); "
                         "traffic = DRAM bytes per launch from profiles/r1_ncu_traffic.json",
                "launch_ms": dom_ms}
    # full-OMP correlation kernel against the measured bf16 tensor peak: the
    # algorithmic correlation flops 2*N*scans (actual scan counts) per launch
    corr = prof_full.get("corr_topk")
    full_roof = None
    if corr:
        c_ms = corr[0] / max(corr[1], 1)
        c_flops = 2.0 * w.n_signal * full_scans * args.steps / max(corr[1], 1)
        full_roof = {"bound": "tensor", "kernel": "corr_topk",
                     "achieved": c_flops / (c_ms * 1e-3) / 1e12, "peak": peaks["bf16_tflops"],
                     "unit": "TFLOP/s",
                     "frac": c_flops / (c_ms * 1e-3) / 1e12 / peaks["bf16_tflops"],
                     "traffic": traffic_tab.get("corr_topk"), "launch_ms": c_ms,
                     "basis": "2*N*scans of the full-OMP batch (actual scan counts) / corr_topk "
                              "time; the bf16 GEMM also scores taken atoms and finished signals"}

    zt_value = world * P * args.steps / (zt_ms * 1e-3)
    full_value = world * P * args.steps / (full_ms * 1e-3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = cpu_threads()
        rate, n, dt = cpu_rate(ci, threads, ys_host.astype(np.float64))
        cpu = {"value": rate, "unit": "signals/s", "cores": threads, "kind": "port",
               "sample": f"{n} signals (passes over the {P} benchmark signals) of configs[{ci}] "
                         f"zero-tree OMP in {dt:.1f} s "
                         f"(oracle/omp_oracle.c restating crossdict's kernel, {threads} threads)"}

    ends = bench_pipeline_ends(peaks) if rank == 0 and world == 1 else None
    ksvd = bench_ksvd_update(args.no_cpu) if rank == 0 and world == 1 else None
    oprec = bench_operator_recovery(args.no_cpu) if rank == 0 and world == 1 else None

    if rank == 0:
        line = {
            "metric": METRIC, "value": zt_value, "unit": "signals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": zt_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE generator, fp32 inputs, fp64 dictionaries)",
            "config": {"workload": f"{w.name} (BASELINE configs[{ci}]) zero-tree OMP: N={w.n_high}, "
                                   f"N_low={w.n_low}, T_high={w.t_high}, T_low={w.t_low}, "
                                   f"Q={w.q}, K={w.k}, {P} signals per GPU, stop K or "
                                   f"|r|<=1e-3|y|",
                       "signals_per_gpu": P, "l2": "flushed between steps (256 MiB write)"},
            "full_omp": {"value": full_value, "unit": "signals/s",
                         "ms_per_step": full_ms / args.steps, "engine": engine_full[0],
                         "roofline": full_roof,
                         "e2e": {"value": world * P * args.steps / e2e_full_total,
                                 "unit": "signals/s", "h2d_bytes_per_step": h2d + P * 8,
                                 "d2h_bytes_per_step": d2h_full}},
            "roofline": roofline,
            "kernels_ms_per_step": {k: v[0] / args.steps for k, v in prof_zt.items()},
            "kernels_full_ms_per_step": {k: v[0] / args.steps for k, v in prof_full.items()},
            "cpu_baseline": cpu,
            "pipeline_ends": ends,
            "ksvd_update": ksvd,
            "operator_recovery": oprec,
            "e2e": {"value": world * P * args.steps / e2e_total, "unit": "signals/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "clocks": clk,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


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


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--signals", type=int, default=0, help="signals per GPU (default: config's)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    if args.impl == "reference":
        return bench_reference(args)
    return bench_ours(args)


if __name__ == "__main__":
    sys.exit(main())
