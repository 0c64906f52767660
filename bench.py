#!/usr/bin/env python
"""Benchmark of the rcscm hot path on B200 (one JSON line on rank 0).

Workload (BASELINE.json configs[1], the single-GPU config the metric is quoted
on): one utterance, M = 4 mics, I = 1025 bins, J = 640 frames, 100 iterations of
the accelerated rule (Algorithm 2, solver_accel.hpp:254), complex128. Synthetic
inputs from the BASELINE recipe (paper_1908_01964_b200/synth.py), seed
1000 * 1 + rank, generated once on the host.

A step = run_algorithm2 on the device with its inputs resident in HBM: one
fused K2 launch (restore params0, the sigma/tau precompute in its prologue,
100 on-chip iterations). K1 and K4 are timed alone (cold L2) as extras.
value  = B * I * J * iters * n_gpus / (max-over-ranks device time per step).
e2e    = the same metric through the C ABI entry point rcscm_gpu_run_algorithm2
         with pinned host buffers in the reference layout (H2D of X, inputs and
         params0, D2H of r_h, r_u, lambda inside the timed region).
naive  = the naive rule (solver_naive.hpp:412) on the same resident inputs.
--impl reference runs the oracle port (the reference's CPU algorithm,
restated in oracle/; the reference itself needs Eigen and cannot be built here).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = 1
FLOPS_ACCEL = 47.0  # canonical flops per slot-iteration
FLOPS_NAIVE = {2: 341.0, 4: 1804.0, 8: 11052.0}
# K1 / K4 algorithmic bytes per slot (complex128): SURVEY 8(d). The timed step's
# K1 is the sigma/tau pass only: read x (16 M) + write sigma_bx, tau_ax, tau_xx (40);
# SURVEY's 88/120/184 also count the r_h0 / r_u0 writes of the setup pass.
BYTES_PRE = {2: 72.0, 4: 104.0, 8: 168.0}
BYTES_WIENER = {2: 96.0, 4: 128.0, 8: 192.0}
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # HGX B200 spec class


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device, lead_in=None):
        self.device = device
        self.proc = None
        # lead_in(seconds): keeps the GPU under load while nvidia-smi starts (an
        # idle lead-in lets the clocks drop: measured on B200, the first K2 steps
        # after 0.3 s of idle run up to 15 % slow and take ~6 steps to recover)
        self.lead_in = lead_in

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
        if self.lead_in is not None:
            self.lead_in(0.3)
        else:
            time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def ncu_traffic(kernel_key):
    """dram bytes per launch from the committed ncu summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(kernel_key, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def workload_config():
    from paper_1908_01964_b200 import synth

    c = synth.CONFIGS[CFG]
    return c


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_problem(u):
    from oracle import oracle as O

    O.build()
    inp = O.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    return O, inp, p0


def cpu_baseline(u, c, budget_s=10.0, threads=None):
    """Oracle port of Algorithm 2 on the host cores over a bounded sample of the
    workload: all I bins, J frames, as many iterations as fit ~budget_s."""
    O, inp, p0 = oracle_problem(u)
    threads = threads or os.cpu_count() or 1
    I, J = u.X.shape[0], u.X.shape[1]
    t0 = time.perf_counter()
    O.run("accel2_binparallel", inp, p0, u.X, O.SolverOptions(iters=2, threads=threads))
    per_it = max((time.perf_counter() - t0) / 2, 1e-6)
    iters = int(max(2, min(c["iters"], budget_s / per_it)))
    # repeat the run until ~budget_s of CPU time has been spent (a 16-thread run
    # of the full config is ~0.2 s, too short for a stable figure)
    runs, dt = 0, 0.0
    while runs < 3 or dt < budget_s:
        t0 = time.perf_counter()
        O.run("accel2_binparallel", inp, p0, u.X, O.SolverOptions(iters=iters, threads=threads))
        dt += time.perf_counter() - t0
        runs += 1
        if dt > 3 * budget_s:
            break
    # reference-faithful single thread (solver_accel.hpp:183-240 is serial), few iterations
    it1 = 3
    r1 = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=it1 + 3))
    t_single = statistics.median(r1.iter_seconds[3:]) if len(r1.iter_seconds) > 3 else r1.iter_seconds[-1]
    return {
        "value": I * J * iters * runs / dt,
        "unit": "TF-slot updates/s",
        "cores": threads,
        "kind": "port",
        "sample": f"oracle Algorithm 2, all {I} bins x {J} frames, {iters} iterations (incl. sigma/tau precompute), "
                  f"{runs} runs ({dt:.1f} s), bins split over {threads} threads; host {cpu_model()}",
        "single_thread_value": I * J / t_single,
        "single_thread_sample": "serial restatement of run_algorithm2 (the reference's accel2 is single-threaded), "
                                "median per-iteration time after 3 warm-ups (metrics.hpp:43-51)",
    }


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1908_01964_b200 import synth

    c = workload_config()
    u = synth.make_config(CFG, utterances=1)[0]
    O, inp, p0 = oracle_problem(u)
    threads = os.cpu_count() or 1
    I, J = u.X.shape[0], u.X.shape[1]
    # size each step as a bounded sample: the full config if it fits ~20 s per step
    t0 = time.perf_counter()
    O.run("accel2_binparallel", inp, p0, u.X, O.SolverOptions(iters=2, threads=threads))
    per_it = max((time.perf_counter() - t0) / 2, 1e-6)
    total_budget = 150.0
    iters = int(max(1, min(c["iters"], total_budget / max(args.steps + args.warmup, 1) / per_it)))
    for _ in range(args.warmup):
        O.run("accel2_binparallel", inp, p0, u.X, O.SolverOptions(iters=iters, threads=threads))
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.run("accel2_binparallel", inp, p0, u.X, O.SolverOptions(iters=iters, threads=threads))
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = I * J * iters * args.steps / tot
    sample = (f"oracle port of Algorithm 2 (solver_accel.hpp:183-240) on the full config-1 problem "
              f"({I} bins x {J} frames), {iters} of {c['iters']} iterations per step, bins over {threads} threads; "
              f"host {cpu_model()}")
    line = {
        "impl": "reference",
        "metric": "TF-slot updates/s (I*J*iters/s), accelerated rule (Algorithm 2)",
        "value": value,
        "unit": "TF-slot updates/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE recipe, seed 1001)",
        "config": {"workload": c["name"], "M": c["M"], "I": c["I"], "J": c["J"], "iters_per_step": iters,
                   "rule": "accel2"},
        "cpu_baseline": {"value": value, "unit": "TF-slot updates/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "TF-slot updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference (C++/Eigen) cannot be built in this image; oracle/ restates its algorithm",
    }
    print(json.dumps(line), flush=True)


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_1908_01964_b200 import GpuContext, Hyperparams, synth
    import paper_1908_01964_b200._capi as C

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    c = workload_config()
    u = synth.make_config(CFG, utterances=1, seed_base=1000 * CFG + rank)[0]
    X, W, A, T, V = synth.stack([u])
    B, I, J, M = X.shape
    iters = c["iters"]
    tstream = torch.cuda.Stream(device=dev)
    ctx = GpuContext(local, stream=tstream.cuda_stream)
    hyper = Hyperparams()
    ctx.session_load(X, W, A, T, V, 0)
    ctx.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    ctx.session_check()
    l2_flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def flush():
        with torch.cuda.stream(tstream):
            l2_flush.fill_(1.0)

    # one step = run_algorithm2 on resident inputs: restore params0, sigma / tau
    # precompute, 100 iterations -- one fused K2 launch (precompute in its prologue)
    step_stages = C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL

    # warm-up
    for _ in range(args.warmup):
        ctx.session_run(step_stages, iters, hyper)
    torch.cuda.synchronize(dev)
    ctx.session_check()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    def lead_in(seconds):  # untimed steps while the clock sampler starts
        t_end = time.perf_counter() + seconds
        while time.perf_counter() < t_end:
            for _ in range(20):
                flush()
                ctx.session_run(step_stages, iters, hyper)
            torch.cuda.synchronize(dev)

    with ClockSampler(local, lead_in) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        launches0 = ctx.launch_count
        for k in range(args.steps):
            flush()  # L2 flush between steps (outside the events)
            e0, e1 = ev[k]
            e0.record(tstream)
            ctx.session_run(step_stages, iters, hyper)
            e1.record(tstream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = (ctx.launch_count - launches0) / args.steps
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    k2_ms = step_ms  # the step is the single fused K2 launch
    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    ctx.session_check()
    slot_iters = B * I * J * iters
    value = slot_iters * world * args.steps / (tot_ms * 1e-3)

    # roofline of K2 (FP64 pipe) against the measured DFMA peak
    tf = ctypes.c_double()
    pm = ctypes.c_double()
    rc = C.load().rcscm_gpu_probe_fp64(ctx.handle, ctypes.byref(tf), ctypes.byref(pm))
    fp64_peak = tf.value if rc == 0 else NOMINAL_FP64_TFLOPS
    k2_avg = sum(k2_ms) / len(k2_ms)
    # algorithmic flops of the fused launch: the sigma / tau forms once per slot
    # (b^H x and (R'^+ a)^H x: 8 M each; x^H R'^+ x with R'^+ Hermitian: 3 M on the
    # diagonal + 8 per lower-triangle pair -> 4 M^2 + 15 M) plus 47 per
    # slot-iteration
    pre_flops = 4.0 * M * M + 15.0 * M
    launch_flops = FLOPS_ACCEL * slot_iters + pre_flops * B * I * J
    achieved = launch_flops / (k2_avg * 1e-3) / 1e12
    roofline = {"bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak, "traffic": ncu_traffic("k_accel"),
                "kernel": "k_accel<PREM=M> (K2 with the sigma/tau precompute fused into its prologue, then the "
                          "on-chip Algorithm 2 iterations)",
                "flops_per_slot_iter": FLOPS_ACCEL, "slot_iters_per_launch": slot_iters,
                "precompute_flops_per_slot": pre_flops, "flops_per_launch": launch_flops,
                "avg_launch_ms": k2_avg,
                "peak_source": "measured live: DFMA probe (rcscm_gpu_probe_fp64) on this GPU; MEASURED_PEAKS.json "
                               "has no FP64 figure",
                "frac_basis": "of measured (FP64 pipe; the kernel is neither HBM- nor tensor-bound)",
                "nominal_peak": NOMINAL_FP64_TFLOPS,
                "frac_of_nominal": achieved / NOMINAL_FP64_TFLOPS}

    # secondary kernels: K1 precompute and K4 wiener (HBM), naive rule (FP64)
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    S = B * I * J

    def timed(stages, n, reps=5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.session_run(stages, n, hyper)
        flush()
        e0.record(tstream)
        for _ in range(reps):
            ctx.session_run(stages, n, hyper)
        e1.record(tstream)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    naive_iters = c["naive_iters"]
    naive_ms = timed(C.STAGE_RESET | C.STAGE_NAIVE, naive_iters, reps=3)
    ctx.session_check()
    stream_kernels = stream_measure(ctx, tstream, flush, hyper, S, M, hbm, X, W, A, T, V, local, torch, C)
    naive = {"value": S * naive_iters / (naive_ms * 1e-3), "unit": "TF-slot updates/s", "iters": naive_iters,
             "ms_per_run": naive_ms,
             "achieved_tflops_canonical": FLOPS_NAIVE.get(M, 0) * S * naive_iters / (naive_ms * 1e-3) / 1e12,
             "canonical_flops_per_slot_iter": FLOPS_NAIVE.get(M),
             "accel_over_naive_per_iteration": (naive_ms / naive_iters) / (k2_avg / iters)}

    # complex64 (FP32) mode of the same step, against the measured FP32 peak
    c64 = c64_measure(local, tstream, X, W, A, T, V, iters, hyper, S, args, torch, C)

    # e2e through the C ABI with pinned host buffers (reference layout)
    # (a fresh context, as a caller of the C ABI has: no session state, its own stream)
    e2e_ctx = GpuContext(local)
    e2e = e2e_measure(e2e_ctx, u, iters, hyper, args, torch, world, dev)
    e2e_ctx.close()

    out = None
    if rank == 0:
        clocks = clk.summary()
        cpu = cpu_baseline(u, c) if world == 1 else None  # rank 0 at N = 1 only
        out = {
            "metric": "TF-slot updates/s (I*J*iters/s), accelerated rule (Algorithm 2)",
            "value": value,
            "unit": "TF-slot updates/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (BASELINE recipe: sinc-coherent diffuse noise + NMF-variance target, 0 dB; seed 1001+rank)",
            "config": {"workload": c["name"], "M": M, "I": I, "J": J, "utterances_per_gpu": B, "iters": iters,
                       "step": "run_algorithm2 on resident inputs: params0, sigma/tau precompute fused into the "
                               "prologue of K2, 100 on-chip iterations (one kernel)",
                       "l2": "flushed between steps (256 MiB write, outside the timed events)",
                       "clock_lead_in": "0.3 s of untimed steps while nvidia-smi starts, so the timed steps "
                                        "do not start from an idle GPU",
                       "parallelism": f"bins sharded by utterance, {world} GPU(s), no collective in the loop"},
            "gpu_launches": launches,
            "breakdown_ms": {"fused_k2": k2_avg},
            "roofline": roofline,
            "stream_kernels": stream_kernels,
            "naive": naive,
            "c64": c64,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "clocks": clocks,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()


def stream_measure(ctx, tstream, flush, hyper, S, M, hbm, X, W, A, T, V, local, torch, C):
    """K1 (standalone precompute) and K4 (Wiener) against the HBM peak: the
    bench-utterance launch timed alone after an L2 flush (68 / 84 MB: launch-
    latency bound), the same launch 8 times back to back on distinct copies
    (steady state), and one launch over a batch of 8 copies (0.5 / 0.7 GB: the
    streaming regime the batched configs run in)."""
    from paper_1908_01964_b200 import GpuContext
    import numpy as np

    def cold(cx, stages, reps=7):
        ts = []
        for r in range(reps + 1):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(tstream)
            cx.session_run(stages, 0, hyper)
            e1.record(tstream)
            e1.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    def entry(ms, bps, n):
        gbs = bps * n / (ms * 1e-3) / 1e9
        return {"ms": ms, "bytes_per_slot": bps, "slots": n, "achieved_gbs": gbs, "peak_gbs": hbm, "frac": gbs / hbm,
                "frac_basis": "of measured (MEASURED_PEAKS.json hbm_gbs)"}

    ctx.session_run(C.STAGE_PRECOMPUTE, 0, hyper)
    out = {"k_pre": entry(cold(ctx, C.STAGE_PRECOMPUTE), BYTES_PRE.get(M, 0), S),
           "k_wiener": entry(cold(ctx, C.STAGE_WIENER), BYTES_WIENER.get(M, 0), S)}

    def copy_cold(nbytes, reps=7):
        # torch's device copy moving the same bytes (half read, half written),
        # timed like the kernels: what a plain stream achieves at this size
        n = max(int(nbytes // 8), 1)
        src = torch.ones(n, dtype=torch.float32, device=f"cuda:{local}")
        dst = torch.empty_like(src)
        ts = []
        for r in range(reps + 1):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(tstream)
            with torch.cuda.stream(tstream):
                dst.copy_(src)
            e1.record(tstream)
            e1.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    for name, bps in (("copy_same_bytes_as_k_pre", BYTES_PRE.get(M, 0)), ("copy_same_bytes_as_k_wiener",
                                                                           BYTES_WIENER.get(M, 0))):
        out[name] = entry(copy_cold(bps * S), bps, S)
    nb = 8
    # the single-utterance launch in steady state: 8 contexts, each holding its own
    # copy of the utterance (0.5 GB in all, > L2), launched back to back after one
    # flush, so each launch streams cold data and the launch latency overlaps
    ctxs = [GpuContext(local, stream=tstream.cuda_stream) for _ in range(nb)]
    for cx in ctxs:
        cx.session_load(X, W, A, T, V, 0)
        cx.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
        cx.session_run(C.STAGE_ACCEL, 3, hyper)

    def chain(stages, reps=5):
        ts = []
        for r in range(reps + 1):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(tstream)
            for cx in ctxs:
                cx.session_run(stages, 0, hyper)
            e1.record(tstream)
            e1.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1) / nb)
        return statistics.median(ts)

    out["k_pre_steady"] = entry(chain(C.STAGE_PRECOMPUTE), BYTES_PRE.get(M, 0), S)
    out["k_wiener_steady"] = entry(chain(C.STAGE_WIENER), BYTES_WIENER.get(M, 0), S)
    for cx in ctxs:
        cx.session_check()
        cx.close()
    big = GpuContext(local, stream=tstream.cuda_stream)
    rep = lambda v: np.concatenate([v] * nb, axis=0)
    big.session_load(rep(X), rep(W), rep(A), rep(T), rep(V), 0)
    big.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    big.session_run(C.STAGE_ACCEL, 3, hyper)
    out["k_pre_batch8"] = entry(cold(big, C.STAGE_PRECOMPUTE), BYTES_PRE.get(M, 0), S * nb)
    out["k_wiener_batch8"] = entry(cold(big, C.STAGE_WIENER), BYTES_WIENER.get(M, 0), S * nb)
    big.session_check()
    big.close()
    out["note"] = ("k_pre / k_wiener: one launch alone after an L2 flush (launch latency included); *_steady: "
                   "the same single-utterance launch, 8 back to back on distinct copies after one flush (cold "
                   "data, latency overlapped); *_batch8: one launch over 8 utterances; algorithmic bytes (K1: "
                   "read x, write sigma_bx, tau_ax, tau_xx; K4: read sigma_bx, tau_ax, r_h, r_u, write dry + image); "
                   "copy_same_bytes_as_*: torch's device copy moving the same bytes, timed the same way (the "
                   "bandwidth a plain stream reaches at this size)")
    return out


def c64_measure(local, tstream, X, W, A, T, V, iters, hyper, S, args, torch, C):
    """The same device step in the complex64 / FP32 mode (output within
    relative-L2 1e-4 of complex128, tests/test_gpu_parity.py)."""
    from paper_1908_01964_b200 import GpuContext

    ctx = GpuContext(local, precision="c64", stream=tstream.cuda_stream)
    ctx.session_load(X, W, A, T, V, 0)
    ctx.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    for _ in range(max(args.warmup, 1)):
        ctx.session_run(C.STAGE_RESET | C.STAGE_PRECOMPUTE, 0, hyper)
        ctx.session_run(C.STAGE_ACCEL, iters, hyper)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for e0, e1, e2 in ev:
        e0.record(tstream)
        ctx.session_run(C.STAGE_RESET | C.STAGE_PRECOMPUTE, 0, hyper)
        e1.record(tstream)
        ctx.session_run(C.STAGE_ACCEL, iters, hyper)
        e2.record(tstream)
    torch.cuda.synchronize()
    ctx.session_check()
    step = sum(a.elapsed_time(c) for a, _, c in ev) / len(ev)
    k2 = sum(b.elapsed_time(c) for _, b, c in ev) / len(ev)
    tf = ctypes.c_double()
    rc = C.load().rcscm_gpu_probe_fp32(ctx.handle, ctypes.byref(tf), None)
    peak = tf.value if rc == 0 else None
    achieved = FLOPS_ACCEL * S * iters / (k2 * 1e-3) / 1e12
    ctx.close()
    return {"value": S * iters / (step * 1e-3), "unit": "TF-slot updates/s", "ms_per_step": step,
            "accel_k2_ms": k2, "achieved_tflops": achieved, "fp32_peak_tflops": peak,
            "frac": achieved / peak if peak else None,
            "note": "same step with x, sigma/tau and the slot arithmetic in single precision; lambda in double"}


def e2e_measure(ctx, u, iters, hyper, args, torch, world=1, dev=None):
    """rcscm_gpu_run_algorithm2 with pinned host inputs/outputs (reference layout).
    With N ranks each rank runs its own utterance; the whole-job value is
    N x I*J*iters over the slowest rank's mean call time, and the byte counts are
    summed over ranks."""
    import paper_1908_01964_b200._capi as C

    lib = C.load()
    inp = ctx.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = ctx.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    I, J, M = u.X.shape

    # page-locked host buffers from cudaHostAlloc, as a C caller would allocate
    # them (torch's pin_memory() blocks measured 27-37 GB/s of H2D on the B200
    # box against 52 GB/s for cudaHostAlloc / cudaHostRegister memory:
    # tools/pin_probe.py)
    rt = ctypes.CDLL("libcudart.so.12")
    held = []

    def pinned_empty(n):
        p = ctypes.c_void_p()
        if rt.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(max(n, 1) * 8), ctypes.c_uint(0)) != 0:
            raise RuntimeError("cudaHostAlloc failed")
        held.append(p)
        return np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(max(n, 1),))[:n]

    def pinned(arr):
        a = np.ascontiguousarray(arr).reshape(-1)
        out = pinned_empty(a.size)
        out[:] = a
        return out

    Xp = pinned(u.X.view(np.float64))
    ap = pinned(inp.a.view(np.float64))
    bp = pinned(inp.b.view(np.float64))
    rpp = pinned(np.ascontiguousarray(inp.R_prime_pinv.transpose(0, 2, 1)).view(np.float64))
    rh0 = pinned(np.ascontiguousarray(p0.r_h.T))
    ru0 = pinned(np.ascontiguousarray(p0.r_u.T))
    l0 = pinned(p0.lam)
    rh = pinned_empty(I * J)
    ru = pinned_empty(I * J)
    lam = pinned_empty(I)
    dp = lambda a: ctypes.cast(a.ctypes.data, C._dp)
    ci = C.CInputs(I, J, M, 0, dp(ap), None, dp(rpp), dp(bp))
    cp = C.CParams(dp(rh0), dp(ru0), dp(l0))
    co = C.CParams(dp(rh), dp(ru), dp(lam))
    h = C.CHyper(hyper.alpha, hyper.beta)
    o = C.COpts(iters, 0, 0, 0.0, 1, 1e-12, 0.0)

    def call():
        rc = lib.rcscm_gpu_run_algorithm2(ctx.handle, ctypes.byref(ci), ctypes.byref(cp), ctypes.byref(h), dp(Xp),
                                          ctypes.byref(o), ctypes.byref(co), None)
        if rc != 0:
            raise RuntimeError(lib.rcscm_gpu_last_error().decode())

    # untimed warm-up: the per-call time settles after ~10 calls (PCIe / clock
    # ramp; measured on B200, tools/e2e_bench_check.py)
    for _ in range(max(args.warmup, 10)):
        call()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    if os.environ.get("RCSCM_E2E_VERBOSE"):
        print("e2e per call (ms):", " ".join(f"{t * 1e3:.3f}" for t in ts), file=sys.stderr)
    dt = sum(ts) / args.steps
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([dt], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    h2d = (Xp.size + ap.size + bp.size + rpp.size + rh0.size + ru0.size + l0.size) * 8
    d2h = (rh.size + ru.size + lam.size) * 8
    for p in held:
        rt.cudaFreeHost(p)
    return {"value": world * I * J * iters / dt, "unit": "TF-slot updates/s", "h2d_bytes_per_step": world * h2d,
            "d2h_bytes_per_step": world * d2h, "ms_per_step": dt * 1e3,
            "path": "rcscm_gpu_run_algorithm2 (C ABI, synchronous) with pinned host buffers, host wall clock"
                    + (f"; {world} ranks, one utterance each, slowest rank's time" if world > 1 else "")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="gpu", choices=["gpu", "reference"])
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
