#!/usr/bin/env python
"""Benchmark of the rcscm hot path on B200 (one JSON line on rank 0).

Headline workload: BASELINE.json configs[3], the largest configuration that fits
one GPU -- 256 independent utterances, each M = 4 mics, I = 513 bins, J = 320
frames (42.0 M time-frequency slots, x = 2.69 GB complex128), 100 iterations of
the accelerated rule (Algorithm 2, solver_accel.hpp:254). Synthetic inputs from
the BASELINE recipe (paper_1908_01964_b200/synth.py), utterance u drawn with
seed 3000 + u, generated once on the host; both arms use the same seeds and
print the same `config` dict.

A step = run_algorithm2 over the whole batch with its inputs resident in HBM:
one fused K2 launch (restore params0, the sigma/tau precompute in its prologue,
100 on-chip iterations per bin).
value  = 256 * I * J * iters / (max-over-ranks device time per step).
With N GPUs (torchrun) the 256 utterances are split into contiguous balanced
ranges, one per rank (strong scaling: total work fixed; no collective in the
solve, the timing MAX is the only NCCL traffic).
e2e    = the same metric through the C ABI entry point rcscm_gpu_run_algorithm2
         with page-locked host buffers in the reference layout: each rank's
         utterances as one call (bins flattened), H2D of X, a, b, R'^+ and
         params0 and D2H of r_h, r_u, lambda inside the timed region.
extras (N = 1): every other BASELINE config (C0, C1, C2, C4 in complex128 and
complex64, C3 in complex64), the naive rule, the Wiener output after the solve,
and the K1 / K4 stream kernels -- each with its own roofline.
--impl reference runs the oracle port (the reference's CPU algorithm restated in
oracle/; the reference itself needs Eigen and cannot be built here) on the host
cores over a bounded sample of the same utterances.
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

CFG = 3  # BASELINE configs[3]: the largest single-GPU configuration
FLOPS_ACCEL = 47.0  # canonical flops per slot-iteration
FLOPS_NAIVE = {2: 341.0, 4: 1804.0, 8: 11052.0}
# K1 / K4 algorithmic bytes per slot (complex128): SURVEY 8(d). The timed K1 is
# the sigma/tau pass only: read x (16 M) + write sigma_bx, tau_ax, tau_xx (40);
# SURVEY's 88/120/184 also count the r_h0 / r_u0 writes of the setup pass.
BYTES_PRE = {2: 72.0, 4: 104.0, 8: 168.0}
BYTES_WIENER = {2: 96.0, 4: 128.0, 8: 192.0}
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # HGX B200 spec class
NOMINAL_FP32_TFLOPS = 2 * NOMINAL_FP64_TFLOPS
METRIC = "TF-slot updates/s (I*J*iters/s), accelerated rule (Algorithm 2)"
UNIT = "TF-slot updates/s"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def partition(n, world):
    """Contiguous balanced ranges (paper_1908_01964_b200.shard.partition)."""
    from paper_1908_01964_b200.shard import partition as p

    return p(n, world)


def headline_config(n_gpus):
    """The `config` dict both arms print (identical for the same --gpus)."""
    from paper_1908_01964_b200 import synth

    c = synth.CONFIGS[CFG]
    return {"workload": c["name"], "M": c["M"], "I": c["I"], "J": c["J"], "utterances": c["B"],
            "iters": c["iters"], "rule": "accel2 (Algorithm 2, solver_accel.hpp:183-258)",
            "seeds": f"utterance u: {1000 * CFG} + u", "precision": "complex128",
            "parallelism": f"{c['B']} utterances in contiguous ranges over {n_gpus} GPU(s), no collective in the solve",
            "l2": "inputs (x 2.69 GB + state) exceed the 126 MB L2; a 256 MiB write + read also flushes it between steps"}


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


def ncu_summary(kernel_key):
    """The committed ncu summary entry (profiles/ncu_summary.json) or {}."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel_key, {})
    except (OSError, ValueError):
        return {}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def gen_batch(cfg, lo, hi, I=None, J=None):
    """Utterances [lo, hi) of BASELINE config `cfg` (seed 1000 cfg + u) stacked as
    X (n, I, J, M), W, A (n, I, M, M), T (n, I, K), V (n, K, J), written in place
    (no second copy of x)."""
    from paper_1908_01964_b200 import synth

    c = synth.CONFIGS[cfg]
    I, J, M = I or c["I"], J or c["J"], c["M"]
    n = hi - lo
    X = np.empty((n, I, J, M), np.complex128)
    W = np.empty((n, I, M, M), np.complex128)
    A = np.empty((n, I, M, M), np.complex128)
    T = np.empty((n, I, 4))
    V = np.empty((n, 4, J))
    for k, u in enumerate(range(lo, hi)):
        ut = synth.make_utterance(M, I, J, c["d"], 1000 * cfg + u)
        X[k], W[k], A[k], T[k], V[k] = ut.X, ut.W, ut.A, ut.T, ut.V
    return X, W, A, T, V


# ---- the reference arm / cpu_baseline: the oracle on the host cores -------------------
def oracle_batch(X, W, A, T, V):
    """Oracle setup (build_noise_scm + init_params per utterance, model.hpp:58-124),
    concatenated over utterances along the bin axis: every equation of
    Algorithm 2 is per bin, so one oracle call over the concatenation is the
    same computation as one call per utterance."""
    from oracle import oracle as O

    O.build()
    ins, ps = [], []
    for k in range(X.shape[0]):
        inp = O.build_noise_scm(W[k], A[k], X[k], 0)
        ins.append(inp)
        ps.append(O.init_params(inp, T[k], V[k], W[k], A[k], X[k]))
    cat = lambda f, xs: np.concatenate([getattr(x, f) for x in xs], axis=0)
    inp = O.Inputs(cat("a", ins), cat("R_prime", ins), cat("R_prime_pinv", ins), cat("b", ins), 0)
    p0 = O.Params(cat("r_h", ps), cat("r_u", ps), cat("lam", ps))
    return O, inp, p0, X.reshape(-1, X.shape[2], X.shape[3])


def oracle_rate(steps, warmup, budget_s, threads):
    """Times the oracle port of Algorithm 2 (all 100 iterations) on the first n of
    the headline's utterances, n sized so steps + warmup runs take ~budget_s.
    Returns (value slot-updates/s, per-step seconds, n, description)."""
    from paper_1908_01964_b200 import synth

    c = synth.CONFIGS[CFG]
    iters = c["iters"]
    X, W, A, T, V = gen_batch(CFG, 0, 1)
    O, inp, p0, Xf = oracle_batch(X, W, A, T, V)
    t0 = time.perf_counter()
    O.run("accel2_binparallel", inp, p0, Xf, O.SolverOptions(iters=iters, threads=threads))
    per_utt = max(time.perf_counter() - t0, 1e-4)
    n = int(max(1, min(c["B"], budget_s / max(steps + warmup, 1) / per_utt)))
    if n > 1:
        X, W, A, T, V = gen_batch(CFG, 0, n)
        O, inp, p0, Xf = oracle_batch(X, W, A, T, V)
    for _ in range(warmup):
        O.run("accel2_binparallel", inp, p0, Xf, O.SolverOptions(iters=iters, threads=threads))
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        O.run("accel2_binparallel", inp, p0, Xf, O.SolverOptions(iters=iters, threads=threads))
        times.append(time.perf_counter() - t0)
    slot_iters = n * c["I"] * c["J"] * iters
    value = slot_iters * steps / sum(times)
    desc = (f"oracle port of Algorithm 2 (solver_accel.hpp:183-240, incl. the sigma/tau precompute), utterances "
            f"0..{n - 1} of the {c['B']} (seeds {1000 * CFG}..{1000 * CFG + n - 1}, the GPU arm's first {n}), all "
            f"{iters} iterations, {steps} timed runs after {warmup} warm-up; bins over {threads} threads; per-utterance "
            f"work is identical so the rate scales linearly to the full batch; host {cpu_model()}")
    return value, times, n, desc


def single_thread_rate():
    """The reference-faithful serial restatement (solver_accel.hpp:183-240 is
    single-threaded): median per-iteration time after 3 warm-ups (metrics.hpp:43-51)."""
    from paper_1908_01964_b200 import synth

    c = synth.CONFIGS[CFG]
    X, W, A, T, V = gen_batch(CFG, 0, 1)
    O, inp, p0, Xf = oracle_batch(X, W, A, T, V)
    r = O.run("accel2", inp, p0, Xf, O.SolverOptions(iters=6))
    t = statistics.median(r.iter_seconds[3:])
    return c["I"] * c["J"] / t


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    value, times, n, desc = oracle_rate(args.steps, args.warmup, 150.0, threads)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE recipe: sinc-coherent diffuse noise + NMF-variance target, 0 dB)",
        "config": headline_config(args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference (C++/Eigen) cannot be built in this image (Eigen absent); oracle/ restates its "
                "algorithm line by line; each step is a bounded sample of the headline batch: "
                f"{n} of {headline_config(args.gpus)['utterances']} utterances, host threads: {threads}",
    }
    print(json.dumps(line), flush=True)


# ---- GPU arm -----------------------------------------------------------------------------
class Dev:
    """Per-process device handles shared by the measurements."""

    def __init__(self, local, torch):
        self.torch = torch
        self.local = local
        self.dev = torch.device("cuda", local)
        self.stream = torch.cuda.Stream(device=self.dev)
        self.l2 = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=self.dev)
        self.l2_acc = torch.empty(1, dtype=torch.float32, device=self.dev)

    def flush(self):
        # a 256 MiB write then a read of it: L2 ends full of CLEAN lines, so the
        # next kernel's misses do not first write back ~126 MB of dirty flush
        # data (measured on B200: a write-only flush costs a following 20 us
        # stream kernel ~2 us, tools/stream_flush_ab.py)
        with self.torch.cuda.stream(self.stream):
            self.l2.fill_(1.0)
            self.l2_acc.copy_(self.l2.sum())

    def event(self):
        return self.torch.cuda.Event(enable_timing=True)


def fp_probe(ctx, fp32=False):
    import paper_1908_01964_b200._capi as C

    tf, ms = ctypes.c_double(), ctypes.c_double()
    fn = C.load().rcscm_gpu_probe_fp32 if fp32 else C.load().rcscm_gpu_probe_fp64
    rc = fn(ctx.handle, ctypes.byref(tf), ctypes.byref(ms))
    return (tf.value, ms.value) if rc == 0 else (None, None)


def accel_roofline(ms, slots, iters, M, peak, f32=False, kernel="", ncu_key=None):
    """FP64 (FP32 in complex64) roofline of one fused K2 launch: 47 flops per
    slot-iteration + the sigma / tau forms once per slot (b^H x and
    (R'^+ a)^H x: 8 M each; x^H R'^+ x from the lower triangle: 4 M^2 + 15 M)."""
    pre = 4.0 * M * M + 15.0 * M
    flops = FLOPS_ACCEL * slots * iters + pre * slots
    achieved = flops / (ms * 1e-3) / 1e12
    nominal = NOMINAL_FP32_TFLOPS if f32 else NOMINAL_FP64_TFLOPS
    nc = ncu_summary(ncu_key) if ncu_key else {}
    return {"bound": "fp32" if f32 else "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak if peak else None, "nominal_peak": nominal, "frac_of_nominal": achieved / nominal,
            "traffic": nc.get("dram_bytes_per_launch"), "kernel": kernel,
            "flops_per_slot_iter": FLOPS_ACCEL, "slot_iters_per_launch": slots * iters,
            "precompute_flops_per_slot": pre, "flops_per_launch": flops, "avg_launch_ms": ms,
            "peak_source": ("measured live on this GPU: " + ("FFMA" if f32 else "DFMA") + " probe (rcscm_gpu_probe_"
                            + ("fp32" if f32 else "fp64") + "); MEASURED_PEAKS.json has no FP64/FP32 figure"),
            "ncu": {k: nc.get(k) for k in ("fp64_pipe_inst_pct", "stall_long_sb_per_issue", "duration_ns")} if nc
            else None}


def session_for(d, cfg, lo=0, hi=None, precision="c128", I=None, J=None, data=None):
    from paper_1908_01964_b200 import GpuContext, synth
    import paper_1908_01964_b200._capi as C

    c = synth.CONFIGS[cfg]
    hi = c["B"] if hi is None else hi
    X, W, A, T, V = data if data is not None else gen_batch(cfg, lo, hi, I, J)
    ctx = GpuContext(d.local, precision=precision, stream=d.stream.cuda_stream)
    ctx.session_load(X, W, A, T, V, 0)
    ctx.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    ctx.session_check()
    return ctx, X.shape


def time_stages(d, ctx, stages, iters, reps, hyper, pre_stages=0, flush=True):
    """Mean / min device time (ms) of session_run(stages) over reps after one
    untimed run; pre_stages run untimed before each (e.g. RESET)."""
    ctx.session_run(stages | pre_stages, iters, hyper)
    ts = []
    for _ in range(reps):
        if pre_stages:
            ctx.session_run(pre_stages, 0, hyper)
        if flush:
            d.flush()
        e0, e1 = d.event(), d.event()
        e0.record(d.stream)
        ctx.session_run(stages, iters, hyper)
        e1.record(d.stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ctx.session_check()
    return statistics.mean(ts), min(ts)


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_1908_01964_b200 import Hyperparams, synth
    import paper_1908_01964_b200._capi as C

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    d = Dev(local, torch)
    if world > 1:
        dist.init_process_group("nccl", device_id=d.dev)
    c = synth.CONFIGS[CFG]
    iters = c["iters"]
    lo, hi = partition(c["B"], world)[rank]
    hyper = Hyperparams()
    data = gen_batch(CFG, lo, hi)
    from paper_1908_01964_b200 import GpuContext
    from paper_1908_01964_b200.shard import ShardedSession

    ctx = GpuContext(d.local, stream=d.stream.cuda_stream)
    sharded = ShardedSession(ctx, c["B"], rank, world, *data)
    sharded.run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    ctx.session_check()
    B, I, J, M = data[0].shape
    step_stages = C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL

    for _ in range(args.warmup):
        ctx.session_run(step_stages, iters, hyper)
    torch.cuda.synchronize(d.dev)
    ctx.session_check()

    ev = [(d.event(), d.event()) for _ in range(args.steps)]

    def lead_in(seconds):  # untimed steps while the clock sampler starts
        t_end = time.perf_counter() + seconds
        while time.perf_counter() < t_end:
            for _ in range(4):
                d.flush()
                ctx.session_run(step_stages, iters, hyper)
            torch.cuda.synchronize(d.dev)

    with ClockSampler(local, lead_in) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(d.dev)
        launches0 = ctx.launch_count
        for k in range(args.steps):
            d.flush()  # L2 flush between steps (outside the events)
            e0, e1 = ev[k]
            e0.record(d.stream)
            ctx.session_run(step_stages, iters, hyper)
            e1.record(d.stream)
        torch.cuda.synchronize(d.dev)
    launches = (ctx.launch_count - launches0) / args.steps
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], device=d.dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        dist.barrier()
    ctx.session_check()
    S_all = c["B"] * c["I"] * c["J"]
    value = S_all * iters * args.steps / (tot_ms * 1e-3)
    fp64_peak, probe_ms = fp_probe(ctx)
    k2_avg = sum(step_ms) / len(step_ms)
    roofline = accel_roofline(k2_avg, B * I * J, iters, M, fp64_peak,
                              kernel=("k_accel<10,1,FULL,-,0,8,DIRECT,double,PREM=4,-,WE=2> (one-warp CTAs)" if B * I >= 2048
                                      else "k_accel<5,1,FULL,-,0,8,DIRECT,double,PREM=4> (64 x 5 CTAs)")
                              + " (K2: sigma/tau precompute fused "
                                     "into the prologue, then the on-chip Algorithm 2 iterations), this rank's "
                                     f"{B} utterances x {I} bins", ncu_key="k_accel_c3")
    roofline["peak_probe"] = {"tflops": fp64_peak, "ms": probe_ms, "sm_mhz_during_bench": None}
    # the final gather of r_h, r_u, lambda and the Wiener dry output to rank 0
    # (the only communication), timed separately after one untimed
    # solve + extract step: device-to-device into transfer tensors, then NCCL
    ctx.session_run(step_stages | C.STAGE_WIENER, iters, hyper)
    ctx.session_check()
    gather = gather_measure(d, sharded, world, B, I, J)
    ctx.close()

    # e2e through the C ABI with pinned host buffers (reference layout), this
    # rank's utterances as one call
    e2e = e2e_measure(d, data, iters, hyper, args, world, S_all)
    del data

    out = None
    extras = run_extras(d, hyper, args) if world == 1 else run_extras_multi(d, hyper, args, rank, world)
    if rank == 0:
        clocks = clk.summary()
        roofline["peak_probe"]["sm_mhz_during_bench"] = clocks.get("sm_mhz")
        cpu = None
        if world == 1:  # rank 0 at N = 1 only
            threads = os.cpu_count() or 1
            v, times, n, desc = oracle_rate(1, 1, 20.0, threads)
            cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc,
                   "single_thread_value": single_thread_rate(),
                   "single_thread_sample": "serial restatement of run_algorithm2 (the reference's accel2 is "
                                           "single-threaded) on utterance 0: median per-iteration time after 3 "
                                           "warm-ups (metrics.hpp:43-51)"}
        out = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": tot_ms / args.steps,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (BASELINE recipe: sinc-coherent diffuse noise + NMF-variance target, 0 dB)",
            "config": headline_config(world),
            "gpu_launches": launches,
            "breakdown_ms": {"fused_k2": k2_avg, "rank0_utterances": B},
            "roofline": roofline,
            "e2e": e2e,
            "gather": gather,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "extras": extras,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_extras(d, hyper, args):
    """Every other BASELINE config, the naive rule, the Wiener output and the
    stream kernels, one session at a time (N = 1)."""
    import paper_1908_01964_b200._capi as C
    from paper_1908_01964_b200 import synth

    torch = d.torch
    out = {}
    peaks = load_peaks()
    hbm = peaks.get("hbm_gbs", 6554.2)
    reps = max(3, min(args.steps, 10))
    step = C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL
    fp64_peak = fp32_peak = None

    def stream_entry(ms, bps, n):
        gbs = bps * n / (ms * 1e-3) / 1e9
        return {"ms": ms, "bytes_per_slot": bps, "slots": n, "achieved_gbs": gbs, "peak_gbs": hbm,
                "frac": gbs / hbm, "frac_basis": "of measured (MEASURED_PEAKS.json hbm_gbs)"}

    for cfg in (0, 1, 2, 4):
        c = synth.CONFIGS[cfg]
        ctx, (B, I, J, M) = session_for(d, cfg)
        if fp64_peak is None:
            fp64_peak, _ = fp_probe(ctx)
        S = B * I * J
        mean, best = time_stages(d, ctx, step, c["iters"], reps, hyper)
        e = {"workload": c["name"], "iters": c["iters"], "ms_per_step": mean, "ms_min": best,
             "value": S * c["iters"] / (mean * 1e-3), "unit": UNIT,
             "roofline": accel_roofline(mean, S, c["iters"], M, fp64_peak, kernel="fused K2 (k_accel, PREM=M)",
                                        ncu_key=f"k_accel_c{cfg}")}
        if cfg in (0, 1):
            # the Wiener output from the resident state (K4) and the standalone
            # precompute (K1), one launch after an L2 flush
            pre, _ = time_stages(d, ctx, C.STAGE_PRECOMPUTE, 0, reps, hyper)
            wie, _ = time_stages(d, ctx, C.STAGE_WIENER, 0, reps, hyper)
            e["k_pre"] = stream_entry(pre, BYTES_PRE[M], S)
            e["k_wiener"] = stream_entry(wie, BYTES_WIENER[M], S)
        if c["naive_iters"]:
            n_it = c["naive_iters"]
            nm, _ = time_stages(d, ctx, C.STAGE_NAIVE, n_it, 2, hyper, pre_stages=C.STAGE_RESET)
            e["naive"] = naive_entry(nm, S, n_it, M, fp64_peak, mean / c["iters"])
        out[f"c{cfg}"] = e
        ctx.close()
        if cfg == 4:
            cx, _ = session_for(d, cfg, precision="c64")
            mean64, best64 = time_stages(d, cx, step, c["iters"], reps, hyper)
            if fp32_peak is None:
                fp32_peak, _ = fp_probe(cx, fp32=True)
            out["c4_c64"] = {"workload": c["name"] + "_c64", "iters": c["iters"], "ms_per_step": mean64,
                             "value": S * c["iters"] / (mean64 * 1e-3), "unit": UNIT,
                             "roofline": accel_roofline(mean64, S, c["iters"], M, fp32_peak, f32=True,
                                                        kernel="K1 (FP32) + K2<float>", ncu_key="k_accel_c4_c64"),
                             "note": "complex64 mode: x, sigma/tau and the slot arithmetic in FP32, lambda in FP64; "
                                     "output within relative-L2 1e-4 of complex128 (tests)"}
            cx.close()
        torch.cuda.empty_cache()

    # the headline batch: complex64, naive, Wiener / precompute stream kernels
    c = synth.CONFIGS[CFG]
    ctx, (B, I, J, M) = session_for(d, CFG)
    S = B * I * J
    base_mean, _ = time_stages(d, ctx, step, c["iters"], 3, hyper)
    pre, _ = time_stages(d, ctx, C.STAGE_PRECOMPUTE, 0, reps, hyper)
    wie, _ = time_stages(d, ctx, C.STAGE_WIENER, 0, reps, hyper)
    nm, _ = time_stages(d, ctx, C.STAGE_NAIVE, c["naive_iters"], 2, hyper, pre_stages=C.STAGE_RESET)
    solve_ext, _ = time_stages(d, ctx, step | C.STAGE_WIENER, c["iters"], 3, hyper)
    out["c3_stream"] = {"k_pre": stream_entry(pre, BYTES_PRE[M], S), "k_wiener": stream_entry(wie, BYTES_WIENER[M], S),
                        "note": "one launch over all 256 utterances after an L2 flush (the streaming regime)"}
    out["c3_naive"] = naive_entry(nm, S, c["naive_iters"], M, fp64_peak, base_mean / c["iters"])
    out["c3_solve_then_extract"] = {"ms_per_step": solve_ext, "value": S * c["iters"] / (solve_ext * 1e-3),
                                    "unit": UNIT, "wiener_extra_ms": solve_ext - base_mean,
                                    "note": "run_algorithm2 then extract_target (dry + image) on the resident batch"}
    ctx.close()
    torch.cuda.empty_cache()
    cx, _ = session_for(d, CFG, precision="c64")
    m64, _ = time_stages(d, cx, step, c["iters"], reps, hyper)
    out["c3_c64"] = {"workload": c["name"] + "_c64", "ms_per_step": m64, "value": S * c["iters"] / (m64 * 1e-3),
                     "unit": UNIT, "roofline": accel_roofline(m64, S, c["iters"], M, fp32_peak, f32=True,
                                                              kernel="K1 (FP32) + K2<float>")}
    cx.close()
    torch.cuda.empty_cache()
    out["peaks"] = {"fp64_dfma_probe_tflops": fp64_peak, "fp32_ffma_probe_tflops": fp32_peak,
                    "fp64_nominal_tflops": NOMINAL_FP64_TFLOPS, "hbm_gbs": hbm}
    return out


def gather_measure(d, sharded, world, B, I, J):
    """Max-over-ranks device time of ShardedSession.gather (fetch into transfer
    tensors + NCCL point-to-point to rank 0) of r_h, r_u, lambda and dry."""
    import torch
    import torch.distributed as dist

    dev = f"cuda:{d.local}"
    for _ in range(2):  # warm-up (NCCL communicator set-up on the first call)
        sharded.gather(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(d.dev)
    t0 = time.perf_counter()
    out = sharded.gather(dev)
    torch.cuda.synchronize(d.dev)
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt], device=d.dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    nbytes = sharded.B * I * (J * (8 + 8 + 16) + 8)
    del out
    return {"ms": dt * 1e3, "bytes_total": nbytes, "bytes_over_links": nbytes * (world - 1) / world,
            "path": "session outputs copied device-to-device into torch transfer tensors, then point-to-point "
                    "to rank 0 (NCCL; the only communication of the job), max over ranks of the wall time "
                    "between device synchronisations"}


def run_extras_multi(d, hyper, args, rank, world):
    """N > 1: config 4 strong-sharded over BINS (rank r solves bins
    partition(2049, N)[r] of the one utterance), max-over-ranks device time."""
    import torch
    import torch.distributed as dist

    import paper_1908_01964_b200._capi as C
    from paper_1908_01964_b200 import GpuContext, synth
    from paper_1908_01964_b200.shard import partition as part

    c = synth.CONFIGS[4]
    X, W, A, T, V = gen_batch(4, 0, 1)
    lo, hi = part(c["I"], world)[rank]
    ctx = GpuContext(d.local, stream=d.stream.cuda_stream)
    ctx.session_load(X[:, lo:hi], W[:, lo:hi], A[:, lo:hi], T[:, lo:hi], V, 0)
    ctx.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    step = C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL
    dist.barrier()
    mean, _ = time_stages(d, ctx, step, c["iters"], max(3, min(args.steps, 10)), hyper)
    t = torch.tensor([mean], device=d.dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ctx.close()
    S = c["I"] * c["J"]
    return {"c4_bins_sharded": {"workload": c["name"], "ms_per_step": float(t.item()), "bins_rank0": hi - lo,
                                "value": S * c["iters"] / (float(t.item()) * 1e-3), "unit": UNIT,
                                "note": f"2049 bins in contiguous ranges over {world} GPUs, max-over-ranks time"}}


def naive_entry(ms, S, iters, M, fp64_peak, accel_ms_per_iter):
    canon = FLOPS_NAIVE.get(M, 0) * S * iters / (ms * 1e-3) / 1e12
    return {"iters": iters, "ms_per_run": ms, "value": S * iters / (ms * 1e-3), "unit": UNIT,
            "throughput_equivalent_tflops": canon, "canonical_flops_per_slot_iter": FLOPS_NAIVE.get(M),
            "throughput_equivalent_frac": canon / fp64_peak if fp64_peak else None,
            "accel_over_naive_per_iteration": (ms / iters) / accel_ms_per_iter,
            "note": "k_naive forms R_x^-1 per slot but consumes R^_u only through b^H R^_u b and tr(R_u^-1 R^_u), "
                    "so it executes fewer flops than the canonical count: the TFLOP/s figure is a throughput-"
                    "equivalent, not a pipe utilisation (see profiles/ncu_summary.json k_naive for the FP64 pipe)"}


def e2e_measure(d, data, iters, hyper, args, world, S_all):
    """rcscm_gpu_run_algorithm2 with page-locked host inputs/outputs (reference
    layout): this rank's utterances as one call (bins flattened utterance-major,
    as a reference caller concatenating RcscmInputs would pass them). Whole-job
    value = all ranks' slot-iterations over the slowest rank's mean call time;
    byte counts are summed over ranks."""
    import paper_1908_01964_b200._capi as C
    from paper_1908_01964_b200 import GpuContext

    torch = d.torch
    X, W, A, T, V = data
    B, I, J, M = X.shape
    ctx = GpuContext(d.local)  # a fresh context, as a caller of the C ABI has
    lib = C.load()
    rt = ctypes.CDLL("libcudart.so.12")
    held = []

    # page-locked host buffers from cudaHostAlloc, as a C caller would allocate
    # them (torch's pin_memory() blocks measured 27-37 GB/s of H2D on the B200
    # box against 52 GB/s for cudaHostAlloc memory: tools/pin_probe.py)
    def pinned_empty(n):
        p = ctypes.c_void_p()
        if rt.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(max(n, 1) * 8), ctypes.c_uint(0)) != 0:
            raise RuntimeError("cudaHostAlloc failed")
        held.append(p)
        return np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(max(n, 1),))[:n]

    nb = B * I
    Xp = pinned_empty(nb * J * M * 2)
    Xp[:] = X.reshape(-1).view(np.float64)
    ap, bp = pinned_empty(nb * M * 2), pinned_empty(nb * M * 2)
    rpp = pinned_empty(nb * M * M * 2)
    rh0, ru0, l0 = pinned_empty(nb * J), pinned_empty(nb * J), pinned_empty(nb)
    rh0v, ru0v = rh0.reshape(J, nb), ru0.reshape(J, nb)  # I x J column-major
    for k in range(B):
        inp = ctx.build_noise_scm(W[k], A[k], X[k], 0)
        p0 = ctx.init_params(inp, T[k], V[k], W[k], A[k], X[k])
        s = slice(k * I, (k + 1) * I)
        ap.reshape(nb, M * 2)[s] = inp.a.view(np.float64).reshape(I, M * 2)
        bp.reshape(nb, M * 2)[s] = inp.b.view(np.float64).reshape(I, M * 2)
        rpp.reshape(nb, M * M * 2)[s] = np.ascontiguousarray(inp.R_prime_pinv.transpose(0, 2, 1)).view(
            np.float64).reshape(I, M * M * 2)
        rh0v[:, s] = p0.r_h.T
        ru0v[:, s] = p0.r_u.T
        l0[s] = p0.lam
    rh, ru, lam = pinned_empty(nb * J), pinned_empty(nb * J), pinned_empty(nb)
    dp = lambda a: ctypes.cast(a.ctypes.data, C._dp)
    ci = C.CInputs(nb, J, M, 0, dp(ap), None, dp(rpp), dp(bp))
    cp = C.CParams(dp(rh0), dp(ru0), dp(l0))
    co = C.CParams(dp(rh), dp(ru), dp(lam))
    h = C.CHyper(hyper.alpha, hyper.beta)
    o = C.COpts(iters, 0, 0, 0.0, 1, 1e-12, 0.0)

    def call():
        rc = lib.rcscm_gpu_run_algorithm2(ctx.handle, ctypes.byref(ci), ctypes.byref(cp), ctypes.byref(h), dp(Xp),
                                          ctypes.byref(o), ctypes.byref(co), None)
        if rc != 0:
            raise RuntimeError(lib.rcscm_gpu_last_error().decode())

    for _ in range(max(args.warmup, 3)):
        call()
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    dt = sum(ts) / args.steps
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([dt], device=d.dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    h2d = (Xp.size + ap.size + bp.size + rpp.size + rh0.size + ru0.size + l0.size) * 8
    d2h = (rh.size + ru.size + lam.size) * 8
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([h2d, d2h], device=d.dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        h2d, d2h = int(t[0].item()), int(t[1].item())
    for p in held:
        rt.cudaFreeHost(p)
    ctx.close()
    return {"value": S_all * iters / dt, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": dt * 1e3, "h2d_gbs": h2d / world / dt / 1e9,
            "path": "rcscm_gpu_run_algorithm2 (C ABI, synchronous) with cudaHostAlloc host buffers in the reference "
                    f"layout, host wall clock; each rank's {B} utterances as one call ({nb} bins)"
                    + (f"; {world} ranks, slowest rank's time" if world > 1 else "")}


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
