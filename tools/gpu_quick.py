"""Quick GPU sanity + timing probe (development helper, run under gpurun)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import __graft_entry__ as G
from oracle import oracle as O
from paper_1908_01964_b200 import GpuContext, Hyperparams, SolverOptions, synth
import paper_1908_01964_b200._capi as C

G.smoke()
ctx = GpuContext(0)
hyper = Hyperparams()
for cfg, I, J in [(0, 64, 320), (1, 64, 640), (4, 16, 4096), (2, 8, 20000), (1, 16, 16)]:
    u = synth.make_config(cfg, utterances=1, I=I, J=J)[0]
    oinp = O.build_noise_scm(u.W, u.A, u.X, 0)
    op0 = O.init_params(oinp, u.T, u.V, u.W, u.A, u.X)
    inp = ctx.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = ctx.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    print(f"cfg{cfg} I={I} J={J}: init parity {O.trajectory_distance(p0, op0):.2e}", flush=True)
    for it in (1, 10):
        g = ctx.run_algorithm2(oinp, op0, hyper, u.X, SolverOptions(iters=it)).params
        o = O.run("accel2", oinp, op0, u.X, O.SolverOptions(iters=it)).params
        line = f"   accel iters={it} {O.trajectory_distance(g, o):.2e}"
        if J <= 4096:
            gn = ctx.run_naive(oinp, op0, hyper, u.X, SolverOptions(iters=it)).params
            on = O.run("naive", oinp, op0, u.X, O.SolverOptions(iters=it)).params
            line += f"  naive {O.trajectory_distance(gn, on):.2e}"
        print(line, flush=True)

# timing C1 full via the session
u = synth.make_config(1, utterances=1)[0]
X, W, A, T, V = synth.stack([u])
ctx.session_load(X, W, A, T, V, 0)
ctx.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
ctx.session_check()
import torch
s = torch.cuda.ExternalStream(ctx.stream)
for stages, iters, name in [(C.STAGE_RESET | C.STAGE_ACCEL, 100, "accel100"), (C.STAGE_RESET | C.STAGE_NAIVE, 10, "naive10"),
                            (C.STAGE_PRECOMPUTE, 0, "precompute"), (C.STAGE_WIENER, 0, "wiener"), (C.STAGE_SETUP, 0, "setup")]:
    for w in range(3):
        ctx.session_run(stages, iters)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for k in range(5):
        ctx.session_run(stages, iters)
    e1.record(s); e1.synchronize()
    ms = e0.elapsed_time(e1) / 5
    slots = u.X.shape[0] * u.X.shape[1]
    print(f"{name}: {ms:.3f} ms  -> {slots * max(iters,1) / (ms * 1e-3) / 1e9:.2f} G slot-updates/s", flush=True)
ctx.session_check()
