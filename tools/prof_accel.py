"""Runs the bench workload's device step (C1 unless --cfg) a few times; used
under ncu to capture k_accel / k_slots / k_naive, and for SPT sweeps."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1908_01964_b200 import GpuContext, Hyperparams, synth
import paper_1908_01964_b200._capi as C

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--naive", action="store_true")
ap.add_argument("--wiener", action="store_true")
ap.add_argument("--I", type=int, default=None)
ap.add_argument("--J", type=int, default=None)
ap.add_argument("--B", type=int, default=1)
ap.add_argument("--c64", action="store_true")
ap.add_argument("--unfused", action="store_true", help="K2 alone (forms from K1's arrays)")
ap.add_argument("--iters", type=int, default=None, help="override the config's iteration count")
ap.add_argument("--epi", action="store_true", help="solve + extract in one call (K2 with the fused Wiener epilogue)")
a = ap.parse_args()
c = dict(synth.CONFIGS[a.cfg])
if a.iters is not None:
    c["iters"] = a.iters
utts = synth.make_config(a.cfg, utterances=a.B, I=a.I, J=a.J)
X, W, A, T, V = synth.stack(utts)
s = torch.cuda.Stream()
ctx = GpuContext(0, precision="c64" if a.c64 else "c128", stream=s.cuda_stream)
ctx.session_load(X, W, A, T, V, 0)
ctx.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
h = Hyperparams()
ev = []
for r in range(a.reps + 5):  # the first 5 are warm-up (clocks ramp after an idle GPU)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.session_run(C.STAGE_RESET | C.STAGE_PRECOMPUTE, 0, h)
    e0.record(s)
    if a.wiener:
        ctx.session_run(C.STAGE_WIENER, 0, h)
    elif a.naive:
        ctx.session_run(C.STAGE_NAIVE, c["naive_iters"], h)
    elif a.unfused:
        ctx.session_run(C.STAGE_ACCEL, c["iters"], h)
    else:  # the bench step: precompute fused into K2
        ctx.session_run(C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL | (C.STAGE_WIENER if a.epi else 0), c["iters"], h)
    e1.record(s)
    ev.append((e0, e1))
torch.cuda.synchronize()
ctx.session_check()
ms = min(e0.elapsed_time(e1) for e0, e1 in ev[5:])
B, I, J, M = X.shape
it = 1 if a.wiener else (c["naive_iters"] if a.naive else c["iters"])
print(f"{'c64' if a.c64 else 'c128'} cfg{a.cfg} B={B} I={I} J={J} {'wiener' if a.wiener else ('naive' if a.naive else 'accel')} spt={os.environ.get('RCSCM_ACCEL_SPT','auto')} "
      f"cl={os.environ.get('RCSCM_ACCEL_CL','auto')}: {ms:.4f} ms  {B*I*J*it/(ms*1e-3)/1e9:.1f} G slot-it/s  "
      f"{47*B*I*J*it/(ms*1e-3)/1e12:.2f} TF(47)")
