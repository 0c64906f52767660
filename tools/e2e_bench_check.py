"""bench.py's e2e leg in isolation: fresh context vs a context on a torch stream
that first ran session work (as in bench.py)."""
import os, sys, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1908_01964_b200 import GpuContext, Hyperparams, synth
import paper_1908_01964_b200._capi as C

u = synth.make_config(1, utterances=1, seed_base=1001)[0]
args = argparse.Namespace(steps=10, warmup=3)
h = Hyperparams()
ctx = GpuContext(0)
print("fresh ctx, own stream:", bench.e2e_measure(ctx, u, 100, h, args, torch)["ms_per_step"])
s = torch.cuda.Stream()
ctx2 = GpuContext(0, stream=s.cuda_stream)
print("torch stream ctx:", bench.e2e_measure(ctx2, u, 100, h, args, torch)["ms_per_step"])
X, W, A, T, V = synth.stack([u])
ctx2.session_load(X, W, A, T, V, 0)
ctx2.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
ctx2.session_run(C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL, 100, h)
print("after session work:", bench.e2e_measure(ctx2, u, 100, h, args, torch)["ms_per_step"])
print("again:", bench.e2e_measure(ctx2, u, 100, h, args, torch)["ms_per_step"])
import time, ctypes, numpy as np
# per-call wall times of a fresh set of pinned buffers
lib = C.load()
for trial in range(2):
    r = bench.e2e_measure(ctx2, u, 100, h, argparse.Namespace(steps=30, warmup=0), torch)
    print("30 calls, no warm-up: mean", r["ms_per_step"])
