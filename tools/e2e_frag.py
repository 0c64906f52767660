import os, sys, time, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_1908_01964_b200 import GpuContext, Hyperparams, synth
class A: warmup = 3; steps = 10
u = synth.make_config(1, utterances=1, seed_base=1001)[0]
ctx = GpuContext(0)
r = bench.e2e_measure(ctx, u, 100, Hyperparams(), A, torch)
print("fresh process:", r["ms_per_step"])
junk = [np.ones(64 * 1024 * 1024) for _ in range(int(sys.argv[1]))]  # 512 MB each
big = torch.empty(512 * 1024 * 1024, dtype=torch.uint8).pin_memory() if len(sys.argv) > 2 else None
r = bench.e2e_measure(ctx, u, 100, Hyperparams(), A, torch)
print("after", sys.argv[1:], ":", r["ms_per_step"])
