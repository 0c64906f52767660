"""Times cmd_extract's pipeline on the device (rcscm_gpu_extract) against the
oracle chain on one host thread, on the reference's test configuration (4 mics,
8.7 s at 16 kHz: 513 bins x 273 frames; K = 10 bases, 50 ILRMA sweeps, 100
Algorithm 2 iterations with the objective every iteration)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1908_01964_b200 import GpuContext
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_extract import _mixture, _oracle_extract  # noqa: E402
from oracle import oracle as O  # noqa: E402

SR = 16000.0
x = _mixture(4, 139200, 1)
ctx = GpuContext(0)
for _ in range(2):
    g = ctx.extract(x, SR, nmf_bases=10, ilrma_iters=50, seed=1, iters=100)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    g = ctx.extract(x, SR, nmf_bases=10, ilrma_iters=50, seed=1, iters=100)
    ts.append(time.perf_counter() - t0)
print(f"gpu extract (host buffers in/out): {min(ts)*1e3:.1f} ms  target_index {g['target_index']}", flush=True)
t0 = time.perf_counter()
tw, nw, n_h, obj = _oracle_extract(O, x, 10, 50, 1, 100)
tc = time.perf_counter() - t0
err = float(np.max(np.abs(g["target"] - tw)) / np.max(np.abs(tw)))
print(f"oracle chain (1 thread): {tc*1e3:.0f} ms  n_h {n_h}  speed-up {tc/min(ts):.0f}x  max rel diff {err:.2e}")
