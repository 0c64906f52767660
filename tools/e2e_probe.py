"""Breakdown of the e2e path: pinned H2D/D2H bandwidth and the C-ABI
run_algorithm2 call with different pipeline chunk counts."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1908_01964_b200 import GpuContext, Hyperparams, synth
import paper_1908_01964_b200._capi as C

n = 42 * 2**20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
print(f"pinned H2D {n/1e6:.0f} MB: {10*n/(time.perf_counter()-t)/1e9:.1f} GB/s")
t = time.perf_counter()
for _ in range(10):
    h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
print(f"pinned D2H {n/1e6:.0f} MB: {10*n/(time.perf_counter()-t)/1e9:.1f} GB/s")

u = synth.make_config(1, utterances=1)[0]
ctx = GpuContext(0)
lib = C.load()
inp = ctx.build_noise_scm(u.W, u.A, u.X, 0)
p0 = ctx.init_params(inp, u.T, u.V, u.W, u.A, u.X)
I, J, M = u.X.shape
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
Xp = pin(u.X.view(np.float64)); ap = pin(inp.a.view(np.float64)); bp = pin(inp.b.view(np.float64))
rpp = pin(np.ascontiguousarray(inp.R_prime_pinv.transpose(0, 2, 1)).view(np.float64))
rh0 = pin(p0.r_h.T); ru0 = pin(p0.r_u.T); l0 = pin(p0.lam)
rh = torch.empty(I * J, dtype=torch.float64).pin_memory(); ru = torch.empty(I * J, dtype=torch.float64).pin_memory(); lam = torch.empty(I, dtype=torch.float64).pin_memory()
dp = lambda t: ctypes.cast(t.data_ptr(), C._dp)
ci = C.CInputs(I, J, M, 0, dp(ap), None, dp(rpp), dp(bp))
cp = C.CParams(dp(rh0), dp(ru0), dp(l0)); co = C.CParams(dp(rh), dp(ru), dp(lam))
hy = C.CHyper(1.1, 1e-16)
for iters in (100, 0):
    o = C.COpts(iters, 0, 0, 0.0, 1, 1e-12, 0.0)
    for ch in ("1", "2", "4", "8", "16"):
        os.environ["RCSCM_PIPELINE_CHUNKS"] = ch
        for _ in range(3):
            lib.rcscm_gpu_run_algorithm2(ctx.handle, ctypes.byref(ci), ctypes.byref(cp), ctypes.byref(hy), dp(Xp), ctypes.byref(o), ctypes.byref(co), None)
        t = time.perf_counter()
        for _ in range(10):
            rc = lib.rcscm_gpu_run_algorithm2(ctx.handle, ctypes.byref(ci), ctypes.byref(cp), ctypes.byref(hy), dp(Xp), ctypes.byref(o), ctypes.byref(co), None)
        dt = (time.perf_counter() - t) / 10
        print(f"iters={iters} chunks={ch}: {dt*1e3:.3f} ms rc={rc}")
