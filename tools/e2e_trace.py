"""CUPTI timeline of one e2e run_algorithm2 call (C ABI, pinned host buffers,
config 1): copies per stream and their overlap with K2."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
from paper_1908_01964_b200 import GpuContext, synth
import paper_1908_01964_b200._capi as C

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
o = C.COpts(100, 0, 0, 0.0, 1, 1e-12, 0.0)
call = lambda: lib.rcscm_gpu_run_algorithm2(ctx.handle, ctypes.byref(ci), ctypes.byref(cp), ctypes.byref(hy), dp(Xp),
                                            ctypes.byref(o), ctypes.byref(co), None)
for _ in range(5):
    call()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    call()
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"{(e.time_range.start - t0):8.1f} -> {(e.time_range.end - t0):8.1f} us  {e.name[:70]}")
import time
for _ in range(3):
    call()
ts = []
for _ in range(20):
    t = time.perf_counter()
    call()
    ts.append(time.perf_counter() - t)
ts.sort()
print(f"wall per call: min {ts[0]*1e3:.3f} ms  median {ts[10]*1e3:.3f} ms")
