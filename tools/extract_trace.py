"""Kernel timeline of one device extract (reference test configuration) via the
CUPTI activity trace of torch.profiler: per-kernel totals, the span from the
first kernel start to the last kernel end, and the idle time between kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_1908_01964_b200 import GpuContext
from test_extract import _mixture

x = _mixture(4, 139200, 1)
ctx = GpuContext(0)
kw = dict(nmf_bases=10, ilrma_iters=50, seed=1, iters=100)
for _ in range(2):
    ctx.extract(x, 16000.0, **kw)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    ctx.extract(x, 16000.0, **kw)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
tot = {}
for e in ev:
    d = e.time_range.end - e.time_range.start
    n, s = tot.get(e.name, (0, 0.0))
    tot[e.name] = (n + 1, s + d)
busy = sum(s for _, s in tot.values())
span = ev[-1].time_range.end - ev[0].time_range.start
print(f"events {len(ev)}  span {span/1e3:.2f} ms  busy {busy/1e3:.2f} ms  idle {(span-busy)/1e3:.2f} ms")
for name, (n, s) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{s/1e3:8.3f} ms  {n:5d}x  {name[:110]}")
# the largest gaps (phase boundaries / host syncs)
gaps = [(ev[k + 1].time_range.start - ev[k].time_range.end, ev[k].name[:50], ev[k + 1].name[:50])
        for k in range(len(ev) - 1)]
gaps.sort(reverse=True)
for g, a, b in gaps[:12]:
    print(f"gap {g:8.1f} us  after {a}  before {b}")
# phase view: every event preceded by > 5 us of idle, with its offset
t0 = ev[0].time_range.start
print("--- timeline (events after > 5 us idle) ---")
for k, e in enumerate(ev):
    g = e.time_range.start - ev[k - 1].time_range.end if k else 0.0
    if k == 0 or g > 5.0:
        print(f"#{k:4d} t={(e.time_range.start - t0)/1e3:7.3f} ms  idle {g:7.1f} us  dur {(e.time_range.end - e.time_range.start):7.1f} us  {e.name[:60]}")
