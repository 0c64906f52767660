"""Cold-L2 device copy time against size (torch copy_, after a 256 MiB write +
read flush): separates the fixed launch / ramp cost of a single stream kernel
from its bandwidth term, T(S) = a + S / BW."""
import statistics

import torch

buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
acc = torch.empty(1, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
rows = []
for mb in (17, 34, 68, 136, 272, 544, 1088, 2176):
    n = mb * 1024 * 1024 // 8  # half read, half written
    src = torch.ones(n, dtype=torch.float32, device="cuda")
    dst = torch.empty_like(src)
    ts = []
    for r in range(9):
        with torch.cuda.stream(s):
            buf.fill_(1.0)
            acc.copy_(buf.sum())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            dst.copy_(src)
            e1.record(s)
        e1.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    t = statistics.median(ts)
    rows.append((mb, t))
    print(f"{mb:6d} MB moved: {t * 1e3:8.1f} us  {mb * 1.048576e6 / (t * 1e-3) / 1e12:6.2f} TB/s")
(m1, t1), (m2, t2) = rows[-2], rows[-1]
bw = (m2 - m1) * 1.048576e6 / ((t2 - t1) * 1e-3)
a = t1 * 1e-3 - m1 * 1.048576e6 / bw
print(f"fit: bandwidth {bw / 1e12:.2f} TB/s, fixed {a * 1e6:.1f} us")
