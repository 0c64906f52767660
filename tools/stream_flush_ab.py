"""K1 (k_pre) and K4 (k_wiener) on the C1 utterance, one launch after an L2
flush, for three flush methods: a 256 MiB write (leaves ~126 MB of DIRTY lines
in L2 that the next kernel's misses must write back), the write followed by a
256 MiB read (L2 ends full of clean lines), and a read only. Also a torch device
copy of the same bytes, timed the same way."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_01964_b200 import GpuContext, Hyperparams, synth  # noqa: E402
import paper_1908_01964_b200._capi as C  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
X, W, A, T, V = synth.stack(synth.make_config(cfg, utterances=1))
s = torch.cuda.Stream()
ctx = GpuContext(0, stream=s.cuda_stream)
ctx.session_load(X, W, A, T, V, 0)
ctx.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
ctx.session_run(C.STAGE_ACCEL, 5, Hyperparams())
buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
acc = torch.empty(1, dtype=torch.float32, device="cuda")


def flush(kind):
    with torch.cuda.stream(s):
        if kind in ("write", "write+read"):
            buf.fill_(1.0)
        if kind in ("write+read", "read"):
            acc.copy_(buf.sum())


def timed(fn, kind, reps=9):
    ts = []
    for r in range(reps + 1):
        flush(kind)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        e1.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


B, I, J, M = X.shape
S = B * I * J
bpre = {2: 72, 4: 104, 8: 168}[M]
bwie = {2: 96, 4: 128, 8: 192}[M]
src = torch.ones(bpre * S // 8, dtype=torch.float32, device="cuda")
dst = torch.empty_like(src)


def copy():
    with torch.cuda.stream(s):
        dst.copy_(src)


for kind in ("write", "write+read", "read"):
    tp = timed(lambda: ctx.session_run(C.STAGE_PRECOMPUTE, 0, Hyperparams()), kind)
    tw = timed(lambda: ctx.session_run(C.STAGE_WIENER, 0, Hyperparams()), kind)
    tc = timed(copy, kind)
    print(f"cfg{cfg} flush={kind:10s} k_pre {tp * 1e3:6.1f} us {bpre * S / tp / 1e6:7.0f} GB/s | "
          f"k_wiener {tw * 1e3:6.1f} us {bwie * S / tw / 1e6:7.0f} GB/s | copy(k_pre bytes) {tc * 1e3:6.1f} us "
          f"{bpre * S / tc / 1e6:7.0f} GB/s")
