"""K2 step time (config 1, fused) under three L2 treatments between steps: a
256 MiB write (dirty lines left in L2), the write followed by a 256 MiB read of
another buffer (L2 left holding clean, unrelated lines), and no flush."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1908_01964_b200 import GpuContext, Hyperparams, synth
import paper_1908_01964_b200._capi as C

u = synth.make_config(1, utterances=1)[0]
X, W, A, T, V = synth.stack([u])
s = torch.cuda.Stream()
ctx = GpuContext(0, stream=s.cuda_stream)
ctx.session_load(X, W, A, T, V, 0)
ctx.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
h = Hyperparams()
wbuf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
rbuf = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
acc = torch.empty(1, dtype=torch.float32, device="cuda")
stages = C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL


def step_ms(mode, n=20):
    out = []
    for _ in range(n):
        with torch.cuda.stream(s):
            if mode in ("write", "write+read"):
                wbuf.fill_(1.0)
            if mode == "write+read":
                acc.copy_(rbuf.sum().reshape(1))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ctx.session_run(stages, 100, h)
        e1.record(s)
        e1.synchronize()
        out.append(e0.elapsed_time(e1))
    out.sort()
    return out[len(out) // 2], out[0]


for _ in range(3):
    ctx.session_run(stages, 100, h)
for mode in ("write", "write+read", "none", "write", "write+read", "none"):
    med, mn = step_ms(mode)
    print(f"{mode:11s} median {med:.4f} ms  min {mn:.4f} ms")

# the bench's loop: flush + events + step, K steps enqueued back to back
for K in (10, 10, 30):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    for k in range(K):
        with torch.cuda.stream(s):
            wbuf.fill_(1.0)
        ev[k][0].record(s)
        ctx.session_run(stages, 100, h)
        ev[k][1].record(s)
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) for a, b in ev]
    print("bench loop K=%d: mean %.4f  steps %s" % (K, sum(t) / K, " ".join("%.4f" % x for x in t[:12])))

# the same after 0.3 s of GPU idle (the clock sampler's lead-in in bench.py)
import time
for K in (10, 10):
    time.sleep(0.3)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    for k in range(K):
        with torch.cuda.stream(s):
            wbuf.fill_(1.0)
        ev[k][0].record(s)
        ctx.session_run(stages, 100, h)
        ev[k][1].record(s)
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) for a, b in ev]
    print("after idle K=%d: mean %.4f  steps %s" % (K, sum(t) / K, " ".join("%.4f" % x for x in t[:12])))
