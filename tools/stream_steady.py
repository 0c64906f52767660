"""Steady-state single-utterance K1 / K4 launches (8 contexts back to back after
one L2 flush), for tuning the stream kernels."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1908_01964_b200 import GpuContext, Hyperparams, synth
import paper_1908_01964_b200._capi as C
s = torch.cuda.Stream()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
X, W, A, T, V = synth.stack(synth.make_config(1, utterances=1))
h = Hyperparams()
ctxs = [GpuContext(0, stream=s.cuda_stream) for _ in range(8)]
for cx in ctxs:
    cx.session_load(X, W, A, T, V, 0)
    cx.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    cx.session_run(C.STAGE_ACCEL, 3, h)
S = X.shape[1] * X.shape[2]
for name, st, bps in (("k_pre", C.STAGE_PRECOMPUTE, 104.0), ("k_wiener", C.STAGE_WIENER, 128.0)):
    ts = []
    for r in range(6):
        with torch.cuda.stream(s):
            flush.fill_(float(r))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for cx in ctxs:
            cx.session_run(st, 0, h)
        e1.record(s)
        e1.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1) / 8)
    ms = statistics.median(ts)
    print(f"SPT={os.environ.get('RCSCM_STREAM_SPT', 'default')} {name}: {ms*1e3:.1f} us {bps*S/(ms*1e-3)/1e9:.0f} GB/s")
