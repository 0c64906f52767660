"""HBM bandwidth of the slot-stream kernels (K1 precompute, K4 Wiener): each
launch timed alone with CUDA events after an L2 flush (cold L2), median of
--reps; B utterances of config --cfg resident through the session API."""
import argparse, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1908_01964_b200 import GpuContext, Hyperparams, synth
import paper_1908_01964_b200._capi as C

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=1)
ap.add_argument("--B", type=int, nargs="+", default=[1, 4])
ap.add_argument("--reps", type=int, default=7)
a = ap.parse_args()
BYTES_PRE = {2: 72.0, 4: 104.0, 8: 168.0}
BYTES_WIENER = {2: 96.0, 4: 128.0, 8: 192.0}
s = torch.cuda.Stream()
flush_buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
h = Hyperparams()
for B in a.B:
    X, W, A, T, V = synth.stack(synth.make_config(a.cfg, utterances=B))
    ctx = GpuContext(0, stream=s.cuda_stream)
    ctx.session_load(X, W, A, T, V, 0)
    ctx.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    ctx.session_run(C.STAGE_ACCEL, 5, h)
    _, I, J, M = X.shape
    S = B * I * J
    for name, st, bps in (("k_pre", C.STAGE_PRECOMPUTE, BYTES_PRE[M]), ("k_wiener", C.STAGE_WIENER, BYTES_WIENER[M])):
        ts = []
        for r in range(a.reps + 1):
            with torch.cuda.stream(s):
                flush_buf.fill_(float(r))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ctx.session_run(st, 0, h)
            e1.record(s)
            e1.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(f"cfg{a.cfg} B={B} M={M} I={I} J={J} {name}: {ms*1e3:.1f} us  {bps*S/(ms*1e-3)/1e9:.0f} GB/s "
              f"({bps*S/1e6:.1f} MB)", flush=True)
    ctx.session_check()
    ctx.close()
