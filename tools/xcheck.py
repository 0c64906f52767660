"""Cluster-exchange protocol check (stands in for compute-sanitizer racecheck /
synccheck, which are closed on the GPU pool). Runs Algorithm 2 on every
cluster size (2..16 CTAs, st.async + mbarrier exchange) and the fused session
step, 20 times each, with the library given in RCSCM_GPU_LIB (the
-DRCSCM_K2_XCHECK build poisons each exchange buffer with NaN after it is read,
so an early or missing partial corrupts the result), and writes the outputs;
compare two runs' outputs with --compare a.npz b.npz (bitwise)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k], equal_nan=False)]
    nans = [k for k in a.files if np.isnan(a[k]).any() or np.isnan(b[k]).any()]
    print(f"compared {len(a.files)} arrays: {len(bad)} differ {bad[:5]}, {len(nans)} with NaN {nans[:5]}")
    sys.exit(1 if bad or nans else 0)

from oracle import oracle as O  # noqa: E402  (inputs only)
from paper_1908_01964_b200 import GpuContext, Hyperparams, SolverOptions, synth  # noqa: E402
import paper_1908_01964_b200._capi as C  # noqa: E402

out = {}
gpu = GpuContext(0)
h = Hyperparams()
for cl in (2, 3, 4, 5, 6, 8, 10, 12, 16):
    os.environ["RCSCM_ACCEL_CL"] = str(cl)
    inp, p, X = O.make_verify_instance(7, 1024 * cl, 2, 40 + cl)
    for r in range(20):
        res = gpu.run_algorithm2(inp, p, h, X, SolverOptions(iters=30)).params
        out[f"cl{cl}_r{r}_lam"] = res.lam
        out[f"cl{cl}_r{r}_ru"] = res.r_u
        assert np.array_equal(res.lam, out[f"cl{cl}_r0_lam"]), (cl, r)
    del os.environ["RCSCM_ACCEL_CL"]
for cfg, J in ((4, 4096), (2, 20000)):
    X, W, A, T, V = synth.stack(synth.make_config(cfg, utterances=1, I=40, J=J))
    gpu.session_load(X, W, A, T, V, 0)
    gpu.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    for r in range(5):
        gpu.session_run(C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL | C.STAGE_WIENER, 50)
        f = gpu.session_fetch()
        out[f"s{cfg}_r{r}_lam"] = f["lam"]
        out[f"s{cfg}_r{r}_dry"] = f["dry"]
gpu.session_check()
np.savez(sys.argv[1], **out)
print("xcheck run ok:", len(out), "arrays; repeated runs bitwise equal")
