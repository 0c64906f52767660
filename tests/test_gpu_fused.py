"""K2 with the Wiener output fused into its epilogue (session ACCEL + WIENER in
one call): one launch computes the solve and extract_target's dry / image
(wiener.hpp:29-41) from registers. Checked against the unfused pair K2 + K4
(RCSCM_FUSE_WIENER=0) -- same formulas, rho_ax carried in K2 versus recomputed
from sigma / tau in K4, so equal to rounding -- and against the oracle's
extract_target after the same number of iterations, on single-CTA bins and on
cluster shapes (J = 4096: 2-CTA clusters; J = 20000: 16-CTA clusters)."""
import numpy as np
import pytest

from parity import output_rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,B,I,J,iters", [(3, 3, 40, 320, 100), (1, 1, 24, 640, 100), (0, 2, 16, 320, 60),
                                             (4, 1, 6, 4096, 100), (2, 1, 2, 20000, 50)])
def test_fused_wiener_epilogue(O, gpu, monkeypatch, cfg, B, I, J, iters):
    from paper_1908_01964_b200 import synth
    import paper_1908_01964_b200._capi as C

    utts = synth.make_config(cfg, utterances=B, I=I, J=J)
    X, W, A, T, V = synth.stack(utts)
    outs = []
    for fuse in ("1", "0"):
        monkeypatch.setenv("RCSCM_FUSE_WIENER", fuse)
        gpu.session_load(X, W, A, T, V, 0)
        gpu.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
        n0 = gpu.launch_count
        gpu.session_run(C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL | C.STAGE_WIENER, iters)
        launches = gpu.launch_count - n0
        gpu.session_check()
        outs.append((gpu.session_fetch(want_image=True), launches))
    (f, nf), (u, nu) = outs
    assert nf == 1 and nu == 2, (nf, nu)
    for k in ("r_h", "r_u", "lam"):
        assert np.array_equal(f[k], u[k]), k
    assert output_rel_err(f["dry"], u["dry"]) <= 1e-11
    assert output_rel_err(f["image"], u["image"]) <= 1e-11
    for k, ut in enumerate(utts):
        inp = O.build_noise_scm(ut.W, ut.A, ut.X, 0)
        p0 = O.init_params(inp, ut.T, ut.V, ut.W, ut.A, ut.X)
        o = O.run("accel2_binparallel", inp, p0, ut.X, O.SolverOptions(iters=iters, threads=8)).params
        oimg, odry = O.extract_target(inp, o, ut.X)
        assert output_rel_err(f["dry"][k], odry) <= 1e-6
        assert output_rel_err(f["image"][k], oimg) <= 1e-6
