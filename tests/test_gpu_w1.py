"""K2's one-warp CTA layout (k_accel WE = 2: the 64-thread x 5-slot CTA of a
J = 320 bin as one warp x 10 slots, no barrier in the iteration loop). It is
chosen by batch size (RCSCM_ACCEL_W1 = the fewest bins that take it), so it
must give every bit the 64 x 5 layout gives -- the same slots per emulated
thread, the same in-thread trees, the same zero-padded block tree -- or a
sharded run would differ from an unsharded one. Checked bitwise through the
session (fused precompute, with and without the fused Wiener epilogue) and
through the C ABI's pipelined run_algorithm2 (column-major parameters)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,B,I", [(3, 2, 40), (0, 2, 40), (3, 1, 7)])
@pytest.mark.parametrize("wiener", [False, True])
def test_one_warp_layout_bitwise_session(gpu, monkeypatch, cfg, B, I, wiener):
    from paper_1908_01964_b200 import synth
    import paper_1908_01964_b200._capi as C

    utts = synth.make_config(cfg, utterances=B, I=I, J=320)
    X, W, A, T, V = synth.stack(utts)
    outs = []
    for w1 in ("1", "0"):
        monkeypatch.setenv("RCSCM_ACCEL_W1", w1)
        gpu.session_load(X, W, A, T, V, 0)
        gpu.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
        st = C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL | (C.STAGE_WIENER if wiener else 0)
        gpu.session_run(st, 37)
        gpu.session_check()
        outs.append(gpu.session_fetch(want_image=wiener))
    a, b = outs
    for k in ("r_h", "r_u", "lam") + (("dry", "image") if wiener else ()):
        assert np.array_equal(a[k], b[k]), k


def test_one_warp_layout_bitwise_capi(gpu, monkeypatch):
    from paper_1908_01964_b200 import Hyperparams, SolverOptions, synth

    u = synth.make_config(3, utterances=1, I=300, J=320)[0]
    inp = gpu.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = gpu.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    res = []
    for w1 in ("1", "0"):
        monkeypatch.setenv("RCSCM_ACCEL_W1", w1)
        res.append(gpu.run_algorithm2(inp, p0, Hyperparams(), u.X, SolverOptions(iters=50)).params)
    a, b = res
    assert np.array_equal(a.r_h, b.r_h) and np.array_equal(a.r_u, b.r_u) and np.array_equal(a.lam, b.lam)
