"""GPU parity at the BASELINE configs' real shapes and full iteration counts.

* C3 through the device-resident session path the bench times: 8 utterances at
  the real shape (M = 4, I = 513, J = 320; seeds 3000..3007, the bench's first
  eight), 100 iterations of Algorithm 2 and the Wiener output, against the
  oracle per utterance: <= 1e-6 on dry and image, and r_h, r_u,
  lambda reported after 100 iterations.
* The naive rule after its full iteration count (100 on C0 / C1 subsets, 10 on
  a C4 subset) -- run_naive then extract_target on both sides, <= 1e-6 on the
  output (the reference pins long naive runs in test_solver_naive.cpp:170-193,
  acceptance.cpp:34-65).
* Non-finite inputs propagate like the reference's std::max floors
  (solver_accel.hpp:57,61,156,173): a NaN in x gives NaN in the same outputs as
  the oracle, and every finite output agrees with it.
"""
import numpy as np
import pytest

from parity import output_rel_err, rel_err

pytestmark = pytest.mark.gpu


def _hyper():
    from paper_1908_01964_b200 import Hyperparams

    return Hyperparams()


def _opts(**kw):
    from paper_1908_01964_b200 import SolverOptions

    return SolverOptions(**kw)


def test_c3_session_real_shape_full_iterations(O, gpu):
    from paper_1908_01964_b200 import synth
    import paper_1908_01964_b200._capi as C

    B = 8
    utts = synth.make_config(3, utterances=B)
    X, W, A, T, V = synth.stack(utts)
    assert X.shape == (B, 513, 320, 4)
    gpu.session_load(X, W, A, T, V, 0)
    gpu.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    # the bench step (params0 restored, precompute fused into K2), then the output
    gpu.session_run(C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL | C.STAGE_WIENER, 100)
    gpu.session_check()
    out = gpu.session_fetch(want_image=True)
    worst = {"dry": 0.0, "image": 0.0, "r_h": 0.0, "r_u": 0.0, "lambda": 0.0}
    for k, u in enumerate(utts):
        inp = O.build_noise_scm(u.W, u.A, u.X, 0)
        p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
        o = O.run("accel2_binparallel", inp, p0, u.X, O.SolverOptions(iters=100, threads=8)).params
        oimg, odry = O.extract_target(inp, o, u.X)
        worst["dry"] = max(worst["dry"], output_rel_err(out["dry"][k], odry))
        worst["image"] = max(worst["image"], output_rel_err(out["image"][k], oimg))
        worst["r_h"] = max(worst["r_h"], float(rel_err(out["r_h"][k], o.r_h).max()))
        worst["r_u"] = max(worst["r_u"], float(rel_err(out["r_u"][k], o.r_u).max()))
        worst["lambda"] = max(worst["lambda"], float(rel_err(out["lam"][k], o.lam).max()))
    print("\nC3 x8 after 100 iterations:", {k: f"{v:.2e}" for k, v in worst.items()})
    assert worst["dry"] <= 1e-6 and worst["image"] <= 1e-6, worst


@pytest.mark.parametrize("cfg,I,J,iters", [(0, 64, 320, 100), (1, 32, 640, 100), (3, 64, 320, 100),
                                           (4, 4, 4096, 10)])
def test_naive_output_full_iterations(O, gpu, cfg, I, J, iters):
    from paper_1908_01964_b200 import synth

    u = synth.make_config(cfg, utterances=1, I=I, J=J)[0]
    inp = O.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    g = gpu.run_naive(inp, p0, _hyper(), u.X, _opts(iters=iters)).params
    o = O.run("naive", inp, p0, u.X, O.SolverOptions(iters=iters, threads=8)).params
    ge = gpu.extract_target(inp, g, u.X)
    oimg, odry = O.extract_target(inp, o, u.X)
    e = (output_rel_err(ge.dry, odry), output_rel_err(ge.image, oimg))
    print(f"\nnaive c{cfg} {iters} it: dry {e[0]:.2e} image {e[1]:.2e} lambda {rel_err(g.lam, o.lam).max():.2e}")
    assert max(e) <= 1e-6, e


def test_nan_in_x_propagates_like_the_reference(O, gpu):
    """Algorithm 2: the NaN reaches the same outputs as in the oracle (std::max
    floors keep it) and every finite output agrees."""
    inp, p, X = O.make_verify_instance(4, 24, 2, 31)
    X = X.copy()
    X[1, 5, 0] = np.nan
    g = gpu.run_algorithm2(inp, p, _hyper(), X, _opts(iters=1)).params
    o = O.run("accel2", inp, p, X, O.SolverOptions(iters=1)).params
    assert np.isnan(o.lam[1])  # the NaN reaches bin 1's lambda
    for f in ("r_h", "r_u", "lam"):
        gv, ov = np.asarray(getattr(g, f)), np.asarray(getattr(o, f))
        assert np.array_equal(np.isnan(gv), np.isnan(ov)), f
        fin = ~np.isnan(ov)
        assert rel_err(gv[fin], ov[fin]).max() <= 1e-9, f


def test_nan_in_x_naive_raises_like_the_reference(O, gpu):
    """The naive rule: bin 1's lambda becomes NaN, so R_u = R' + lambda b b^H is
    not PD and the M-step raises NumericalError at bin 1 (solver_naive.hpp:363-367)
    on both sides."""
    from paper_1908_01964_b200 import NumericalError

    inp, p, X = O.make_verify_instance(4, 24, 2, 31)
    X = X.copy()
    X[1, 5, 0] = np.nan
    with pytest.raises(O.NumericalError, match=r"m_step: singular R\^\(u\) at bin 1"):
        O.run("naive", inp, p, X, O.SolverOptions(iters=1))
    with pytest.raises(NumericalError, match=r"m_step: singular R\^\(u\) at bin 1"):
        gpu.run_naive(inp, p, _hyper(), X, _opts(iters=1))
