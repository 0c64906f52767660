"""Bins longer than the on-chip kernel holds (J > 32768 frames): Algorithm 2
streams the iterate through HBM (accel_stream.cuh, two launches per
iteration). The reference's loop takes any J (solver_accel.hpp:143-158).
Checked at J = 40000 on the BASELINE recipe (config-2 style, M = 2): one
iteration against the binary128 truth (the same bars as tests/test_gpu_truth.py),
the Wiener output after 50 iterations against the oracle (<= 1e-6),
trajectories and the objective through the C ABI, bitwise determinism and
bitwise invariance to how bins are split."""
import numpy as np
import pytest

from parity import output_rel_err
from truth_cases import C_ACCEL, bound_units, field_errors

pytestmark = pytest.mark.gpu


def _hyper():
    from paper_1908_01964_b200 import Hyperparams

    return Hyperparams()


def _opts(**kw):
    from paper_1908_01964_b200 import SolverOptions

    return SolverOptions(**kw)


@pytest.fixture(scope="module")
def long_case(O):
    from paper_1908_01964_b200 import synth

    u = synth.make_config(2, utterances=1, I=3, J=40000)[0]
    inp = O.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    return u, inp, p0


def test_long_bins_one_iteration_vs_truth(O, gpu, long_case):
    u, inp, p0 = long_case
    tr, B = O.truth_accel_one_iter(inp, p0, u.X)
    g = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=1)).params
    eg = field_errors(g, tr)
    assert eg["r_h"].max() <= 1e-9 and eg["lambda"].max() <= 1e-9
    ug = bound_units(g, tr, B)
    assert ((eg["r_u"] <= 1e-9) | (ug["r_u"] <= C_ACCEL)).all()


def test_long_bins_output_full_iterations(O, gpu, long_case):
    u, inp, p0 = long_case
    g = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=50)).params
    o = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=50)).params
    lam_rel = np.abs(g.lam - o.lam) / np.abs(o.lam)
    assert lam_rel.max() <= 1e-8, lam_rel.max()
    ge = gpu.extract_target(inp, g, u.X)
    oimg, odry = O.extract_target(inp, o, u.X)
    assert output_rel_err(ge.dry, odry) <= 1e-6
    assert output_rel_err(ge.image, oimg) <= 1e-6


def test_long_bins_trajectory_objective_determinism(O, gpu, long_case):
    from paper_1908_01964_b200 import RcscmInputs, RcscmParams

    u, inp, p0 = long_case
    res = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=4, record_trajectory=True, compute_objective=True))
    oo = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=4, compute_objective=True, record_trajectory=True))
    assert len(res.trajectory) == 4 and len(res.objective) == 5
    assert np.allclose(res.objective, oo.objective, rtol=1e-9, atol=0)
    for k in range(4):
        assert O.trajectory_distance(res.trajectory[k], oo.trajectory[k]) < 1e-8
    a = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=6)).params
    b = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=6)).params
    assert np.array_equal(a.r_u, b.r_u) and np.array_equal(a.lam, b.lam)
    parts = []
    for sl in (slice(0, 1), slice(1, 3)):
        pi = RcscmInputs(inp.a[sl], inp.R_prime[sl], inp.R_prime_pinv[sl], inp.b[sl], 0)
        parts.append(gpu.run_algorithm2(pi, RcscmParams(p0.r_h[sl], p0.r_u[sl], p0.lam[sl]), _hyper(), u.X[sl],
                                        _opts(iters=6)).params)
    assert np.array_equal(np.concatenate([q.r_u for q in parts]), a.r_u)
    assert np.array_equal(np.concatenate([q.lam for q in parts]), a.lam)


def test_long_bins_session(O, gpu):
    """The device session runs the streaming kernel too (PRECOMPUTE + ACCEL +
    WIENER on a 40000-frame batch of two utterances)."""
    from paper_1908_01964_b200 import synth
    import paper_1908_01964_b200._capi as C

    utts = synth.make_config(2, utterances=2, I=2, J=40000)
    X, W, A, T, V = synth.stack(utts)
    gpu.session_load(X, W, A, T, V, 0)
    gpu.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    gpu.session_run(C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL | C.STAGE_WIENER, 20)
    gpu.session_check()
    out = gpu.session_fetch()
    for k, u in enumerate(utts):
        inp = O.build_noise_scm(u.W, u.A, u.X, 0)
        p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
        o = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=20)).params
        _, odry = O.extract_target(inp, o, u.X)
        assert output_rel_err(out["dry"][k], odry) <= 1e-6
