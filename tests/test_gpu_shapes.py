"""Channel counts beyond the BASELINE configs: every M from 1 to 16 runs the
same kernels (templated per M, dispatch.cuh), like the reference's Eigen::Dynamic
path (solver_naive.hpp:248-262, 388-406); M > 16 is refused with
UnsupportedError (RCSCM_UNSUPPORTED, code 5) before any launch."""
import numpy as np
import pytest

from parity import output_rel_err

pytestmark = pytest.mark.gpu


def _hyper():
    from paper_1908_01964_b200 import Hyperparams

    return Hyperparams()


def _opts(**kw):
    from paper_1908_01964_b200 import SolverOptions

    return SolverOptions(**kw)


@pytest.mark.parametrize("M", [5, 6, 7, 9, 10, 11, 12, 13, 14, 15, 16])
def test_every_mic_count(O, gpu, M):
    inp, p, X = O.make_verify_instance(3, 24, M, 500 + M)
    for backend, fn in (("accel2", gpu.run_algorithm2), ("naive", gpu.run_naive), ("accel1", gpu.run_algorithm1)):
        g = fn(inp, p, _hyper(), X, _opts(iters=1)).params
        o = O.run(backend, inp, p, X, O.SolverOptions(iters=1)).params
        assert O.trajectory_distance(g, o) <= 1e-9, (backend, O.trajectory_distance(g, o))
    g = gpu.run_algorithm2(inp, p, _hyper(), X, _opts(iters=10)).params
    o = O.run("accel2", inp, p, X, O.SolverOptions(iters=10)).params
    ge = gpu.extract_target(inp, g, X)
    oimg, odry = O.extract_target(inp, o, X)
    assert output_rel_err(ge.dry, odry) <= 1e-6 and output_rel_err(ge.image, oimg) <= 1e-6


@pytest.mark.parametrize("M", [9, 12])
def test_setup_for_large_mic_counts(O, gpu, M):
    from conftest import random_demixing, random_spectrogram

    W, A = random_demixing(4, M, 70 + M)
    X = random_spectrogram(4, 40, M, 80 + M)
    gi = gpu.build_noise_scm(W, A, X, 0)
    oi = O.build_noise_scm(W, A, X, 0)
    for f in ("a", "b", "R_prime", "R_prime_pinv"):
        g, o = getattr(gi, f), getattr(oi, f)
        assert np.max(np.abs(g - o)) <= 1e-9 * max(1.0, np.max(np.abs(o))), f
    T = np.abs(np.random.default_rng(M).standard_normal((4, 3))) + 0.1
    V = np.abs(np.random.default_rng(M + 1).standard_normal((3, 40))) + 0.1
    gp = gpu.init_params(oi, T, V, W, A, X)
    op = O.init_params(oi, T, V, W, A, X)
    assert O.trajectory_distance(gp, op) <= 1e-9


def test_more_than_16_mics_is_unsupported(O, gpu):
    from paper_1908_01964_b200 import RcscmInputs, RcscmParams
    from paper_1908_01964_b200.api import UnsupportedError

    M = 17
    inp = RcscmInputs(np.ones((2, M), complex), np.zeros((2, M, M), complex), np.zeros((2, M, M), complex),
                      np.ones((2, M), complex), 0)
    p = RcscmParams(np.ones((2, 4)), np.ones((2, 4)), np.ones(2))
    with pytest.raises(UnsupportedError, match="mics = 17"):
        gpu.run_algorithm2(inp, p, _hyper(), np.ones((2, 4, M), complex), _opts(iters=1))
    with pytest.raises(UnsupportedError, match="mics = 17"):
        gpu.run_naive(inp, p, _hyper(), np.ones((2, 4, M), complex), _opts(iters=1))
