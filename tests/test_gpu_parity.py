"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Instances: the reference's own seeded instances (make_verify_instance, the
generator of proj/tests/ and `rcscm verify`) and the BASELINE synthetic recipe
(paper_1908_01964_b200.synth) at sizes the oracle finishes in seconds, plus the
full C1 configuration. Bars (tests/parity.py): <= 1e-9 elementwise relative on
r_h, r_u, lambda after one iteration (r_u condition-aware on the synthetic
recipe), trajectories <= 1e-8 over 50 iterations (acceptance.cpp:34-65), and
<= 1e-6 on the Wiener output after the full iteration count.
"""
import numpy as np
import pytest

from parity import check_params, naive_condition, output_rel_err, ru_condition_scale

pytestmark = pytest.mark.gpu


def _hyper():
    from paper_1908_01964_b200 import Hyperparams

    return Hyperparams()


def _opts(**kw):
    from paper_1908_01964_b200 import SolverOptions

    return SolverOptions(**kw)


def _synthetic(O, cfg, I, J):
    from paper_1908_01964_b200 import synth

    u = synth.make_config(cfg, utterances=1, I=I, J=J)[0]
    inp = O.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    return u, inp, p0


# ---- the reference's own instances -------------------------------------------------
@pytest.mark.parametrize("I,J,M", [(8, 16, 2), (8, 16, 3), (8, 128, 4), (64, 16, 8), (64, 128, 2), (8, 16, 1)])
def test_verify_instances_one_iteration(O, gpu, I, J, M):
    inp, p, X = O.make_verify_instance(I, J, M, 1000 * I + 10 * J + M)
    for backend, fn in (("accel2", gpu.run_algorithm2), ("naive", gpu.run_naive), ("accel1", gpu.run_algorithm1)):
        g = fn(inp, p, _hyper(), X, _opts(iters=1)).params
        o = O.run(backend, inp, p, X, O.SolverOptions(iters=1)).params
        r = check_params(g, o)
        assert r["ok"], (backend, r)


@pytest.mark.parametrize("I,J,M", [(8, 16, 2), (8, 16, 4), (8, 128, 3), (64, 16, 8)])
def test_verify_grid_trajectories(O, gpu, I, J, M):
    """cmd_verify / acceptance criterion 1: naive == accel trajectories <= 1e-8,
    here GPU-naive vs GPU-accel vs oracle-naive over 50 iterations."""
    inp, p, X = O.make_verify_instance(I, J, M, 7000 + M)
    opt = _opts(iters=50, record_trajectory=True)
    ga = gpu.run_algorithm2(inp, p, _hyper(), X, opt)
    gn = gpu.run_naive(inp, p, _hyper(), X, opt)
    g1 = gpu.run_algorithm1(inp, p, _hyper(), X, opt)
    on = O.run("naive", inp, p, X, O.SolverOptions(iters=50, record_trajectory=True))
    assert len(ga.trajectory) == len(gn.trajectory) == len(g1.trajectory) == 50
    worst = 0.0
    for k in range(50):
        worst = max(worst, O.trajectory_distance(ga.trajectory[k], on.trajectory[k]),
                    O.trajectory_distance(gn.trajectory[k], on.trajectory[k]),
                    O.trajectory_distance(g1.trajectory[k], on.trajectory[k]),
                    O.trajectory_distance(ga.trajectory[k], gn.trajectory[k]))
    assert worst <= 1e-8, worst


# ---- BASELINE synthetic recipe ------------------------------------------------------
SYNTH = [(0, 64, 320), (1, 64, 640), (2, 6, 20000), (3, 32, 320), (4, 12, 4096), (1, 5, 17)]


@pytest.mark.parametrize("cfg,I,J", SYNTH)
def test_synthetic_setup_parity(O, gpu, cfg, I, J):
    from paper_1908_01964_b200 import synth

    u = synth.make_config(cfg, utterances=1, I=I, J=J)[0]
    gi = gpu.build_noise_scm(u.W, u.A, u.X, 0)
    oi = O.build_noise_scm(u.W, u.A, u.X, 0)
    for f in ("a", "b", "R_prime", "R_prime_pinv"):
        g, o = getattr(gi, f), getattr(oi, f)
        assert np.max(np.abs(g - o)) <= 1e-9 * max(1.0, np.max(np.abs(o))), f
    gp = gpu.init_params(oi, u.T, u.V, u.W, u.A, u.X)
    op = O.init_params(oi, u.T, u.V, u.W, u.A, u.X)
    assert check_params(gp, op)["ok"]


@pytest.mark.parametrize("cfg,I,J", SYNTH)
def test_synthetic_one_iteration(O, gpu, cfg, I, J):
    u, inp, p0 = _synthetic(O, cfg, I, J)
    S = ru_condition_scale(O, inp, p0, u.X)
    g = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=1)).params
    o = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=1)).params
    r = check_params(g, o, S)
    assert r["ok"], ("accel2", r)
    if J <= 5000:
        kappa, S_h = naive_condition(inp, p0, u.X)
        g = gpu.run_naive(inp, p0, _hyper(), u.X, _opts(iters=1)).params
        o = O.run("naive", inp, p0, u.X, O.SolverOptions(iters=1)).params
        r = check_params(g, o, S, kappa=kappa, S_h=S_h)
        assert r["ok"], ("naive", r)


@pytest.mark.parametrize("cfg,I,J,iters", [(0, 64, 320, 100), (1, 32, 640, 100), (2, 4, 20000, 50), (4, 8, 4096, 100)])
def test_synthetic_output_full_iterations(O, gpu, cfg, I, J, iters):
    """<= 1e-6 on the extracted target STFT after the full iteration count."""
    u, inp, p0 = _synthetic(O, cfg, I, J)
    g = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=iters)).params
    o = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=iters)).params
    ge = gpu.extract_target(inp, g, u.X)
    oimg, odry = O.extract_target(inp, o, u.X)
    assert output_rel_err(ge.dry, odry) <= 1e-6
    assert output_rel_err(ge.image, oimg) <= 1e-6


def test_full_c1_one_iteration_and_output(O, gpu):
    """Full BASELINE config 1 (M=4, I=1025, J=640): GPU vs oracle."""
    from paper_1908_01964_b200 import synth

    u = synth.make_config(1, utterances=1)[0]
    inp = O.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    S = ru_condition_scale(O, inp, p0, u.X)
    g = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=1)).params
    o = O.run("accel2_binparallel", inp, p0, u.X, O.SolverOptions(iters=1, threads=8)).params
    r = check_params(g, o, S)
    assert r["ok"], r
    g = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=100)).params
    o = O.run("accel2_binparallel", inp, p0, u.X, O.SolverOptions(iters=100, threads=8)).params
    assert output_rel_err(gpu.extract_target(inp, g, u.X).dry, O.extract_target(inp, o, u.X)[1]) <= 1e-6


# ---- known answers of the reference's tests, on the GPU path --------------------------
def _scalar_problem():
    from paper_1908_01964_b200 import RcscmInputs, RcscmParams

    inp = RcscmInputs(np.ones((1, 1), complex), np.zeros((1, 1, 1), complex), np.zeros((1, 1, 1), complex),
                      np.ones((1, 1), complex), 0)
    p = RcscmParams(np.ones((1, 1)), np.ones((1, 1)), np.array([2.0]))
    return inp, p, np.full((1, 1, 1), 3.0 + 0j)


def test_naive_scalar_known_answer(gpu):
    """test_solver_naive.cpp:44-58: r^ = 5/3, so r_h = (5/3 + beta)/(alpha + 2)."""
    inp, p, X = _scalar_problem()
    r = gpu.run_naive(inp, p, _hyper(), X, _opts(iters=1)).params
    assert r.r_h[0, 0] == pytest.approx((5 / 3 + 1e-16) / 3.1, rel=1e-12)


def test_iters_zero_passthrough(O, gpu):  # test_solver_accel.cpp:289-298, test_solver_naive.cpp:147-156
    inp, p, X = O.make_verify_instance(2, 4, 3, 12)
    for fn in (gpu.run_algorithm2, gpu.run_naive, gpu.run_algorithm1):
        r = fn(inp, p, _hyper(), X, _opts(iters=0)).params
        assert np.array_equal(r.r_h, p.r_h) and np.array_equal(r.r_u, p.r_u) and np.array_equal(r.lam, p.lam)


# ---- Algorithm 1 (first-stage acceleration, K6) -------------------------------------
@pytest.mark.parametrize("cfg,I,J", [(0, 16, 320), (1, 8, 640), (4, 4, 1024), (1, 5, 17)])
def test_algorithm1_synthetic(O, gpu, cfg, I, J):
    """run_algorithm1 vs the oracle's Algorithm 1: one iteration (r_u
    condition-aware as for Algorithm 2), and 30-iteration trajectories against
    GPU Algorithm 2 within the reference's cross-backend bar."""
    u, inp, p0 = _synthetic(O, cfg, I, J)
    S = ru_condition_scale(O, inp, p0, u.X)
    g = gpu.run_algorithm1(inp, p0, _hyper(), u.X, _opts(iters=1)).params
    o = O.run("accel1", inp, p0, u.X, O.SolverOptions(iters=1)).params
    r = check_params(g, o, S)
    assert r["ok"], r
    g1 = gpu.run_algorithm1(inp, p0, _hyper(), u.X, _opts(iters=30)).params
    o1 = O.run("accel1", inp, p0, u.X, O.SolverOptions(iters=30)).params
    assert output_rel_err(gpu.extract_target(inp, g1, u.X).dry, O.extract_target(inp, o1, u.X)[1]) <= 1e-6


def test_algorithm1_scalar_rho_first_stage(gpu):
    """test_solver_accel.cpp:112-128: R' = 0, a = b = 1, lambda = 2, x = 0 ->
    rho_aa = 1/2, rho_ax = rho_xx = 0; one iteration from r_h = r_u = 1 then
    gives gamma = 1/(1 + 1/2), r_h = (gamma + beta)/(alpha + 2), lambda = gamma
    (|s_ab|^2 = 1, s_bx = 0) and r_u = max(gamma rho_aa(lambda) / 1, eps)."""
    from paper_1908_01964_b200 import RcscmInputs, RcscmParams

    inp = RcscmInputs(np.ones((1, 1), complex), np.zeros((1, 1, 1), complex), np.zeros((1, 1, 1), complex),
                      np.ones((1, 1), complex), 0)
    p = RcscmParams(np.ones((1, 3)), np.ones((1, 3)), np.array([2.0]))
    r = gpu.run_algorithm1(inp, p, _hyper(), np.zeros((1, 3, 1), complex), _opts(iters=1)).params
    g = 1.0 / 1.5
    assert r.r_h[0, 0] == pytest.approx((g * (1 + g * 0) + 1e-16) / 3.1, rel=1e-13)
    assert r.lam[0] == pytest.approx(g, rel=1e-13)
    assert r.r_u[0, 0] == pytest.approx(g * (1.0 / g) * 1.0, rel=1e-13)


def test_algorithm1_objective_monotone_and_threads(O, gpu):
    """test_solver_accel.cpp:320-332 (monotone objective over 100 iterations) and
    :351-368 (results independent of the threads option), for Algorithm 1."""
    inp, p, X = O.make_verify_instance(4, 12, 3, 14)
    res = gpu.run_algorithm1(inp, p, _hyper(), X, _opts(iters=100, compute_objective=True))
    obj = np.asarray(res.objective)
    assert len(obj) == 101
    assert np.all(obj[1:] >= obj[:-1] - 1e-7 * np.abs(obj[:-1]))
    oo = O.run("accel1", inp, p, X, O.SolverOptions(iters=100, compute_objective=True))
    assert np.allclose(obj, oo.objective, rtol=1e-9, atol=0)
    inp, p, X = O.make_verify_instance(7, 10, 3, 16)
    a = gpu.run_algorithm1(inp, p, _hyper(), X, _opts(iters=25)).params
    b = gpu.run_algorithm1(inp, p, _hyper(), X, _opts(iters=25, threads=4)).params
    assert np.array_equal(a.r_h, b.r_h) and np.array_equal(a.r_u, b.r_u) and np.array_equal(a.lam, b.lam)


def test_algorithm1_errors(O, gpu):
    """solver_accel.hpp:90-97: a nonpositive lambda / singular R^(u) raise
    NumericalError naming the bin."""
    from paper_1908_01964_b200 import NumericalError, RcscmParams

    inp, p, X = O.make_verify_instance(3, 4, 2, 21)
    lam = p.lam.copy()
    lam[1] = -1.0
    with pytest.raises(NumericalError, match="rho_first_stage: nonpositive lambda at bin 1"):
        gpu.run_algorithm1(inp, RcscmParams(p.r_h, p.r_u, lam), _hyper(), X, _opts(iters=1))
    Rp = inp.R_prime.copy()
    Rp[2] = -np.eye(2)
    import dataclasses

    with pytest.raises(NumericalError, match="rho_first_stage: singular R\\^\\(u\\) at bin 2"):
        gpu.run_algorithm1(dataclasses.replace(inp, R_prime=Rp), p, _hyper(), X, _opts(iters=1))


@pytest.mark.parametrize("J", [16, 640])
def test_sigma_ab_zero_bins(O, gpu, J):
    """Bins whose b is orthogonal to a (sigma_ab = a^H b = 0) take K2's literal
    lambda form (no |sigma_ab|^2 scaling); mixed with ordinary bins in one launch."""
    import dataclasses

    inp, p, X = O.make_verify_instance(6, J, 3, 4242 + J)
    b = inp.b.copy()
    for i in (1, 4):
        a = inp.a[i]
        v = b[i] - a * (np.vdot(a, b[i]) / np.vdot(a, a))  # remove the a component
        b[i] = v / np.linalg.norm(v)
    inp = dataclasses.replace(inp, b=b)
    assert abs(np.vdot(inp.a[1], inp.b[1])) < 1e-15 and abs(np.vdot(inp.a[0], inp.b[0])) > 1e-3
    for iters in (1, 20):
        g = gpu.run_algorithm2(inp, p, _hyper(), X, _opts(iters=iters)).params
        o = O.run("accel2", inp, p, X, O.SolverOptions(iters=iters)).params
        if iters == 1:
            r = check_params(g, o)
            assert r["ok"], r
        else:
            assert O.trajectory_distance(g, o) <= 1e-8


def test_rh_zero_collapse(O, gpu):  # test_solver_naive.cpp:60-65 / test_wiener.cpp:9-15
    inp, p, X = O.make_verify_instance(2, 6, 3, 1)
    p.r_h[:] = 0
    r = gpu.run_naive(inp, p, _hyper(), X, _opts(iters=1)).params
    assert np.all(r.r_h == max(1e-16 / 3.1, 1e-12))
    e = gpu.extract_target(inp, p, X)
    assert np.max(np.abs(e.dry)) == 0.0 and np.max(np.abs(e.image)) == 0.0


def test_wiener_dense_and_complement(O, gpu):  # test_wiener.cpp:31-62
    inp, p, X = O.make_verify_instance(4, 10, 4, 3)
    e = gpu.extract_target(inp, p, X)
    for i in range(4):
        a = inp.a[i]
        Ru = inp.R_prime[i] + p.lam[i] * np.outer(inp.b[i], inp.b[i].conj())
        for t in range(10):
            rh = p.r_h[i, t]
            s = rh * (a.conj() @ np.linalg.solve(rh * np.outer(a, a.conj()) + p.r_u[i, t] * Ru, X[i, t]))
            assert abs(e.dry[i, t] - s) < 1e-9 * max(1, abs(s))
            assert np.linalg.norm(e.image[i, t] - e.dry[i, t] * a) < 1e-12
    noise = gpu.extract_noise(inp, p, X)
    assert np.max(np.abs(X - e.image - noise)) == 0.0  # bitwise complement
    oimg, odry = O.extract_target(inp, p, X)
    assert output_rel_err(e.dry, odry) < 1e-12


def test_wiener_noiseless_limit(O, gpu):  # test_wiener.cpp:17-29
    inp, p, X = O.make_verify_instance(2, 4, 3, 2)
    c = 1.5 - 0.8j
    X = c * np.repeat(inp.a[:, None, :], 4, axis=1)
    p.r_u[:] = 1e-14
    p.r_h[:] = 1.0
    assert np.max(np.abs(gpu.extract_target(inp, p, X).dry - c)) < 1e-6


def test_gamma_fault_detected(O, gpu):  # test_solver_accel.cpp:334-349
    inp, p, X = O.make_verify_instance(3, 8, 3, 15)
    naive = gpu.run_naive(inp, p, _hyper(), X, _opts(iters=10, record_trajectory=True))
    bad = gpu.run_algorithm2(inp, p, _hyper(), X, _opts(iters=10, record_trajectory=True, gamma_fault=1e-3))
    assert max(O.trajectory_distance(a, b) for a, b in zip(naive.trajectory, bad.trajectory)) > 1e-8


def test_objective_and_monotone(O, gpu):  # test_solver_accel.cpp:320-332, test_solver_naive.cpp:170-181
    inp, p, X = O.make_verify_instance(4, 12, 3, 14)
    assert gpu.map_objective(inp, p, _hyper(), X) == pytest.approx(O.map_objective(inp, p, X), rel=1e-12)
    for fn in (gpu.run_algorithm2, gpu.run_naive):
        obj = fn(inp, p, _hyper(), X, _opts(iters=100, compute_objective=True)).objective
        assert len(obj) == 101
        for k in range(1, 101):
            assert obj[k] >= obj[k - 1] - 1e-7 * abs(obj[k - 1])


@pytest.mark.parametrize("cfg,I,J,iters", [(0, 16, 320, 100), (1, 8, 640, 60), (4, 3, 4096, 30), (2, 2, 20000, 20)])
def test_objective_in_kernel(O, gpu, cfg, I, J, iters):
    """compute_objective without an early stop evaluates the objective inside
    K2 after every iteration (per-CTA partials; J = 4096 / 20000 run as
    clusters): equal to the oracle's per-iteration map_objective within 1e-9,
    to the per-iteration launch path (rel_obj_tol > 0 that never fires) within
    1e-12, and the parameters and trajectory bitwise equal to a run without
    the objective."""
    u, inp, p0 = _synthetic(O, cfg, I, J)
    res = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=iters, compute_objective=True, record_trajectory=True))
    oo = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=iters, compute_objective=True))
    assert len(res.objective) == iters + 1 and len(res.iter_seconds) == iters
    assert np.allclose(res.objective, oo.objective, rtol=1e-9, atol=0)
    step = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=iters, compute_objective=True, rel_obj_tol=1e-300))
    assert np.allclose(res.objective, step.objective, rtol=1e-12, atol=0)
    plain = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=iters, record_trajectory=True))
    for f in ("r_h", "r_u", "lam"):
        assert np.array_equal(getattr(res.params, f), getattr(plain.params, f)), f
        assert np.array_equal(getattr(res.trajectory[-1], f), getattr(plain.trajectory[-1], f)), f


def test_early_stop(O, gpu):  # test_solver_naive.cpp:209-218
    inp, p, X = O.make_verify_instance(2, 6, 2, 10)
    res = gpu.run_naive(inp, p, _hyper(), X, _opts(iters=500, compute_objective=True, rel_obj_tol=1e-6))
    assert len(res.iter_seconds) < 500


def test_errors(O, gpu):
    from paper_1908_01964_b200 import InvalidInputError, NumericalError

    inp, p, X = O.make_verify_instance(2, 4, 2, 19)
    with pytest.raises(InvalidInputError):
        gpu.run_algorithm2(inp, p, _hyper(), X, _opts(iters=-1))
    with pytest.raises(InvalidInputError):
        gpu.build_noise_scm(np.stack([np.eye(2)] * 2), np.stack([np.eye(2)] * 2), X, 2)
    # identity demixing on data with no energy in channel 1 -> R' = 0: two null eigenvalues
    X0 = X.copy()
    X0[:, :, 1] = 0
    with pytest.raises(InvalidInputError, match="null_eigenvector"):
        gpu.build_noise_scm(np.stack([np.eye(2, dtype=complex)] * 2), np.stack([np.eye(2, dtype=complex)] * 2), X0, 0)
    bad = p.r_h.copy()
    bad[1, 2] = np.nan
    from paper_1908_01964_b200 import RcscmParams

    with pytest.raises(NumericalError, match="bin 1, frame 2"):
        gpu.map_objective(inp, RcscmParams(bad, p.r_u, p.lam), _hyper(), X)
    # singular R_x: r_u = 0 and r_h = 0 -> e_step singular covariance at (bin 0, frame 0)
    z = RcscmParams(np.zeros_like(p.r_h), np.zeros_like(p.r_u), p.lam)
    with pytest.raises(NumericalError, match="e_step: singular covariance at bin 0, frame 0"):
        gpu.run_naive(inp, z, _hyper(), X, _opts(iters=1))


def test_empty_and_tiny_shapes(O, gpu):
    from paper_1908_01964_b200 import RcscmInputs, RcscmParams

    e = RcscmInputs(np.zeros((0, 2), complex), np.zeros((0, 2, 2), complex), np.zeros((0, 2, 2), complex),
                    np.zeros((0, 2), complex), 0)
    r = gpu.run_algorithm2(e, RcscmParams(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0)), _hyper(),
                           np.zeros((0, 3, 2), complex), _opts(iters=3))
    assert r.params.r_h.shape == (0, 3)
    inp, p, X = O.make_verify_instance(3, 1, 2, 5)  # J = 1
    for backend, fn in (("accel2", gpu.run_algorithm2), ("naive", gpu.run_naive)):
        g = fn(inp, p, _hyper(), X, _opts(iters=5)).params
        o = O.run(backend, inp, p, X, O.SolverOptions(iters=5)).params
        assert O.trajectory_distance(g, o) < 1e-9


def test_maximum_frames(O, gpu):
    """The on-chip kernel's largest bin (16-CTA cluster x 256 threads x 8 slots =
    32768 frames) and one frame more (the HBM-streaming kernel) both match the
    oracle within 1e-9."""
    for J, seed in ((32768, 17), (32769, 18)):
        inp, p, X = O.make_verify_instance(2, J, 2, seed)
        g = gpu.run_algorithm2(inp, p, _hyper(), X, _opts(iters=3)).params
        o = O.run("accel2", inp, p, X, O.SolverOptions(iters=3)).params
        assert O.trajectory_distance(g, o) < 1e-9, J


def test_deterministic_and_shard_invariant(O, gpu):
    """Bitwise: repeated runs, and bins solved in two shards == one launch
    (the multi-GPU sharding argument)."""
    from paper_1908_01964_b200 import RcscmInputs, RcscmParams

    inp, p, X = O.make_verify_instance(10, 40, 4, 21)
    full = gpu.run_algorithm2(inp, p, _hyper(), X, _opts(iters=25)).params
    again = gpu.run_algorithm2(inp, p, _hyper(), X, _opts(iters=25)).params
    assert np.array_equal(full.r_u, again.r_u) and np.array_equal(full.lam, again.lam)
    parts = []
    for sl in (slice(0, 3), slice(3, 10)):
        pi = RcscmInputs(inp.a[sl], inp.R_prime[sl], inp.R_prime_pinv[sl], inp.b[sl], 0)
        pp = RcscmParams(p.r_h[sl], p.r_u[sl], p.lam[sl])
        parts.append(gpu.run_algorithm2(pi, pp, _hyper(), X[sl], _opts(iters=25)).params)
    assert np.array_equal(np.concatenate([q.r_h for q in parts]), full.r_h)
    assert np.array_equal(np.concatenate([q.r_u for q in parts]), full.r_u)
    assert np.array_equal(np.concatenate([q.lam for q in parts]), full.lam)


def test_session_pipeline_matches_entry_points(O, gpu):
    """Device-resident pipeline (setup -> precompute -> accel -> wiener) on a
    batch of 3 utterances equals the oracle per utterance."""
    from paper_1908_01964_b200 import synth
    import paper_1908_01964_b200._capi as C

    utts = synth.make_config(3, utterances=3, I=16, J=64)
    X, W, A, T, V = synth.stack(utts)
    gpu.session_load(X, W, A, T, V, 0)
    gpu.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL | C.STAGE_WIENER, 30)
    gpu.session_check()
    out = gpu.session_fetch(want_image=True)
    for k, u in enumerate(utts):
        inp = O.build_noise_scm(u.W, u.A, u.X, 0)
        p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
        o = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=30)).params
        oimg, odry = O.extract_target(inp, o, u.X)
        assert output_rel_err(out["dry"][k], odry) <= 1e-6
        assert output_rel_err(out["image"][k], oimg) <= 1e-6


@pytest.mark.parametrize("cfg,I,J", [(0, 24, 320), (1, 16, 640), (4, 6, 640), (4, 4, 4096), (2, 2, 20000)])
def test_fused_precompute_bitwise(O, gpu, monkeypatch, cfg, I, J):
    """K2 with the sigma / tau precompute fused into its prologue (one kernel for
    PRECOMPUTE | ACCEL) equals K1 + K2 bitwise, including the forms it keeps for
    the Wiener stage; M = 2, 4, 8, single-CTA bins and clusters (J = 4096, 20000)."""
    from paper_1908_01964_b200 import synth
    import paper_1908_01964_b200._capi as C

    X, W, A, T, V = synth.stack(synth.make_config(cfg, utterances=2, I=I, J=J))
    outs = []
    for fuse in ("1", "0"):
        monkeypatch.setenv("RCSCM_FUSE_PRE", fuse)
        gpu.session_load(X, W, A, T, V, 0)
        gpu.session_run(C.STAGE_SETUP)
        n0 = gpu.launch_count
        gpu.session_run(C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL, 12)
        launches = gpu.launch_count - n0
        gpu.session_run(C.STAGE_WIENER)
        gpu.session_check()
        outs.append((gpu.session_fetch(want_image=True), launches))
    (f, nf), (u, nu) = outs
    assert nf == 1 and nu == 2, (nf, nu)
    for k in ("r_h", "r_u", "lam", "dry", "image"):
        assert np.array_equal(f[k], u[k]), k


def test_pipelined_entry_point_bitwise(O, gpu, monkeypatch):
    """The copy/compute-pipelined run_algorithm2 (bins in chunks, uploads on
    two copy streams, the output sent back in 2D row-block segments while later
    chunks run) equals the single-shot path bitwise, for any segment count."""
    u, inp, p0 = _synthetic(O, 1, 300, 64)
    monkeypatch.setenv("RCSCM_PIPELINE_CHUNKS", "1")
    single = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=20)).params
    for chunks, segs in (("5", "1"), ("5", "2"), ("5", "5"), ("7", "3")):
        monkeypatch.setenv("RCSCM_PIPELINE_CHUNKS", chunks)
        monkeypatch.setenv("RCSCM_D2H_SEGS", segs)
        piped = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=20)).params
        assert np.array_equal(single.r_h, piped.r_h), (chunks, segs)
        assert np.array_equal(single.r_u, piped.r_u), (chunks, segs)
        assert np.array_equal(single.lam, piped.lam), (chunks, segs)


def test_pipelined_cluster_bitwise(O, gpu, monkeypatch):
    """The pipelined run_algorithm2 on a cluster shape (J = 4096, M = 8: 2-CTA
    clusters with the fused precompute reading and writing r_h / r_u in the
    caller's column-major layout) equals the single-shot path bitwise."""
    inp, p0, X = O.make_verify_instance(256, 4096, 8, 77)
    monkeypatch.setenv("RCSCM_PIPELINE_CHUNKS", "1")
    single = gpu.run_algorithm2(inp, p0, _hyper(), X, _opts(iters=8)).params
    monkeypatch.setenv("RCSCM_PIPELINE_CHUNKS", "3")
    piped = gpu.run_algorithm2(inp, p0, _hyper(), X, _opts(iters=8)).params
    assert np.array_equal(single.r_h, piped.r_h)
    assert np.array_equal(single.r_u, piped.r_u)
    assert np.array_equal(single.lam, piped.lam)


# ---- complex64 (FP32) mode: relative-L2 <= 1e-4 on the output ----------------------
def _rel_l2(got, ref):
    got = np.asarray(got)
    ref = np.asarray(ref)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


@pytest.fixture(scope="module")
def gpu64():
    from paper_1908_01964_b200 import GpuContext

    return GpuContext(0, precision="c64")


@pytest.mark.parametrize("cfg,I,J,iters", [(0, 64, 320, 100), (1, 32, 640, 100), (4, 8, 4096, 100), (2, 4, 20000, 50)])
def test_c64_output_rel_l2(O, gpu64, cfg, I, J, iters):
    u, inp, p0 = _synthetic(O, cfg, I, J)
    g = gpu64.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=iters)).params
    o = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=iters)).params
    ge = gpu64.extract_target(inp, g, u.X)
    oimg, odry = O.extract_target(inp, o, u.X)
    assert _rel_l2(ge.dry, odry) <= 1e-4, _rel_l2(ge.dry, odry)
    assert _rel_l2(ge.image, oimg) <= 1e-4
    assert _rel_l2(g.lam, o.lam) <= 1e-4


def test_c64_session_pipeline(O, gpu64):
    from paper_1908_01964_b200 import synth
    import paper_1908_01964_b200._capi as C

    utts = synth.make_config(4, utterances=2, I=8, J=4096)
    X, W, A, T, V = synth.stack(utts)
    gpu64.session_load(X, W, A, T, V, 0)
    gpu64.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL | C.STAGE_WIENER, 100)
    gpu64.session_check()
    out = gpu64.session_fetch(want_image=True)
    for k, u in enumerate(utts):
        inp = O.build_noise_scm(u.W, u.A, u.X, 0)
        p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
        o = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=100)).params
        oimg, odry = O.extract_target(inp, o, u.X)
        assert _rel_l2(out["dry"][k], odry) <= 1e-4
        assert _rel_l2(out["image"][k], oimg) <= 1e-4


@pytest.mark.parametrize("prec", ["c128", "c64"])
def test_session_reset_replays(O, gpu, gpu64, prec):
    """RESET restores params0 lazily: RESET+ACCEL replays the first run bitwise,
    RESET followed by a fetch returns params0, and RESET+NAIVE starts from params0."""
    from paper_1908_01964_b200 import synth
    import paper_1908_01964_b200._capi as C

    g = gpu if prec == "c128" else gpu64
    utts = synth.make_config(1, utterances=2, I=24, J=640)
    X, W, A, T, V = synth.stack(utts)
    g.session_load(X, W, A, T, V, 0)
    g.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    p0 = g.session_fetch()
    g.session_run(C.STAGE_ACCEL, 7)
    first = g.session_fetch()
    g.session_run(C.STAGE_ACCEL, 3)  # moves the iterate on
    g.session_run(C.STAGE_RESET | C.STAGE_ACCEL, 7)
    again = g.session_fetch()
    for k in ("r_h", "r_u", "lam"):
        assert np.array_equal(first[k], again[k]), k
        assert not np.array_equal(first[k], p0[k]), k
    g.session_run(C.STAGE_RESET)
    back = g.session_fetch()
    for k in ("r_h", "r_u", "lam"):
        assert np.array_equal(back[k], p0[k]), k
    g.session_run(C.STAGE_ACCEL, 3)
    g.session_run(C.STAGE_RESET | C.STAGE_NAIVE, 2)
    nv = g.session_fetch()
    u = utts[1]
    inp = O.build_noise_scm(u.W, u.A, u.X, 0)
    o0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    if prec == "c128":
        o = O.run("naive", inp, o0, u.X, O.SolverOptions(iters=2)).params
        assert np.allclose(nv["lam"][1], o.lam, rtol=1e-8, atol=0)
    g.session_check()


@pytest.mark.parametrize("cfg,I,J,cl", [(4, 6, 4096, "2"), (4, 6, 4096, "4"), (2, 2, 20000, "16")])
def test_cluster_constant_placement_bitwise(O, gpu, monkeypatch, cfg, I, J, cl):
    """A cluster shape gives the same bits whether the per-slot constants live in
    registers or in shared memory (the default for clusters): placement changes
    residency, not arithmetic. Both agree with the oracle's lambda within 1e-9."""
    u, inp, p0 = _synthetic(O, cfg, I, J)
    monkeypatch.setenv("RCSCM_ACCEL_CL", cl)
    runs = []
    for smem in ("0", "1"):
        monkeypatch.setenv("RCSCM_ACCEL_SMEM", smem)
        runs.append(gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=10)).params)
    assert np.array_equal(runs[0].r_h, runs[1].r_h)
    assert np.array_equal(runs[0].r_u, runs[1].r_u)
    assert np.array_equal(runs[0].lam, runs[1].lam)
    o = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=10)).params
    rel = np.abs(runs[1].lam - o.lam) / np.maximum(np.maximum(np.abs(runs[1].lam), np.abs(o.lam)), 1e-12)
    assert rel.max() <= 1e-9, rel.max()


def test_build_inputs_and_run_accel_entry_points(O, gpu):
    """rcscm_gpu_build_inputs == build_noise_scm + init_params and
    rcscm_gpu_run_accel(stage) == run_algorithm1 / run_algorithm2, bitwise; a stage
    other than 1 or 2 is InvalidInputError."""
    from paper_1908_01964_b200 import synth
    from paper_1908_01964_b200.api import InvalidInputError

    u = synth.make_config(1, utterances=1, I=12, J=64)[0]
    inp, p0 = gpu.build_inputs(u.W, u.A, u.X, 0, u.T, u.V)
    ref_inp = gpu.build_noise_scm(u.W, u.A, u.X, 0)
    ref_p0 = gpu.init_params(ref_inp, u.T, u.V, u.W, u.A, u.X)
    for k in ("a", "R_prime", "R_prime_pinv", "b"):
        assert np.array_equal(getattr(inp, k), getattr(ref_inp, k)), k
    for k in ("r_h", "r_u", "lam"):
        assert np.array_equal(getattr(p0, k), getattr(ref_p0, k)), k
    for stage, fn in ((1, gpu.run_algorithm1), (2, gpu.run_algorithm2)):
        a = gpu.run_accel(stage, inp, p0, _hyper(), u.X, _opts(iters=7)).params
        b = fn(inp, p0, _hyper(), u.X, _opts(iters=7)).params
        assert np.array_equal(a.r_h, b.r_h) and np.array_equal(a.r_u, b.r_u) and np.array_equal(a.lam, b.lam)
    with pytest.raises(InvalidInputError, match="stage must be 1 or 2"):
        gpu.run_accel(3, inp, p0, _hyper(), u.X, _opts(iters=1))
