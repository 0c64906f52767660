"""Oracle pins: ports of proj/tests/test_solver_naive.cpp:13-218 and
proj/tests/test_wiener.cpp:9-93 onto the oracle."""
import numpy as np
import pytest

from conftest import rel_error


def _dense_e_step(inp, p, X):
    """test_solver_naive.cpp:13-40: independent dense evaluation."""
    I, J, M = X.shape
    hr = np.zeros((I, J))
    hu = np.zeros((I, J, M, M), complex)
    for i in range(I):
        a = inp.a[i]
        Rut = inp.R_prime[i] + p.lam[i] * np.outer(inp.b[i], inp.b[i].conj())
        for t in range(J):
            rh, ru, x = p.r_h[i, t], p.r_u[i, t], X[i, t]
            Rxi = np.linalg.inv(rh * np.outer(a, a.conj()) + ru * Rut)
            hr[i, t] = rh - rh * rh * np.real(a.conj() @ Rxi @ a) + abs(rh * (a.conj() @ (Rxi @ x)).conjugate()) ** 2
            G = ru * Rut @ Rxi
            hu[i, t] = ru * Rut - G @ (ru * Rut) + G @ np.outer(x, x.conj()) @ G.conj().T
    return hr, hu


def _scalar(O):
    inp = O.Inputs(np.ones((1, 1), complex), np.zeros((1, 1, 1), complex), np.zeros((1, 1, 1), complex),
                   np.ones((1, 1), complex), 0)
    p = O.Params(np.ones((1, 1)), np.ones((1, 1)), np.array([2.0]))
    return inp, p, np.full((1, 1, 1), 3.0 + 0j)


def test_e_step_scalar_hand(O):  # test_solver_naive.cpp:44-58: R^x = 3, r^ = 1 - 1/3 + 1 = 5/3
    inp, p, X = _scalar(O)
    hr, _ = O.e_step(inp, p, X)
    assert hr[0, 0] == pytest.approx(5 / 3, rel=1e-12)
    # chained through the M-step: r_h = (5/3 + beta)/(alpha + 2)  (SPEC update_rh example)
    res = O.run("naive", inp, p, X, O.SolverOptions(iters=1))
    assert res.params.r_h[0, 0] == pytest.approx((5 / 3 + 1e-16) / 3.1, rel=1e-12)


def test_e_step_rh_zero(O):  # :60-65
    inp, p, X = O.make_verify_instance(2, 6, 3, 1)
    p.r_h[:] = 0
    hr, _ = O.e_step(inp, p, X)
    assert np.max(np.abs(hr)) == 0.0


def test_e_step_psd_and_dense(O):  # :67-84
    inp, p, X = O.make_verify_instance(4, 12, 4, 2)
    hr, hu = O.e_step(inp, p, X)
    dhr, dhu = _dense_e_step(inp, p, X)
    assert np.all(hr >= 0)
    for i in range(4):
        for t in range(12):
            assert rel_error(hr[i, t], dhr[i, t]) < 1e-10
            assert rel_error(hu[i, t], dhu[i, t]) < 1e-10
            sym = (hu[i, t] + hu[i, t].conj().T) / 2
            assert np.linalg.eigvalsh(sym)[0] > -1e-9 * np.real(np.trace(sym))


def test_m_step_trivial_fixed_point(O):  # :86-119
    inp, p, X = O.make_verify_instance(2, 5, 3, 3)
    hu = np.zeros((2, 5, 3, 3), complex)
    for i in range(2):
        hu[i, :] = inp.R_prime[i] + p.lam[i] * np.outer(inp.b[i], inp.b[i].conj())
    nxt = O.m_step(np.zeros((2, 5)), hu, inp, p)
    assert np.max(np.abs(nxt.r_h - max(1e-16 / 3.1, 1e-12))) == 0.0
    for i in range(2):
        lam_new = np.mean(p.lam[i] / p.r_u[i])
        assert nxt.lam[i] == pytest.approx(lam_new, rel=1e-10)
        assert np.allclose(nxt.r_u[i], (3 - 1 + p.lam[i] / lam_new) / 3, rtol=1e-10)


def test_m_step_scripted(O):  # :121-145
    inp, p, X = O.make_verify_instance(3, 8, 4, 4)
    hr, hu = O.e_step(inp, p, X)
    nxt = O.m_step(hr, hu, inp, p)
    for i in range(3):
        b = inp.b[i]
        lam = 0.0
        for t in range(8):
            assert rel_error(nxt.r_h[i, t], max((hr[i, t] + 1e-16) / 3.1, 1e-12)) < 1e-12
            lam += np.real(b.conj() @ hu[i, t] @ b) / p.r_u[i, t]
        lam = max(lam / 8, 1e-12)
        assert rel_error(nxt.lam[i], lam) < 1e-12
        Ru = inp.R_prime[i] + lam * np.outer(b, b.conj())
        for t in range(8):
            ru = np.real(np.trace(np.linalg.inv(Ru) @ hu[i, t])) / 4
            assert rel_error(nxt.r_u[i, t], max(ru, 1e-12)) < 1e-10


def test_naive_iters_zero(O):  # :147-156
    inp, p, X = O.make_verify_instance(2, 4, 2, 5)
    res = O.run("naive", inp, p, X, O.SolverOptions(iters=0))
    assert O.trajectory_distance(res.params, p) == 0.0


def test_fused_equals_explicit(O):  # :158-168
    inp, p, X = O.make_verify_instance(3, 10, 4, 6)
    res = O.run("naive", inp, p, X, O.SolverOptions(iters=1))
    hr, hu = O.e_step(inp, p, X)
    assert O.trajectory_distance(res.params, O.m_step(hr, hu, inp, p)) < 1e-12


def test_naive_monotone_objective(O):  # :170-181
    inp, p, X = O.make_verify_instance(4, 16, 3, 7)
    obj = O.run("naive", inp, p, X, O.SolverOptions(iters=100, compute_objective=True)).objective
    assert len(obj) == 101
    for k in range(1, 101):
        assert obj[k] >= obj[k - 1] - 1e-7 * abs(obj[k - 1])


def test_naive_fixed_point(O):  # :183-193
    inp, p, X = O.make_verify_instance(2, 8, 3, 8)
    conv = O.run("naive", inp, p, X, O.SolverOptions(iters=4000)).params
    probe = O.run("naive", inp, conv, X, O.SolverOptions(iters=1)).params
    assert O.trajectory_distance(probe, conv) < 1e-9


def test_naive_threads_bitwise(O):  # :195-207
    inp, p, X = O.make_verify_instance(7, 12, 4, 9)
    one = O.run("naive", inp, p, X, O.SolverOptions(iters=20)).params
    four = O.run("naive", inp, p, X, O.SolverOptions(iters=20, threads=4)).params
    assert O.trajectory_distance(one, four) == 0.0


def test_naive_early_stop(O):  # :209-218
    inp, p, X = O.make_verify_instance(2, 6, 2, 10)
    res = O.run("naive", inp, p, X, O.SolverOptions(iters=500, compute_objective=True, rel_obj_tol=1e-6))
    assert len(res.iter_seconds) < 500


# ---- wiener.hpp ---------------------------------------------------------------
def test_wiener_rh_zero(O):  # test_wiener.cpp:9-15
    inp, p, X = O.make_verify_instance(3, 8, 3, 1)
    p.r_h[:] = 0
    image, dry = O.extract_target(inp, p, X)
    assert np.max(np.abs(dry)) == 0.0 and np.max(np.abs(image)) == 0.0


def test_wiener_noiseless(O):  # :17-29
    inp, p, X = O.make_verify_instance(2, 4, 3, 2)
    c = 1.5 - 0.8j
    X = c * np.repeat(inp.a[:, None, :], 4, axis=1)
    p.r_u[:] = 1e-14
    p.r_h[:] = 1.0
    _, dry = O.extract_target(inp, p, X)
    assert np.max(np.abs(dry - c)) < 1e-6


def test_wiener_dense(O):  # :31-49
    inp, p, X = O.make_verify_instance(4, 10, 4, 3)
    image, dry = O.extract_target(inp, p, X)
    for i in range(4):
        a = inp.a[i]
        Ru = inp.R_prime[i] + p.lam[i] * np.outer(inp.b[i], inp.b[i].conj())
        for t in range(10):
            rh = p.r_h[i, t]
            s = rh * (a.conj() @ np.linalg.solve(rh * np.outer(a, a.conj()) + p.r_u[i, t] * Ru, X[i, t]))
            assert abs(dry[i, t] - s) < 1e-9 * max(1, abs(s))
            assert np.linalg.norm(image[i, t] - dry[i, t] * a) < 1e-12


def test_noise_complement_bitwise(O):  # :51-62
    inp, p, X = O.make_verify_instance(3, 6, 3, 4)
    image, _ = O.extract_target(inp, p, X)
    noise = O.extract_noise(inp, p, X)
    assert np.max(np.abs(X - image - noise)) == 0.0


def test_noise_zero_when_target_is_x(O):  # :64-74
    inp, p, X = O.make_verify_instance(2, 4, 2, 5)
    X = (2 + 1j) * np.repeat(inp.a[:, None, :], 4, axis=1)
    p.r_u[:] = 1e-14
    p.r_h[:] = 1.0
    assert np.max(np.abs(O.extract_noise(inp, p, X))) < 1e-5


def test_noise_posterior_mean(O):  # :76-93
    inp, p, X = O.make_verify_instance(3, 8, 4, 6)
    noise = O.extract_noise(inp, p, X)
    for i in range(3):
        a = inp.a[i]
        Ru = inp.R_prime[i] + p.lam[i] * np.outer(inp.b[i], inp.b[i].conj())
        for t in range(8):
            ru = p.r_u[i, t]
            u = ru * Ru @ np.linalg.solve(p.r_h[i, t] * np.outer(a, a.conj()) + ru * Ru, X[i, t])
            assert np.linalg.norm(noise[i, t] - u) < 1e-9 * max(1, np.linalg.norm(u))
