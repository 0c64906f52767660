"""Oracle pins: ports of proj/tests/test_solver_accel.cpp:23-365 onto the
oracle's restatement of solver_accel.hpp (instances from make_verify_instance
with the reference's own seeds)."""
import numpy as np
import pytest

from conftest import Rng, rel_error


def test_precompute_sigma(O):  # test_solver_accel.cpp:23-41
    inp, p, X = O.make_verify_instance(3, 6, 4, 1)
    inp.a[0] -= inp.b[0] * (inp.b[0].conj() @ inp.a[0])  # force a ⊥ b in bin 0
    s = O.precompute(inp, X)
    assert abs(s.sigma_ab[0]) < 1e-12
    for i in range(3):
        assert abs(s.sigma_ab[i] - inp.a[i].conj() @ inp.b[i]) < 1e-14
        for t in range(6):
            assert abs(s.sigma_bx[i, t] - inp.b[i].conj() @ X[i, t]) < 1e-14


def test_precompute_tau(O):  # :43-81
    inp = O.Inputs(np.array([[1, 0]], complex), np.diag([2.0, 0.0])[None].astype(complex),
                   np.diag([0.5, 0.0])[None].astype(complex), np.array([[0, 1]], complex), 0)
    X = Rng(3).complex_matrix(4, 2)[None]
    s = O.precompute(inp, X)
    assert s.tau_aa[0] == pytest.approx(0.5, rel=1e-14)
    inp.a[0] = 3.0 * inp.b[0]  # a ∝ b: annihilated by the pseudoinverse
    assert O.precompute(inp, X).tau_aa[0] < 1e-14
    rnd, _, Xr = O.make_verify_instance(3, 8, 4, 4)
    sr = O.precompute(rnd, Xr)
    for i in range(3):
        P = rnd.R_prime_pinv[i]
        assert rel_error(sr.tau_aa[i], np.real(rnd.a[i].conj() @ P @ rnd.a[i])) < 1e-12
        for t in range(8):
            x = Xr[i, t]
            assert sr.tau_xx[i, t] >= 0
            assert rel_error(sr.tau_xx[i, t], np.real(x.conj() @ P @ x)) < 1e-12
            ax = rnd.a[i].conj() @ P @ x
            assert abs(sr.tau_ax[i, t] - ax) < 1e-12 * max(1.0, abs(sr.tau_ax[i, t]))


def test_compute_gamma(O):  # :83-110
    _, p, _ = O.make_verify_instance(2, 4, 3, 5)
    trho = np.ones(2)
    assert np.max(np.abs(O.compute_gamma(np.zeros((2, 4)), p.r_u, trho))) == 0.0
    g = O.compute_gamma(np.ones((2, 4)), np.ones((2, 4)), trho)
    assert np.max(np.abs(g - 0.5)) < 1e-15
    _, rp, _ = O.make_verify_instance(2, 4, 3, 6)
    trho = np.array([0.3, 1.7])
    g = O.compute_gamma(rp.r_h, rp.r_u, trho)
    exp = rp.r_h / (rp.r_u + rp.r_h * trho[:, None])
    assert np.max(np.abs(g - exp) / exp) < 1e-14
    assert np.all(g * trho[:, None] >= 0) and np.all(g * trho[:, None] < 1)


def test_rho_first_stage_scalar(O):  # :112-128
    inp = O.Inputs(np.ones((1, 1), complex), np.zeros((1, 1, 1), complex), np.zeros((1, 1, 1), complex),
                   np.ones((1, 1), complex), 0)
    raa, rax, rxx = O.rho_first_stage(inp, np.zeros((1, 3, 1), complex), np.array([2.0]))
    assert raa[0] == pytest.approx(0.5, rel=1e-14)
    assert np.max(np.abs(rax)) == 0.0 and np.max(np.abs(rxx)) == 0.0


def test_rho_stages_vs_dense(O):  # :130-159
    inp, p, X = O.make_verify_instance(4, 10, 4, 7)
    s = O.precompute(inp, X)
    raa1, rax1, rxx1 = O.rho_first_stage(inp, X, p.lam)
    raa2, rax2, rxx2 = O.rho_second_stage(s, p.lam)
    for i in range(4):
        Rinv = np.linalg.inv(inp.R_prime[i] + p.lam[i] * np.outer(inp.b[i], inp.b[i].conj()))
        aa = np.real(inp.a[i].conj() @ Rinv @ inp.a[i])
        assert rel_error(raa1[i], aa) < 1e-10 and rel_error(raa2[i], aa) < 1e-10
        for t in range(10):
            x = X[i, t]
            ax = inp.a[i].conj() @ Rinv @ x
            xx = np.real(x.conj() @ Rinv @ x)
            assert abs(rax1[i, t] - ax) < 1e-10 * max(1, abs(ax))
            assert abs(rax2[i, t] - ax) < 1e-10 * max(1, abs(ax))
            assert rel_error(rxx1[i, t], xx) < 1e-10 and rel_error(rxx2[i, t], xx) < 1e-10


def test_rho_second_stage_lambda_limits(O):  # :161-183
    inp, _, X = O.make_verify_instance(1, 4, 3, 8)
    s = O.precompute(inp, X)
    s.sigma_ab[0] = 0.0
    for lam in (1e-3, 1.0, 1e3):
        raa, _, _ = O.rho_second_stage(s, np.array([lam]), want_xx=False)
        assert rel_error(raa[0], s.tau_aa[0]) < 1e-14
    s.sigma_ab[0] = 0.4 - 0.3j
    prev = np.inf
    for lam in (1e-2, 1.0, 1e2, 1e4):
        raa, _, _ = O.rho_second_stage(s, np.array([lam]), want_xx=False)
        assert s.tau_aa[0] < raa[0] < prev
        prev = raa[0]


def test_intermediate_identities(O):  # :185-211
    inp, p, X = O.make_verify_instance(3, 6, 4, 9)
    trho_aa, trho_ax, _ = O.rho_first_stage(inp, X, p.lam, want_xx=False)
    for i in range(3):
        Ru = inp.R_prime[i] + p.lam[i] * np.outer(inp.b[i], inp.b[i].conj())
        a = inp.a[i]
        for t in range(6):
            rh, ru = p.r_h[i, t], p.r_u[i, t]
            Rxi = np.linalg.inv(rh * np.outer(a, a.conj()) + ru * Ru)
            assert rel_error(np.real(a.conj() @ Rxi @ a), trho_aa[i] / (ru + rh * trho_aa[i])) < 1e-10
            ax = a.conj() @ Rxi @ X[i, t]
            exp = trho_ax[i, t] / (ru + rh * trho_aa[i])
            assert abs(ax - exp) < 1e-10 * max(1, abs(exp))


def test_updates_match_naive_m_step(O):  # :213-241
    inp, p, X = O.make_verify_instance(3, 8, 4, 10)
    hr, hu = O.e_step(inp, p, X)
    naive = O.m_step(hr, hu, inp, p)
    s = O.precompute(inp, X)
    trho_aa, trho_ax, _ = O.rho_first_stage(inp, X, p.lam, want_xx=False)
    g = O.compute_gamma(p.r_h, p.r_u, trho_aa)
    r_h = O.update_rh(g, p.r_u, trho_ax)
    assert np.max(np.abs(r_h - naive.r_h) / np.maximum(np.abs(naive.r_h), 1e-12)) < 1e-9
    lam = O.update_lambda(g, p.r_u, s.sigma_ab, s.sigma_bx, trho_ax)
    for i in range(3):
        assert rel_error(lam[i], naive.lam[i]) < 1e-9
    raa, rax, rxx = O.rho_first_stage(inp, X, lam)
    r_u = O.update_ru(g, p.r_u, raa, rax, trho_ax, rxx, 4)
    assert np.max(np.abs(r_u - naive.r_u) / np.maximum(np.abs(naive.r_u), 1e-12)) < 1e-9


def test_update_rules_scalar_cases(O):  # :243-287
    inp, p, X = O.make_verify_instance(1, 3, 2, 11)
    s = O.precompute(inp, X)
    zero3 = np.zeros((1, 3))
    r_h = O.update_rh(zero3, p.r_u, np.zeros((1, 3), complex))
    assert np.max(np.abs(r_h - max(1e-16 / 3.1, 1e-12))) == 0.0
    lam = O.update_lambda(np.full((1, 3), 0.25), p.r_u, s.sigma_ab, np.zeros((1, 3), complex),
                          np.zeros((1, 3), complex), eps=0.0)
    assert rel_error(lam[0], 0.25 * abs(s.sigma_ab[0]) ** 2) < 1e-12
    lam = O.update_lambda(np.full((1, 3), 0.5), p.r_u, np.zeros(1, complex), s.sigma_bx,
                          np.zeros((1, 3), complex), eps=0.0)
    assert rel_error(lam[0], np.mean(np.abs(s.sigma_bx[0]) ** 2 / p.r_u[0])) < 1e-12
    r_u = O.update_ru(zero3, p.r_u, np.ones(1), np.zeros((1, 3), complex), np.zeros((1, 3), complex),
                      np.full((1, 3), 6.0), 2)
    assert np.max(np.abs(r_u - 3.0)) < 1e-14
    r_u = O.update_ru(zero3, p.r_u, np.ones(1), np.zeros((1, 3), complex), np.zeros((1, 3), complex),
                      np.zeros((1, 3)), 2)
    assert np.max(np.abs(r_u - 1e-12)) == 0.0


def test_iters_zero_passthrough(O):  # :289-298
    inp, p, X = O.make_verify_instance(2, 4, 3, 12)
    for backend in ("accel1", "accel2"):
        res = O.run(backend, inp, p, X, O.SolverOptions(iters=0))
        assert O.trajectory_distance(res.params, p) == 0.0


def test_trajectory_equality(O):  # :300-318
    inp, p, X = O.make_verify_instance(8, 16, 4, 13)
    opt = O.SolverOptions(iters=50, record_trajectory=True)
    naive = O.run("naive", inp, p, X, opt)
    for backend in ("accel1", "accel2"):
        acc = O.run(backend, inp, p, X, opt)
        assert len(acc.trajectory) == 50
        for k in range(50):
            assert O.trajectory_distance(naive.trajectory[k], acc.trajectory[k]) < 1e-8


def test_monotone_objective(O):  # :320-332
    inp, p, X = O.make_verify_instance(4, 12, 3, 14)
    for backend in ("accel1", "accel2"):
        obj = O.run(backend, inp, p, X, O.SolverOptions(iters=100, compute_objective=True)).objective
        assert len(obj) == 101
        for k in range(1, len(obj)):
            assert obj[k] >= obj[k - 1] - 1e-7 * abs(obj[k - 1])


def test_gamma_fault_detected(O):  # :334-349
    inp, p, X = O.make_verify_instance(3, 8, 3, 15)
    opt = O.SolverOptions(iters=10, record_trajectory=True)
    naive = O.run("naive", inp, p, X, opt)
    opt.gamma_fault = 1e-3
    bad = O.run("accel2", inp, p, X, opt)
    assert max(O.trajectory_distance(a, b) for a, b in zip(naive.trajectory, bad.trajectory)) > 1e-8


def test_thread_count_bitwise(O):  # :351-365
    inp, p, X = O.make_verify_instance(7, 10, 3, 16)
    for backend in ("accel1", "accel2"):
        one = O.run(backend, inp, p, X, O.SolverOptions(iters=25))
        four = O.run(backend, inp, p, X, O.SolverOptions(iters=25, threads=4))
        assert np.array_equal(one.params.r_h, four.params.r_h)
        assert np.array_equal(one.params.r_u, four.params.r_u)
        assert np.array_equal(one.params.lam, four.params.lam)
    bp = O.run("accel2_binparallel", inp, p, X, O.SolverOptions(iters=25, threads=4))
    ser = O.run("accel2", inp, p, X, O.SolverOptions(iters=25))
    assert O.trajectory_distance(bp.params, ser.params) == 0.0


@pytest.mark.parametrize("I,J,M", [(8, 16, 2), (8, 16, 3), (8, 128, 4), (64, 16, 8)])
def test_verify_grid(O, I, J, M):  # tools/rcscm.cpp:223-275 (cmd_verify), seed = 1000 I + 10 J + M
    inp, p, X = O.make_verify_instance(I, J, M, 1000 * I + 10 * J + M)
    opt = O.SolverOptions(iters=50, record_trajectory=True)
    naive = O.run("naive", inp, p, X, opt)
    a1 = O.run("accel1", inp, p, X, opt)
    a2 = O.run("accel2", inp, p, X, opt)
    worst = max(max(O.trajectory_distance(n, x), O.trajectory_distance(n, y))
                for n, x, y in zip(naive.trajectory, a1.trajectory, a2.trajectory))
    assert worst <= 1e-8
