"""Oracle pins: ports of proj/tests/test_model.cpp:36-225 (build_noise_scm,
init_params, map_objective) onto the oracle."""
import numpy as np
import pytest

from conftest import random_demixing, random_spectrogram, rel_error


def test_build_identity_m2(O):  # test_model.cpp:36-49
    x = random_spectrogram(3, 40, 2, 1)
    W = np.stack([np.eye(2, dtype=complex)] * 3)
    inp = O.build_noise_scm(W, W, x, 0)
    for i in range(3):
        mean_p2 = np.sum(np.abs(x[i, :, 1]) ** 2) / 40
        assert abs(inp.R_prime[i][0, 0]) < 1e-14
        assert abs(inp.R_prime[i][1, 1] - mean_p2) < 1e-12 * mean_p2
        assert np.linalg.norm(inp.b[i] - np.array([1, 0])) < 1e-10
        assert np.linalg.norm(inp.a[i] - np.array([1, 0])) < 1e-12


def test_build_rank_null_pinv(O):  # :51-67
    x = random_spectrogram(5, 60, 4, 2)
    W, A = random_demixing(5, 4, 3)
    inp = O.build_noise_scm(W, A, x, 1)
    assert inp.n_h == 1
    for i in range(5):
        ev = np.linalg.eigvalsh(inp.R_prime[i])
        assert np.sum(ev > 1e-10 * ev[3]) == 3
        assert np.linalg.norm(inp.R_prime[i] @ inp.b[i]) < 1e-8 * ev[3]
        P = inp.R_prime_pinv[i]
        assert rel_error(P @ inp.R_prime[i] @ P, P) < 1e-8
        assert np.linalg.norm(inp.a[i] - A[i][:, 1]) < 1e-12


def test_build_sum_of_backprojected(O):  # :69-88
    x = random_spectrogram(4, 30, 3, 4)
    W, A = random_demixing(4, 3, 5)
    n_h = 2
    inp = O.build_noise_scm(W, A, x, n_h)
    for i in range(4):
        ref = np.zeros((3, 3), complex)
        for n in range(3):
            if n == n_h:
                continue
            for t in range(30):
                y = A[i][:, n] * (W[i][n] @ x[i, t])
                ref += np.outer(y, y.conj())
        assert rel_error(inp.R_prime[i], ref / 30) < 1e-10


def test_build_partition(O):  # :90-110
    x = random_spectrogram(3, 50, 4, 6)
    W, A = random_demixing(3, 4, 7)
    inp = O.build_noise_scm(W, A, x, 0)
    for i in range(3):
        y = x[i] @ W[i].T  # (J, M) demixed
        p = np.abs(y) ** 2
        full = np.einsum("rn,tn,cn->rc", A[i], p, A[i].conj()) / 50
        tp = p[:, 0].mean()
        assert rel_error(full, inp.R_prime[i] + tp * np.outer(inp.a[i], inp.a[i].conj())) < 1e-9


def test_build_target_out_of_range(O):  # :112-117
    x = random_spectrogram(2, 20, 2, 8)
    W, A = random_demixing(2, 2, 9)
    for n_h in (2, -1):
        with pytest.raises(O.InvalidInputError):
            O.build_noise_scm(W, A, x, n_h)


def test_init_all_ones_nmf(O):  # :119-132
    x = random_spectrogram(3, 25, 2, 10)
    W, A = random_demixing(3, 2, 11)
    inp = O.build_noise_scm(W, A, x, 0)
    p = O.init_params(inp, np.ones((3, 10)), np.ones((10, 25)), W, A, x)
    assert np.max(np.abs(p.r_h - 10.0)) < 1e-12
    assert p.r_u.min() >= 1e-12 and p.lam.min() >= 1e-12


def test_init_lambda_second_eig(O):  # :134-148
    x = random_spectrogram(4, 40, 4, 12)
    W, A = random_demixing(4, 4, 13)
    inp = O.build_noise_scm(W, A, x, 0)
    p = O.init_params(inp, np.ones((4, 2)), np.ones((2, 40)), W, A, x)
    for i in range(4):
        assert p.lam[i] == pytest.approx(np.linalg.eigvalsh(inp.R_prime[i])[1], rel=1e-10)


def test_init_ru_formula(O):  # :150-169
    x = random_spectrogram(3, 20, 3, 14)
    W, A = random_demixing(3, 3, 15)
    n_h = 1
    inp = O.build_noise_scm(W, A, x, n_h)
    p = O.init_params(inp, np.ones((3, 2)), np.ones((2, 20)), W, A, x)
    for i in range(3):
        for t in range(20):
            y = W[i] @ x[i, t]
            y[n_h] = 0
            yh = A[i] @ y  # ilrma.hpp:78-83
            expected = max(np.real(yh.conj() @ inp.R_prime_pinv[i] @ yh) / 3, 1e-12)
            assert p.r_u[i, t] == pytest.approx(expected, rel=1e-10)


def _scalar_inputs(O):
    return O.Inputs(np.ones((1, 1), complex), np.zeros((1, 1, 1), complex), np.zeros((1, 1, 1), complex),
                    np.ones((1, 1), complex), 0)


def test_objective_scalar(O):  # :188-206
    inp = _scalar_inputs(O)
    p = O.Params(np.ones((1, 1)), np.ones((1, 1)), np.ones(1))
    x = np.ones((1, 1, 1), complex)
    expected = -np.log(2 * np.pi) - 0.5 - 2.1 * 0.0 - 1e-16
    assert O.map_objective(inp, p, x) == pytest.approx(expected, rel=1e-12)


def test_objective_phase_invariant(O):  # :208-217
    inp, p, X = O.make_verify_instance(3, 10, 3, 18)
    base = O.map_objective(inp, p, X)
    assert O.map_objective(inp, p, X * np.exp(0.7j)) == pytest.approx(base, rel=1e-12)


def test_objective_reports_slot(O):  # :219-225
    inp, p, X = O.make_verify_instance(2, 4, 2, 19)
    p.r_h[1, 2] = np.nan
    with pytest.raises(O.NumericalError, match="bin 1, frame 2"):
        O.map_objective(inp, p, X)


def test_objective_dense(O):  # independent numpy evaluation of model.hpp:129-157
    inp, p, X = O.make_verify_instance(3, 7, 4, 20)
    ref = 0.0
    for i in range(3):
        Ru = inp.R_prime[i] + p.lam[i] * np.outer(inp.b[i], inp.b[i].conj())
        for t in range(7):
            Rx = p.r_h[i, t] * np.outer(inp.a[i], inp.a[i].conj()) + p.r_u[i, t] * Ru
            _, logdet = np.linalg.slogdet(np.pi * Rx)
            quad = np.real(X[i, t].conj() @ np.linalg.solve(Rx, X[i, t]))
            ref += -logdet - quad - 2.1 * np.log(p.r_h[i, t]) - 1e-16 / p.r_h[i, t]
    assert O.map_objective(inp, p, X) == pytest.approx(ref, rel=1e-12)
