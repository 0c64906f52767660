"""Sphering and Gaussian ILRMA (ilrma.hpp): the oracle restatement pinned by the
reference's own cases (proj/tests/test_ilrma.cpp), and the GPU path against the
oracle. Random spectrograms are numpy-seeded (the reference's Rng draws are not
reproduced; its checks are seed-free). The NMF initial draws use the C++
standard library exactly as the reference does (mt19937_64 + uniform (0.1, 1])."""
import numpy as np
import pytest


def _spec(I, J, M, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal((I, J, M)) + 1j * r.standard_normal((I, J, M))


def _cov(x):  # x (J, M)
    return x.T @ x.conj() / x.shape[0]


# ---- oracle pinned by the reference cases ----------------------------------------
def test_oracle_sphere(O):
    """test_ilrma.cpp:27-52: whitened covariance = I; scale invariance; M = 1
    gives unit variance; J <= M rejected."""
    x = _spec(6, 200, 4, 1)
    _, xw = O.sphere(x)
    for i in range(6):
        assert np.linalg.norm(_cov(xw[i]) - np.eye(4)) < 1e-6
    x = _spec(3, 100, 3, 2)
    _, a = O.sphere(x)
    _, b = O.sphere(10.0 * x)
    for i in range(3):
        assert np.linalg.norm(a[i] - b[i]) < 1e-8 * np.linalg.norm(a[i])
    _, w1 = O.sphere(_spec(2, 300, 1, 3))
    assert np.allclose(np.sum(np.abs(w1) ** 2, axis=(1, 2)) / 300.0, 1.0)
    with pytest.raises(O.InvalidInputError, match="need more frames"):
        O.sphere(_spec(2, 3, 3, 4))


def test_oracle_ilrma_reference_cases(O):
    """test_ilrma.cpp:91-154: iters = 0 keeps W = I with a nonnegative fitted NMF;
    deterministic given the seed with W A = I; the objective never increases over
    growing iteration counts; K < 1 and iters < 0 rejected."""
    x = _spec(4, 50, 2, 5)
    W, A, T, V = O.run_ilrma(x, 4, 0, 7)
    assert np.all(np.linalg.norm(W - np.eye(2), axis=(1, 2)) < 1e-12)
    assert T.min() >= 0 and V.min() >= 0
    x = _spec(6, 80, 3, 6)
    a = O.run_ilrma(x, 3, 10, 11)
    b = O.run_ilrma(x, 3, 10, 11)
    assert np.array_equal(a[0], b[0])
    assert np.all(np.linalg.norm(a[0] @ a[1] - np.eye(3), axis=(1, 2)) < 1e-8)
    x = _spec(6, 60, 2, 9)
    prev = np.inf
    for iters in (1, 3, 6, 10, 20):
        W, A, T, V = O.run_ilrma(x, 4, iters, 21)
        obj = O.ilrma_objective(x, W, T, V)
        assert obj <= prev + 1e-7 * abs(prev)
        prev = obj
    x = _spec(2, 30, 2, 10)
    with pytest.raises(O.InvalidInputError):
        O.run_ilrma(x, 0, 5, 1)
    with pytest.raises(O.InvalidInputError):
        O.run_ilrma(x, 2, -1, 1)
