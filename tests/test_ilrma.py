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


# ---- GPU ------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("I,J,M", [(6, 200, 4), (5, 64, 2), (3, 80, 8), (2, 300, 1)])
def test_gpu_sphere_matches_oracle(O, gpu, I, J, M):
    x = _spec(I, J, M, 100 + M)
    Q, xw = gpu.sphere(x)
    Qo, xwo = O.sphere(x)
    assert np.max(np.abs(Q - Qo)) <= 1e-10 * np.max(np.abs(Qo))
    assert np.max(np.abs(xw - xwo)) <= 1e-10 * np.max(np.abs(xwo))
    for i in range(I):
        assert np.linalg.norm(_cov(xw[i]) - np.eye(M)) < 1e-6


def _sensitivity(O, x, K, iters, seed):
    """Largest relative response of the oracle's W, A, T, V to two independent
    1e-15 relative perturbations of x: ILRMA's IP / NMF sweeps amplify rounding
    noise (for some instances to ~1e-6 after 20 sweeps), so no two
    implementations that sum in different orders can agree more closely."""
    base = O.run_ilrma(x, K, iters, seed)
    ob = O.ilrma_objective(x, base[0], base[2], base[3])
    worst = dobj = 0.0
    for s in (1, 2):
        xp = x * (1 + 1e-15 * np.random.default_rng(s).standard_normal(x.shape))
        pert = O.run_ilrma(xp, K, iters, seed)
        for g, o in zip(pert, base):
            worst = max(worst, float(np.max(np.abs(g - o)) / np.max(np.abs(o))))
        dobj = max(dobj, abs(O.ilrma_objective(x, pert[0], pert[2], pert[3]) - ob))
    return worst, dobj


@pytest.mark.gpu
@pytest.mark.parametrize("I,J,M,K,iters", [(4, 50, 2, 4, 0), (6, 80, 3, 3, 10), (8, 64, 4, 10, 5),
                                           (8, 64, 4, 10, 20), (5, 40, 2, 2, 5), (4, 320, 8, 10, 10)])
def test_gpu_ilrma_matches_oracle(O, gpu, I, J, M, K, iters):
    """GPU run_ilrma against the oracle from the same seeded initialisation (30 NMF
    fitting passes, then `iters` NMF + IP sweeps): W, A, T, V within
    max(1e-8, 50 x the oracle's own response to rounding-level input noise)
    relative -- 1e-8 on well-conditioned instances; W A = I; the objective
    within max(1e-9 relative, 50 x its own rounding-noise response)."""
    _, x = O.sphere(_spec(I, J, M, 7 * I + M))
    W, A, T, V = gpu.run_ilrma(x, K, iters, 11)
    Wo, Ao, To, Vo = O.run_ilrma(x, K, iters, 11)
    sens, dobj = _sensitivity(O, x, K, iters, 11)
    bar = max(1e-8, 50.0 * sens)
    rel = lambda g, o: float(np.max(np.abs(g - o)) / np.max(np.abs(o)))
    errs = [rel(W, Wo), rel(A, Ao), rel(T, To), rel(V, Vo)]
    assert max(errs) <= bar, (errs, bar)
    assert np.all(np.linalg.norm(W @ A - np.eye(M), axis=(1, 2)) < 1e-8)
    og, oo = O.ilrma_objective(x, W, T, V), O.ilrma_objective(x, Wo, To, Vo)
    assert abs(og - oo) <= max(1e-9 * abs(oo), 50.0 * dobj), (og, oo, dobj)


@pytest.mark.gpu
def test_gpu_ilrma_reference_cases(O, gpu):
    """test_ilrma.cpp:91-154 on the GPU: W = I at iters = 0, deterministic, the
    objective non-increasing over growing iteration counts, validation errors."""
    from paper_1908_01964_b200 import InvalidInputError

    W, A, T, V = gpu.run_ilrma(_spec(4, 50, 2, 5), 4, 0, 7)
    assert np.all(np.linalg.norm(W - np.eye(2), axis=(1, 2)) < 1e-12) and T.min() >= 0 and V.min() >= 0
    x = _spec(6, 80, 3, 6)
    a, b = gpu.run_ilrma(x, 3, 10, 11), gpu.run_ilrma(x, 3, 10, 11)
    assert all(np.array_equal(u, v) for u, v in zip(a, b))
    x = _spec(6, 60, 2, 9)
    prev = np.inf
    for iters in (1, 3, 6, 10, 20):
        W, A, T, V = gpu.run_ilrma(x, 4, iters, 21)
        obj = O.ilrma_objective(x, W, T, V)
        assert obj <= prev + 1e-7 * abs(prev)
        prev = obj
    with pytest.raises(InvalidInputError, match="K must be >= 1"):
        gpu.run_ilrma(x, 0, 5, 1)
    with pytest.raises(InvalidInputError, match="iters must be >= 0"):
        gpu.run_ilrma(x, 2, -1, 1)
    with pytest.raises(InvalidInputError, match="need more frames"):
        gpu.sphere(_spec(2, 3, 3, 4))
