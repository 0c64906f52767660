"""Oracle pins: ports of proj/tests/test_linalg.cpp:10-185 (known answers +
dense oracles) onto the oracle's restatement of linalg.hpp."""
import numpy as np
import pytest

from conftest import Rng, rel_error


def test_eig_identity_and_diagonal(O):  # test_linalg.cpp:10-24
    vals, vecs = O.hermitian_eig(np.eye(2))
    assert vals == pytest.approx([1.0, 1.0])
    assert rel_error(vecs @ vecs.conj().T, np.eye(2)) < 1e-12
    vals, vecs = O.hermitian_eig(np.diag([3.0, 1.0]))
    assert vals == pytest.approx([1.0, 3.0])
    assert abs(vecs[1, 0]) == pytest.approx(1.0)
    assert abs(vecs[0, 1]) == pytest.approx(1.0)


def test_eig_seeded_reconstruction(O):  # test_linalg.cpp:26-36
    h = Rng(42).hermitian_pd(4)
    vals, vecs = O.hermitian_eig(h)
    recon = (vecs * vals) @ vecs.conj().T
    assert rel_error(recon, h) < 1e-10
    assert np.linalg.norm(vecs.conj().T @ vecs - np.eye(4)) < 1e-10
    assert np.all(np.diff(vals) >= 0)
    # independent check against LAPACK
    assert np.max(np.abs(vals - np.linalg.eigvalsh(h))) < 1e-12 * np.max(np.abs(vals))


def test_eig_rejects_non_hermitian(O):  # test_linalg.cpp:38-43
    bad = np.array([[0, 1], [2, 0]], dtype=complex)
    with pytest.raises(O.InvalidInputError):
        O.hermitian_eig(bad)


def test_pinv_diagonal_rank_deficient(O):  # :45-51
    p = O.pseudo_inverse_psd(np.diag([2.0, 0.0]).astype(complex))
    assert abs(p[0, 0] - 0.5) < 1e-14
    assert abs(p[1, 1]) < 1e-14


def test_pinv_full_rank_is_inverse(O):  # :53-60
    h = Rng(7).hermitian_pd(4)
    p = O.pseudo_inverse_psd(h)
    assert rel_error(h @ p, np.eye(4)) < 1e-10
    assert rel_error(O.pseudo_inverse_psd(p), h) < 1e-8


def test_pinv_rank_one_projector(O):  # :62-68
    b = Rng(11).complex_vector(3)
    b /= np.linalg.norm(b)
    h = np.outer(b, b.conj())
    assert rel_error(O.pseudo_inverse_psd(h), h) < 1e-10


def test_pinv_h_hplus_h(O):  # :70-75
    h = Rng(13).rank_deficient_psd(5)
    p = O.pseudo_inverse_psd(h)
    assert rel_error(h @ p @ h, h) < 1e-9
    # dense LAPACK pinv as independent oracle
    assert rel_error(p, np.linalg.pinv(h, rcond=1e-10, hermitian=True)) < 1e-9


def test_pinv_rejects_indefinite(O):  # :77-81
    with pytest.raises(O.InvalidInputError):
        O.pseudo_inverse_psd(np.diag([1.0, -1.0]).astype(complex))


def test_null_vector_diagonal(O):  # :83-91
    b = O.null_eigenvector(np.diag([1.0, 2.0, 0.0]).astype(complex))
    assert abs(b[2] - 1.0) < 1e-12
    assert abs(b[0]) < 1e-12 and abs(b[1]) < 1e-12


def test_null_vector_known_eigenbasis(O):  # :93-105
    q, _ = np.linalg.qr(Rng(21).complex_matrix(3, 3))
    h = q @ np.diag([1.0, 2.0, 0.0]) @ q.conj().T
    b = O.null_eigenvector((h + h.conj().T) / 2)
    expected = O.normalize_phase(q[:, 2])
    assert np.linalg.norm(b - expected) < 1e-10
    assert abs(np.linalg.norm(b) - 1.0) < 1e-12


def test_normalize_phase_pivot_rule(O):  # linalg.hpp:58-70
    v = np.array([1e-12, 2j, 1 + 1j])
    w = O.normalize_phase(v)
    assert abs(w[1].imag) < 1e-15 and w[1].real > 0  # first entry above 1e-8 * max
    assert np.allclose(np.abs(w), np.abs(v))


def test_null_vector_two_zero_eigs_rejected(O):  # :107-112
    with pytest.raises(O.InvalidInputError):
        O.null_eigenvector(np.diag([1.0, 0.0, 0.0]).astype(complex))
    with pytest.raises(O.InvalidInputError):
        O.null_eigenvector(np.eye(3, dtype=complex))


def test_sherman_morrison_trivial(O):  # :114-129
    rng = Rng(31)
    r = rng.hermitian_pd(3)
    rinv = np.linalg.inv(r)
    a = rng.complex_vector(3)
    assert rel_error(O.sherman_morrison_inverse(rinv, a, 0.0, 2.0), 0.5 * rinv) < 1e-14
    assert abs(O.sherman_morrison_inverse(np.eye(1), np.ones(1), 1.0, 1.0)[0, 0] - 0.5) < 1e-14
    with pytest.raises(O.InvalidInputError):
        O.sherman_morrison_inverse(rinv, a, 1.0, 0.0)


@pytest.mark.parametrize("m", [2, 3, 4, 8])
def test_sherman_morrison_dense(O, m):  # :131-145
    for seed in range(5):
        rng = Rng(1000 * m + seed)
        r = rng.hermitian_pd(m)
        a = rng.complex_vector(m)
        c = 0.5 + abs(rng.real())
        d = 0.5 + abs(rng.real())
        direct = np.linalg.inv(c * np.outer(a, a.conj()) + d * r)
        assert rel_error(O.sherman_morrison_inverse(np.linalg.inv(r), a, c, d), direct) < 1e-9


def test_restored_inverse_diag_and_scalar(O):  # :147-162
    rp = np.diag([1.0, 0.0]).astype(complex)
    inv = O.rank_one_restored_inverse(O.pseudo_inverse_psd(rp), np.array([0, 1], complex), 2.0)
    assert abs(inv[0, 0] - 1.0) < 1e-14 and abs(inv[1, 1] - 0.5) < 1e-14
    assert abs(O.rank_one_restored_inverse(np.zeros((1, 1)), np.ones(1), 3.0)[0, 0] - 1 / 3) < 1e-14


def test_restored_inverse_dense(O):  # :164-175
    rp = Rng(57).rank_deficient_psd(4)
    pinv = O.pseudo_inverse_psd(rp)
    b = O.null_eigenvector(rp)
    for lam in (1e-6, 1e-2, 1.0, 1e3):
        inv = O.rank_one_restored_inverse(pinv, b, lam)
        assert rel_error(inv @ (rp + lam * np.outer(b, b.conj())), np.eye(4)) < 1e-8


def test_restored_inverse_preconditions(O):  # :177-185
    rng = Rng(58)
    rp = rng.rank_deficient_psd(3)
    pinv = O.pseudo_inverse_psd(rp)
    b = O.null_eigenvector(rp)
    with pytest.raises(O.InvalidInputError):
        O.rank_one_restored_inverse(pinv, b, 0.0)
    with pytest.raises(O.InvalidInputError):
        O.rank_one_restored_inverse(pinv, 2 * b, 1.0)
    out = rng.complex_vector(3)
    with pytest.raises(O.InvalidInputError):
        O.rank_one_restored_inverse(pinv, out / np.linalg.norm(out), 1.0)


@pytest.mark.parametrize("m", [2, 3, 4, 5, 8])
def test_hermitian_pd_inverse(O, m):  # solver_naive.hpp:46-146 closed forms / LLT
    r = Rng(90 + m).hermitian_pd(m)
    assert rel_error(O.hermitian_pd_inverse(r), np.linalg.inv(r)) < 1e-12
    with pytest.raises(O.NumericalError):
        O.hermitian_pd_inverse(-np.eye(m, dtype=complex))
