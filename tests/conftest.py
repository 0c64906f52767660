import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA) device; runs through the C ABI")


@pytest.fixture(scope="session")
def O():
    """The CPU oracle (test infrastructure; the checker, never the product)."""
    from oracle import oracle as mod

    mod.build()
    return mod


@pytest.fixture(scope="session")
def gpu():
    from paper_1908_01964_b200 import GpuContext

    return GpuContext(0)


def rel_error(a, b):
    """test_util.hpp:42-48: ||a - b|| / max(||a||, ||b||, 1e-300)."""
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(a), np.linalg.norm(b), 1e-300))


class Rng:
    """Stand-in for test_util.hpp:12-40 (numpy generator; seeds differ from the
    reference's mt19937_64 but the structure of each draw is the same)."""

    def __init__(self, seed):
        self.g = np.random.default_rng(seed)

    def real(self):
        return float(self.g.standard_normal())

    def complex_vector(self, n):
        return self.g.standard_normal(n) + 1j * self.g.standard_normal(n)

    def complex_matrix(self, r, c):
        return self.g.standard_normal((r, c)) + 1j * self.g.standard_normal((r, c))

    def hermitian_pd(self, n):
        g = self.complex_matrix(n, n)
        return g @ g.conj().T + 0.1 * np.eye(n)

    def rank_deficient_psd(self, n):
        g = self.complex_matrix(n, n - 1)
        r = g @ g.conj().T
        return (r + r.conj().T) / 2


def random_spectrogram(I, J, M, seed):
    return Rng(seed).complex_matrix(I * J, M).reshape(I, J, M)


def random_demixing(I, M, seed):
    """test_model.cpp:23-32: complex Gaussian + 2 I, A = W^{-1}."""
    rng = Rng(seed)
    W = np.stack([rng.complex_matrix(M, M) + 2 * np.eye(M) for _ in range(I)])
    return W, np.linalg.inv(W)
