"""Seeded synthetic STFT-domain inputs for BASELINE.json's configs.

The reference's experiments use the JNAS corpus and measured room responses
(PAPER.md:431-442), which are not available here; BASELINE.json defines an
STFT-domain recipe instead, restated from SURVEY.md section 8(d):

  W_i = G + c I (G complex Gaussian, c = M; "2 I" for M = 2), A_i = W_i^{-1}, a_i = A_i[:, 0], n_h = 0
  target  s_ij ~ CN(0, v_ij),  v_ij = sum_k t_ik v_kj,  t, v ~ Gamma(0.5, 1), K = 4
  noise   n_ij = sigma_ij C_i^{1/2} z_ij,  sigma^2 ~ Gamma(1, 1),  z ~ CN(0, I_M),
          C_i[m, n] = sin(k)/k,  k = 2 pi f_i |m - n| d / c  (value 1 at k = 0),
          f_i = i * 8000 / (I - 1) Hz, c = 343 m/s, C^{1/2} by clamped eigendecomposition
  mix     x_ij = a_i s_ij + g n_ij, g such that sum ||a s||^2 = sum ||g n||^2 (0 dB broadband,
          the convention of synth.hpp:156-161)
Initialisation then follows the reference: build_noise_scm(W, A, x, n_h = 0) and
init_params with NmfModel T[0] = t, V[0] = v (model.hpp:58-124).

Generation is host-side input preparation (numpy), not part of the measured path.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# BASELINE.json "configs" (index -> recipe); iters are the accel / naive counts.
CONFIGS = {
    0: dict(name="c0_m2_i513_j320", M=2, I=513, J=320, B=1, d=0.05, iters=100, naive_iters=100),
    1: dict(name="c1_m4_i1025_j640", M=4, I=1025, J=640, B=1, d=0.05, iters=100, naive_iters=100),
    2: dict(name="c2_m2_i513_j20000", M=2, I=513, J=20000, B=1, d=0.05, iters=50, naive_iters=0),
    3: dict(name="c3_b256_m4_i513_j320", M=4, I=513, J=320, B=256, d=0.05, iters=100, naive_iters=100),
    4: dict(name="c4_m8_i2049_j4096", M=8, I=2049, J=4096, B=1, d=0.04, iters=100, naive_iters=10),
}


@dataclass
class Utterance:
    X: np.ndarray  # (I, J, M) complex128
    W: np.ndarray  # (I, M, M)
    A: np.ndarray  # (I, M, M)
    T: np.ndarray  # (I, K)
    V: np.ndarray  # (K, J)
    n_h: int = 0


def coherence_sqrt(M: int, I: int, d: float, c: float = 343.0) -> np.ndarray:
    """C_i^{1/2} for the spherically isotropic field, (I, M, M) real."""
    f = np.arange(I) * 8000.0 / max(I - 1, 1)
    dist = np.abs(np.arange(M)[:, None] - np.arange(M)[None, :]) * d
    k = 2.0 * np.pi * f[:, None, None] * dist[None] / c
    with np.errstate(invalid="ignore", divide="ignore"):
        C = np.where(k == 0.0, 1.0, np.sin(k) / np.where(k == 0.0, 1.0, k))
    w, U = np.linalg.eigh(C)
    w = np.sqrt(np.clip(w, 0.0, None))
    return np.einsum("imk,ik,ink->imn", U, w, U)


def make_utterance(M: int, I: int, J: int, d: float, seed: int, K: int = 4) -> Utterance:
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((I, M, M)) + 1j * rng.standard_normal((I, M, M))
    W = G + M * np.eye(M)[None]
    A = np.linalg.inv(W)
    a = A[:, :, 0]
    t = rng.gamma(0.5, 1.0, size=(I, K))
    v = rng.gamma(0.5, 1.0, size=(K, J))
    var = t @ v
    s = np.sqrt(var / 2.0) * (rng.standard_normal((I, J)) + 1j * rng.standard_normal((I, J)))
    sig = np.sqrt(rng.gamma(1.0, 1.0, size=(I, J)))
    z = (rng.standard_normal((I, J, M)) + 1j * rng.standard_normal((I, J, M))) / np.sqrt(2.0)
    Ch = coherence_sqrt(M, I, d)
    n = sig[:, :, None] * np.einsum("imn,ijn->ijm", Ch, z)
    img = a[:, None, :] * s[:, :, None]
    g = np.sqrt(np.sum(np.abs(img) ** 2) / np.sum(np.abs(n) ** 2))
    X = np.ascontiguousarray(img + g * n)
    return Utterance(X, np.ascontiguousarray(W), np.ascontiguousarray(A), t, v, 0)


def make_config(cfg: int, utterances: int = None, seed_base: int = None, I: int = None, J: int = None):
    """Utterances of BASELINE config `cfg` (seed = 1000 * cfg + u); I / J may be
    shrunk for parity tests that must also run on the CPU oracle."""
    c = CONFIGS[cfg]
    B = c["B"] if utterances is None else utterances
    base = 1000 * cfg if seed_base is None else seed_base
    return [make_utterance(c["M"], I or c["I"], J or c["J"], c["d"], base + u) for u in range(B)]


def stack(utts):
    """-> X (B, I, J, M), W, A (B, I, M, M), T (B, I, K), V (B, K, J)."""
    return (np.stack([u.X for u in utts]), np.stack([u.W for u in utts]), np.stack([u.A for u in utts]),
            np.stack([u.T for u in utts]), np.stack([u.V for u in utts]))
