"""ctypes front-end of the CPU ORACLE (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this module, and only as the checker: the product package
``paper_1908_01964_b200`` never imports it.

Python-side arrays use natural numpy shapes; conversion to the reference's
Eigen column-major layout happens here (see rcscm_oracle.h):
  X, image, noise : (I, J, M) complex128      a, b : (I, M) complex128
  Rp, Rpp, W, A   : (I, M, M) complex128 [r, c]
  r_h, r_u        : (I, J) float64            lambda : (I,) float64
  T : (I, K)  V : (K, J)                      dry, sigma_bx, tau_ax : (I, J) complex128
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "librcscm_oracle.so")

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_i64 = ctypes.c_int64


class InvalidInputError(ValueError):
    """Mirror of rcscm::InvalidInputError (types.hpp:20-23)."""


class NumericalError(RuntimeError):
    """Mirror of rcscm::NumericalError (types.hpp:27-30)."""


class OracleSolverOpts(ctypes.Structure):
    _fields_ = [
        ("iters", ctypes.c_int),
        ("compute_objective", ctypes.c_int),
        ("record_trajectory", ctypes.c_int),
        ("rel_obj_tol", ctypes.c_double),
        ("threads", ctypes.c_int),
        ("eps_var", ctypes.c_double),
        ("gamma_fault", ctypes.c_double),
    ]


def build(force: bool = False) -> str:
    """Compile librcscm_oracle.so with the committed Makefile."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
        os.path.getmtime(os.path.join(_HERE, f)) for f in ("rcscm_oracle.cpp", "rcscm_oracle.h")
    ):
        subprocess.run(["make", "-C", _HERE, "-B" if force else "all"], check=True,
                       stdout=subprocess.DEVNULL)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = ctypes.CDLL(_LIB_PATH)
        _lib.oracle_last_error.restype = ctypes.c_char_p
        _lib.oracle_trajectory_distance.restype = ctypes.c_double
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().oracle_last_error().decode()
    if rc == 2:
        raise InvalidInputError(msg)
    if rc == 3:
        raise NumericalError(msg)
    raise RuntimeError(f"oracle error {rc}: {msg}")


# ---- layout helpers -------------------------------------------------------
def _p(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def mats_to_ref(m: np.ndarray) -> np.ndarray:
    """(I, M, M) natural [r, c] -> contiguous per-bin column-major buffer."""
    return np.ascontiguousarray(np.asarray(m, dtype=np.complex128).transpose(0, 2, 1))


def mats_from_ref(buf: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(buf.transpose(0, 2, 1))


def ij_to_ref(a: np.ndarray, dtype=np.float64) -> np.ndarray:
    """(I, J) -> Eigen column-major I x J buffer (element (i, t) at i + t*I)."""
    return np.ascontiguousarray(np.asarray(a, dtype=dtype).T)


def ij_from_ref(buf: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(buf.T)


def _c(a, dtype=np.complex128):
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


# ---- data types mirroring model.hpp ---------------------------------------
@dataclass
class Inputs:
    """model.hpp:16-25 RcscmInputs (natural numpy shapes)."""
    a: np.ndarray
    R_prime: np.ndarray
    R_prime_pinv: np.ndarray
    b: np.ndarray
    n_h: int = 0

    @property
    def num_bins(self):
        return self.a.shape[0]

    @property
    def mics(self):
        return self.a.shape[1]


@dataclass
class Params:
    """model.hpp:29-33 RcscmParams."""
    r_h: np.ndarray
    r_u: np.ndarray
    lam: np.ndarray

    def copy(self):
        return Params(self.r_h.copy(), self.r_u.copy(), self.lam.copy())


@dataclass
class SolverOptions:
    """solver_naive.hpp:14-22."""
    iters: int = 200
    compute_objective: bool = False
    record_trajectory: bool = False
    rel_obj_tol: float = 0.0
    threads: int = 1
    eps_var: float = 1e-12
    gamma_fault: float = 0.0


@dataclass
class SolverResult:
    """solver_naive.hpp:24-29."""
    params: Params
    objective: list = field(default_factory=list)
    iter_seconds: list = field(default_factory=list)
    trajectory: list = field(default_factory=list)


# ---- linalg.hpp -----------------------------------------------------------
def hermitian_eig(H):
    H = np.asarray(H, dtype=np.complex128)
    M = H.shape[0]
    vals = np.zeros(M)
    vecs = np.zeros((M, M), dtype=np.complex128)
    _check(lib().oracle_hermitian_eig(M, _p(_c(H.T)), _p(vals), _p(vecs)))
    return vals, vecs.T.copy()


def pseudo_inverse_psd(H, rank_tol=1e-10):
    H = np.asarray(H, dtype=np.complex128)
    M = H.shape[0]
    out = np.zeros((M, M), dtype=np.complex128)
    _check(lib().oracle_pseudo_inverse_psd(M, _p(_c(H.T)), ctypes.c_double(rank_tol), _p(out)))
    return out.T.copy()


def null_eigenvector(H, rank_tol=1e-10):
    H = np.asarray(H, dtype=np.complex128)
    M = H.shape[0]
    out = np.zeros(M, dtype=np.complex128)
    _check(lib().oracle_null_eigenvector(M, _p(_c(H.T)), ctypes.c_double(rank_tol), _p(out)))
    return out


def normalize_phase(v):
    v = _c(v)
    out = np.zeros_like(v)
    _check(lib().oracle_normalize_phase(v.shape[0], _p(v), _p(out)))
    return out


def sherman_morrison_inverse(Rinv, a, c, d):
    Rinv = np.asarray(Rinv, dtype=np.complex128)
    M = Rinv.shape[0]
    out = np.zeros((M, M), dtype=np.complex128)
    _check(lib().oracle_sherman_morrison_inverse(M, _p(_c(Rinv.T)), _p(_c(a)), ctypes.c_double(c),
                                                 ctypes.c_double(d), _p(out)))
    return out.T.copy()


def rank_one_restored_inverse(Rpp, b, lam):
    Rpp = np.asarray(Rpp, dtype=np.complex128)
    M = Rpp.shape[0]
    out = np.zeros((M, M), dtype=np.complex128)
    _check(lib().oracle_rank_one_restored_inverse(M, _p(_c(Rpp.T)), _p(_c(b)), ctypes.c_double(lam),
                                                  _p(out)))
    return out.T.copy()


def hermitian_pd_inverse(R):
    """solver_naive.hpp:46-146 (S = 2, 3, 4 closed form; LLT otherwise)."""
    R = np.asarray(R, dtype=np.complex128)
    M = R.shape[0]
    out = np.zeros((M, M), dtype=np.complex128)
    _check(lib().oracle_hermitian_pd_inverse(M, _p(_c(R.T)), _p(out)))
    return out.T.copy()


# ---- model.hpp ------------------------------------------------------------
def build_noise_scm(W, A, X, n_h, rank_tol=1e-10) -> Inputs:
    X = _c(X)
    I, J, M = X.shape
    a = np.zeros((I, M), np.complex128)
    b = np.zeros((I, M), np.complex128)
    Rp = np.zeros((I, M, M), np.complex128)
    Rpp = np.zeros((I, M, M), np.complex128)
    _check(lib().oracle_build_noise_scm(_i64(I), _i64(J), M, _p(X), _p(mats_to_ref(W)), _p(mats_to_ref(A)),
                                        int(n_h), ctypes.c_double(rank_tol), _p(a), _p(Rp), _p(Rpp), _p(b)))
    return Inputs(a, mats_from_ref(Rp), mats_from_ref(Rpp), b, int(n_h))


def init_params(inputs: Inputs, T, V, W, A, X) -> Params:
    X = _c(X)
    I, J, M = X.shape
    T = np.asarray(T, np.float64)
    V = np.asarray(V, np.float64)
    K = T.shape[1]
    r_h = np.zeros(I * J)
    r_u = np.zeros(I * J)
    lam = np.zeros(I)
    _check(lib().oracle_init_params(_i64(I), _i64(J), M, K, _p(X), _p(mats_to_ref(W)), _p(mats_to_ref(A)),
                                    int(inputs.n_h), _p(mats_to_ref(inputs.R_prime)),
                                    _p(mats_to_ref(inputs.R_prime_pinv)), _p(ij_to_ref(T)), _p(ij_to_ref(V)),
                                    _p(r_h), _p(r_u), _p(lam)))
    return Params(r_h.reshape(J, I).T.copy(), r_u.reshape(J, I).T.copy(), lam)


def map_objective(inputs: Inputs, p: Params, X, alpha=1.1, beta=1e-16) -> float:
    X = _c(X)
    I, J, M = X.shape
    out = ctypes.c_double(0.0)
    _check(lib().oracle_map_objective(_i64(I), _i64(J), M, _p(_c(inputs.a)), _p(mats_to_ref(inputs.R_prime)),
                                      _p(_c(inputs.b)), _p(ij_to_ref(p.r_h)), _p(ij_to_ref(p.r_u)),
                                      _p(_c(p.lam, np.float64)), ctypes.c_double(alpha), ctypes.c_double(beta),
                                      _p(X), ctypes.byref(out)))
    return out.value


# ---- solver_accel.hpp -----------------------------------------------------
@dataclass
class Scratch:
    sigma_ab: np.ndarray
    sigma_bx: np.ndarray
    tau_aa: np.ndarray
    tau_ax: np.ndarray
    tau_xx: np.ndarray


def precompute(inputs: Inputs, X) -> Scratch:
    X = _c(X)
    I, J, M = X.shape
    sab = np.zeros(I, np.complex128)
    sbx = np.zeros(I * J, np.complex128)
    taa = np.zeros(I)
    tax = np.zeros(I * J, np.complex128)
    txx = np.zeros(I * J)
    _check(lib().oracle_precompute(_i64(I), _i64(J), M, _p(_c(inputs.a)), _p(mats_to_ref(inputs.R_prime_pinv)),
                                   _p(_c(inputs.b)), _p(X), _p(sab), _p(sbx), _p(taa), _p(tax), _p(txx)))
    f = lambda v: v.reshape(J, I).T.copy()
    return Scratch(sab, f(sbx), taa, f(tax), f(txx))


def compute_gamma(r_h, r_u, trho_aa):
    I, J = r_h.shape
    g = np.zeros(I * J)
    _check(lib().oracle_compute_gamma(_i64(I), _i64(J), _p(ij_to_ref(r_h)), _p(ij_to_ref(r_u)),
                                      _p(_c(trho_aa, np.float64)), _p(g)))
    return g.reshape(J, I).T.copy()


def rho_first_stage(inputs: Inputs, X, lam, want_xx=True):
    X = _c(X)
    I, J, M = X.shape
    raa = np.zeros(I)
    rax = np.zeros(I * J, np.complex128)
    rxx = np.zeros(I * J) if want_xx else None
    _check(lib().oracle_rho_first_stage(_i64(I), _i64(J), M, _p(mats_to_ref(inputs.R_prime)), _p(_c(inputs.a)),
                                        _p(_c(inputs.b)), _p(X), _p(_c(lam, np.float64)), _p(raa), _p(rax),
                                        _p(rxx)))
    f = lambda v: None if v is None else v.reshape(J, I).T.copy()
    return raa, f(rax), f(rxx)


def rho_second_stage(s: Scratch, lam, want_xx=True):
    I, J = s.sigma_bx.shape
    raa = np.zeros(I)
    rax = np.zeros(I * J, np.complex128)
    rxx = np.zeros(I * J) if want_xx else None
    _check(lib().oracle_rho_second_stage(_i64(I), _i64(J), _p(_c(s.sigma_ab)), _p(ij_to_ref(s.sigma_bx, np.complex128)),
                                         _p(_c(s.tau_aa, np.float64)), _p(ij_to_ref(s.tau_ax, np.complex128)),
                                         _p(ij_to_ref(s.tau_xx)), _p(_c(lam, np.float64)), _p(raa), _p(rax),
                                         _p(rxx)))
    f = lambda v: None if v is None else v.reshape(J, I).T.copy()
    return raa, f(rax), f(rxx)


def update_rh(gamma, r_u, trho_ax, alpha=1.1, beta=1e-16, eps=1e-12):
    I, J = gamma.shape
    out = np.zeros(I * J)
    _check(lib().oracle_update_rh(_i64(I), _i64(J), _p(ij_to_ref(gamma)), _p(ij_to_ref(r_u)),
                                  _p(ij_to_ref(trho_ax, np.complex128)), ctypes.c_double(alpha),
                                  ctypes.c_double(beta), ctypes.c_double(eps), _p(out)))
    return out.reshape(J, I).T.copy()


def update_lambda(gamma, r_u, sigma_ab, sigma_bx, trho_ax, eps=1e-12):
    I, J = gamma.shape
    out = np.zeros(I)
    _check(lib().oracle_update_lambda(_i64(I), _i64(J), _p(ij_to_ref(gamma)), _p(ij_to_ref(r_u)),
                                      _p(_c(sigma_ab)), _p(ij_to_ref(sigma_bx, np.complex128)),
                                      _p(ij_to_ref(trho_ax, np.complex128)), ctypes.c_double(eps), _p(out)))
    return out


def update_ru(gamma, r_u, rho_aa, rho_ax, trho_ax, rho_xx, M, eps=1e-12):
    I, J = gamma.shape
    out = np.zeros(I * J)
    _check(lib().oracle_update_ru(_i64(I), _i64(J), int(M), _p(ij_to_ref(gamma)), _p(ij_to_ref(r_u)),
                                  _p(_c(rho_aa, np.float64)), _p(ij_to_ref(rho_ax, np.complex128)),
                                  _p(ij_to_ref(trho_ax, np.complex128)), _p(ij_to_ref(rho_xx)),
                                  ctypes.c_double(eps), _p(out)))
    return out.reshape(J, I).T.copy()


# ---- solver_naive.hpp -----------------------------------------------------
def e_step(inputs: Inputs, p: Params, X):
    X = _c(X)
    I, J, M = X.shape
    hr = np.zeros(I * J)
    hu = np.zeros((I, J, M, M), np.complex128)
    _check(lib().oracle_e_step(_i64(I), _i64(J), M, _p(_c(inputs.a)), _p(mats_to_ref(inputs.R_prime)),
                               _p(_c(inputs.b)), _p(ij_to_ref(p.r_h)), _p(ij_to_ref(p.r_u)),
                               _p(_c(p.lam, np.float64)), _p(X), _p(hr), _p(hu)))
    return hr.reshape(J, I).T.copy(), hu.transpose(0, 1, 3, 2).copy()


def m_step(hat_r_h, hat_R_u, inputs: Inputs, p_old: Params, alpha=1.1, beta=1e-16, eps=1e-12) -> Params:
    I, J = hat_r_h.shape
    M = inputs.mics
    r_h = np.zeros(I * J)
    r_u = np.zeros(I * J)
    lam = np.zeros(I)
    hu = np.ascontiguousarray(np.asarray(hat_R_u, np.complex128).transpose(0, 1, 3, 2))
    _check(lib().oracle_m_step(_i64(I), _i64(J), M, _p(ij_to_ref(hat_r_h)), _p(hu), _p(mats_to_ref(inputs.R_prime)),
                               _p(_c(inputs.b)), _p(ij_to_ref(p_old.r_u)), ctypes.c_double(alpha),
                               ctypes.c_double(beta), ctypes.c_double(eps), _p(r_h), _p(r_u), _p(lam)))
    return Params(r_h.reshape(J, I).T.copy(), r_u.reshape(J, I).T.copy(), lam)


# ---- drivers ----------------------------------------------------------------
BACKENDS = {"naive": 0, "accel1": 1, "accel2": 2, "accel2_binparallel": 3}


def run(backend: str, inputs: Inputs, params0: Params, X, opt: SolverOptions = None,
        alpha=1.1, beta=1e-16) -> SolverResult:
    """run_naive / run_algorithm1 / run_algorithm2 (solver_naive.hpp:412,
    solver_accel.hpp:246,254)."""
    opt = opt or SolverOptions()
    X = _c(X)
    I, J, M = X.shape
    o = OracleSolverOpts(int(opt.iters), int(opt.compute_objective), int(opt.record_trajectory),
                         float(opt.rel_obj_tol), int(opt.threads), float(opt.eps_var), float(opt.gamma_fault))
    n = max(int(opt.iters), 0)
    r_h = np.zeros(I * J)
    r_u = np.zeros(I * J)
    lam = np.zeros(I)
    obj = np.zeros(n + 1)
    secs = np.zeros(max(n, 1))
    n_obj = ctypes.c_int(0)
    n_it = ctypes.c_int(0)
    traj = opt.record_trajectory
    th = np.zeros(n * I * J) if traj else None
    tu = np.zeros(n * I * J) if traj else None
    tl = np.zeros(n * I) if traj else None
    _check(lib().oracle_run(BACKENDS[backend], _i64(I), _i64(J), M, _p(_c(inputs.a)),
                            _p(mats_to_ref(inputs.R_prime)), _p(mats_to_ref(inputs.R_prime_pinv)),
                            _p(_c(inputs.b)), _p(ij_to_ref(params0.r_h)), _p(ij_to_ref(params0.r_u)),
                            _p(_c(params0.lam, np.float64)), ctypes.c_double(alpha), ctypes.c_double(beta),
                            _p(X), ctypes.byref(o), _p(r_h), _p(r_u), _p(lam), _p(obj), ctypes.byref(n_obj),
                            _p(secs), ctypes.byref(n_it), _p(th), _p(tu), _p(tl)))
    f = lambda v: v.reshape(J, I).T.copy()
    res = SolverResult(Params(f(r_h), f(r_u), lam), list(obj[: n_obj.value]), list(secs[: n_it.value]))
    if traj:
        for k in range(n_it.value):
            res.trajectory.append(Params(f(th[k * I * J:(k + 1) * I * J]), f(tu[k * I * J:(k + 1) * I * J]),
                                         tl[k * I:(k + 1) * I].copy()))
    return res


def run_naive(inputs, params0, X, opt=None, **kw):
    return run("naive", inputs, params0, X, opt, **kw)


def run_algorithm1(inputs, params0, X, opt=None, **kw):
    return run("accel1", inputs, params0, X, opt, **kw)


def run_algorithm2(inputs, params0, X, opt=None, **kw):
    return run("accel2", inputs, params0, X, opt, **kw)


# ---- wiener.hpp -------------------------------------------------------------
def extract_target(inputs: Inputs, p: Params, X):
    X = _c(X)
    I, J, M = X.shape
    image = np.zeros((I, J, M), np.complex128)
    dry = np.zeros(I * J, np.complex128)
    _check(lib().oracle_extract_target(_i64(I), _i64(J), M, _p(_c(inputs.a)), _p(mats_to_ref(inputs.R_prime_pinv)),
                                       _p(_c(inputs.b)), _p(ij_to_ref(p.r_h)), _p(ij_to_ref(p.r_u)),
                                       _p(_c(p.lam, np.float64)), _p(X), _p(image), _p(dry)))
    return image, dry.reshape(J, I).T.copy()


def extract_noise(inputs: Inputs, p: Params, X):
    X = _c(X)
    I, J, M = X.shape
    noise = np.zeros((I, J, M), np.complex128)
    _check(lib().oracle_extract_noise(_i64(I), _i64(J), M, _p(_c(inputs.a)), _p(mats_to_ref(inputs.R_prime_pinv)),
                                      _p(_c(inputs.b)), _p(ij_to_ref(p.r_h)), _p(ij_to_ref(p.r_u)),
                                      _p(_c(p.lam, np.float64)), _p(X), _p(noise)))
    return noise


# ---- ilrma.hpp --------------------------------------------------------------
def sphere(X):
    """ilrma.hpp:53-73 -> (Q (I, M, M), whitened X (I, J, M))."""
    X = _c(X)
    I, J, M = X.shape
    Q = np.zeros((I, M, M), np.complex128)
    Xw = np.zeros_like(X)
    _check(lib().oracle_sphere(_i64(I), _i64(J), M, _p(X), _p(Q), _p(Xw)))
    return mats_from_ref(Q), Xw


def run_ilrma(X, K: int, iters: int, seed: int):
    """ilrma.hpp:145-240 -> (W (I, M, M), A (I, M, M), T (M, I, K), V (M, K, J))."""
    X = _c(X)
    I, J, M = X.shape
    W = np.zeros((I, M, M), np.complex128)
    A = np.zeros((I, M, M), np.complex128)
    T = np.zeros(M * I * K)
    V = np.zeros(M * K * J)
    _check(lib().oracle_run_ilrma(_i64(I), _i64(J), M, int(K), int(iters), ctypes.c_uint64(seed), _p(X), _p(W),
                                  _p(A), _p(T), _p(V)))
    Tn = T.reshape(M, K, I).transpose(0, 2, 1).copy()  # [n] I x K col-major
    Vn = V.reshape(M, J, K).transpose(0, 2, 1).copy()  # [n] K x J col-major
    return mats_from_ref(W), mats_from_ref(A), Tn, Vn


def ilrma_objective(X, W, T, V) -> float:
    """ilrma.hpp:86-98."""
    X = _c(X)
    I, J, M = X.shape
    K = T.shape[2]
    Tr = np.ascontiguousarray(np.asarray(T, np.float64).transpose(0, 2, 1)).ravel()
    Vr = np.ascontiguousarray(np.asarray(V, np.float64).transpose(0, 2, 1)).ravel()
    out = ctypes.c_double()
    _check(lib().oracle_ilrma_objective(_i64(I), _i64(J), M, int(K), _p(X), _p(mats_to_ref(_c(W))), _p(Tr), _p(Vr),
                                        ctypes.byref(out)))
    return out.value


# ---- stft.hpp (numpy restatement; the DFT is numpy's pocketfft) --------------
def hamming_window(n: int) -> np.ndarray:
    """stft.hpp:12-17: periodic Hamming, 0.54 - 0.46 cos(2 pi k / n)."""
    return np.array([0.54 - 0.46 * np.cos(2.0 * np.pi * k / n) for k in range(n)])


def wola_dual_window(win: np.ndarray, hop: int) -> np.ndarray:
    """stft.hpp:22-29: d[k] = w[k] / sum of w^2 hitting k modulo hop."""
    n = len(win)
    denom = np.zeros(hop)
    for k in range(n):
        denom[k % hop] += win[k] * win[k]
    return np.array([win[k] / denom[k % hop] for k in range(n)])


def stft_params(sample_rate: float, win_ms: float, hop_ms: float):
    """stft.hpp:37-46 (std::lround: half away from zero)."""
    if not (win_ms > hop_ms and hop_ms > 0):
        raise InvalidInputError("stft: require win_ms > hop_ms > 0")
    rnd = lambda v: int(np.floor(abs(v) + 0.5)) * (1 if v >= 0 else -1)
    win, hop = rnd(win_ms * 1e-3 * sample_rate), rnd(hop_ms * 1e-3 * sample_rate)
    if win < 2 or hop < 1:
        raise InvalidInputError("stft: window shorter than 2 samples")
    return win, hop


def stft_analyze(samples, sample_rate: float, win_ms: float, hop_ms: float):
    """stft.hpp:50-88. samples (M, len) -> (X (I, J, M) complex, win, hop)."""
    x = np.asarray(samples, np.float64)
    if x.ndim != 2 or x.shape[0] == 0 or x.shape[1] == 0:
        raise InvalidInputError("stft_analyze: empty waveform")
    win, hop = stft_params(sample_rate, win_ms, hop_ms)
    M, n = x.shape
    pad = win - hop
    J = (n + pad + hop - 1) // hop
    w = hamming_window(win)
    X = np.zeros((win // 2 + 1, J, M), np.complex128)
    for ch in range(M):
        for j in range(J):
            start = j * hop - pad
            frame = np.zeros(win)
            lo, hi = max(start, 0), min(start + win, n)
            if hi > lo:
                frame[lo - start:hi - start] = x[ch, lo:hi] * w[lo - start:hi - start]
            X[:, j, ch] = np.fft.rfft(frame)
    return X, win, hop


def stft_synthesize(X, sample_rate: float, win_ms: float, hop_ms: float, win_samples: int, hop_samples: int,
                    source_samples: int = 0):
    """stft.hpp:92-129 (weighted overlap-add with the dual window, frames in order)."""
    X = _c(X)
    if X.shape[0] == 0:
        raise InvalidInputError("stft_synthesize: empty spectrogram")
    win, hop = stft_params(sample_rate, win_ms, hop_ms)
    if win != win_samples or hop != hop_samples:
        raise InvalidInputError("stft_synthesize: window/hop do not match analysis")
    if X.shape[0] != win // 2 + 1:
        raise InvalidInputError("stft_synthesize: bin count inconsistent with window")
    _, J, M = X.shape
    pad = win - hop
    n = source_samples if source_samples > 0 else J * hop - pad
    dual = wola_dual_window(hamming_window(win), hop)
    out = np.zeros((M, n))
    for ch in range(M):
        for j in range(J):
            frame = np.fft.irfft(X[:, j, ch], n=win)
            start = j * hop - pad
            lo, hi = max(start, 0), min(start + win, n)
            if hi > lo:
                out[ch, lo:hi] += frame[lo - start:hi - start] * dual[lo - start:hi - start]
    return out


# ---- verify.hpp -------------------------------------------------------------
def make_verify_instance(I, J, M, seed):
    X = np.zeros((I, J, M), np.complex128)
    a = np.zeros((I, M), np.complex128)
    b = np.zeros((I, M), np.complex128)
    Rp = np.zeros((I, M, M), np.complex128)
    Rpp = np.zeros((I, M, M), np.complex128)
    r_h = np.zeros(I * J)
    r_u = np.zeros(I * J)
    lam = np.zeros(I)
    _check(lib().oracle_make_verify_instance(_i64(I), _i64(J), M, ctypes.c_uint64(seed), _p(X), _p(a), _p(Rp),
                                             _p(Rpp), _p(b), _p(r_h), _p(r_u), _p(lam)))
    f = lambda v: v.reshape(J, I).T.copy()
    return Inputs(a, mats_from_ref(Rp), mats_from_ref(Rpp), b, 0), Params(f(r_h), f(r_u), lam), X


def trajectory_distance(p: Params, q: Params) -> float:
    """verify.hpp:60-68: max elementwise |x-y| / max(|x|, |y|, 1e-12)."""
    def d(x, y):
        x = np.asarray(x, np.float64)
        y = np.asarray(y, np.float64)
        den = np.maximum(np.maximum(np.abs(x), np.abs(y)), 1e-12)
        return float(np.max(np.abs(x - y) / den)) if x.size else 0.0
    return max(d(p.r_h, q.r_h), d(p.r_u, q.r_u), d(p.lam, q.lam))


# ---- binary128 ground truth (truth.cpp) ---------------------------------------
_TRUTH_PATH = os.path.join(_HERE, "librcscm_truth.so")
_tlib = None


def truth_lib():
    """librcscm_truth.so: one iteration of Algorithm 2 / the naive rule and the
    Wiener dry output evaluated in IEEE binary128 on the same double inputs
    (test infrastructure: the yardstick both double implementations -- this
    oracle and the CUDA path -- are measured against)."""
    global _tlib
    if _tlib is None:
        if not os.path.exists(_TRUTH_PATH) or os.path.getmtime(_TRUTH_PATH) < os.path.getmtime(
                os.path.join(_HERE, "truth.cpp")):
            subprocess.run(["make", "-C", _HERE, "librcscm_truth.so"], check=True, stdout=subprocess.DEVNULL)
        _tlib = ctypes.CDLL(_TRUTH_PATH)
    return _tlib


def truth_accel_one_iter(inputs: Inputs, params0: Params, X, alpha=1.1, beta=1e-16, eps=1e-12):
    """-> (Params after one Algorithm 2 iteration in binary128 rounded to
    double, Params of the first-order rounding scales B (r_h, r_u per slot,
    lambda per bin): a double evaluation of the same formulas is expected
    within C eps B of the truth, see truth.cpp)."""
    X = _c(X)
    I, J, M = X.shape
    r_h, r_u, lam = np.zeros(I * J), np.zeros(I * J), np.zeros(I)
    Bh, Bu, Bl = np.zeros(I * J), np.zeros(I * J), np.zeros(I)
    rc = truth_lib().truth_accel_one_iter(
        _i64(I), _i64(J), M, _p(_c(inputs.a)), _p(mats_to_ref(inputs.R_prime_pinv)), _p(_c(inputs.b)),
        _p(ij_to_ref(params0.r_h)), _p(ij_to_ref(params0.r_u)), _p(_c(params0.lam, np.float64)),
        ctypes.c_double(alpha), ctypes.c_double(beta), ctypes.c_double(eps), _p(X), _p(r_h), _p(r_u), _p(lam),
        _p(Bh), _p(Bu), _p(Bl))
    if rc:
        raise NumericalError("truth_accel_one_iter failed")
    f = lambda v: v.reshape(J, I).T.copy()
    return Params(f(r_h), f(r_u), lam), Params(f(Bh), f(Bu), Bl)


def truth_naive_one_iter(inputs: Inputs, params0: Params, X, alpha=1.1, beta=1e-16, eps=1e-12):
    """-> (Params after one naive iteration (solver_naive.hpp:153-386) in
    binary128, Params of the rounding scales B incl. kappa(R_x), kappa(R_u))."""
    X = _c(X)
    I, J, M = X.shape
    r_h, r_u, lam = np.zeros(I * J), np.zeros(I * J), np.zeros(I)
    Bh, Bu, Bl = np.zeros(I * J), np.zeros(I * J), np.zeros(I)
    rc = truth_lib().truth_naive_one_iter(
        _i64(I), _i64(J), M, _p(_c(inputs.a)), _p(mats_to_ref(inputs.R_prime)), _p(_c(inputs.b)),
        _p(ij_to_ref(params0.r_h)), _p(ij_to_ref(params0.r_u)), _p(_c(params0.lam, np.float64)),
        ctypes.c_double(alpha), ctypes.c_double(beta), ctypes.c_double(eps), _p(X), _p(r_h), _p(r_u), _p(lam),
        _p(Bh), _p(Bu), _p(Bl))
    if rc:
        raise NumericalError("truth_naive_one_iter: singular matrix")
    f = lambda v: v.reshape(J, I).T.copy()
    return Params(f(r_h), f(r_u), lam), Params(f(Bh), f(Bu), Bl)


def truth_wiener_dry(inputs: Inputs, p: Params, X):
    """-> dry (I, J) of extract_target (wiener.hpp:19-43) in binary128."""
    X = _c(X)
    I, J, M = X.shape
    dry = np.zeros(I * J, np.complex128)
    truth_lib().truth_wiener(_i64(I), _i64(J), M, _p(_c(inputs.a)), _p(mats_to_ref(inputs.R_prime_pinv)),
                             _p(_c(inputs.b)), _p(ij_to_ref(p.r_h)), _p(ij_to_ref(p.r_u)),
                             _p(_c(p.lam, np.float64)), _p(X), _p(dry))
    return dry.reshape(J, I).T.copy()
