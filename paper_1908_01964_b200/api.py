"""Python mirror of the reference's hot-path interface over the C ABI.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/rcscm/{model,solver_naive,solver_accel,wiener}.hpp:

  build_noise_scm(demix_W, demix_A, X, n_h, rank_tol)   model.hpp:58-90
  init_params(inputs, T, V, demix_W, demix_A, X)         model.hpp:95-124
  map_objective(inputs, params, hyper, X)                model.hpp:129-157
  run_naive(inputs, params0, hyper, X, opt)              solver_naive.hpp:412-450
  run_algorithm1(inputs, params0, hyper, X, opt)         solver_accel.hpp:245-250
  run_algorithm2(inputs, params0, hyper, X, opt)         solver_accel.hpp:254-258
  extract_target(inputs, params, X)                      wiener.hpp:19-43
  extract_noise(inputs, params, X)                       wiener.hpp:46-53

Errors raise InvalidInputError / NumericalError like the reference's
exceptions (types.hpp:20-30). Arrays use natural numpy shapes; conversion to
the reference's Eigen column-major buffers happens here, the numerics run in
librcscm_gpu.so on the GPU.

Shapes: X (I, J, M) complex128; a, b (I, M); R_prime, R_prime_pinv, W, A
(I, M, M) [r, c]; r_h, r_u (I, J); lam (I,); T (I, K); V (K, J).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi as C


class InvalidInputError(ValueError):
    """rcscm::InvalidInputError (types.hpp:20-23)."""


class NumericalError(RuntimeError):
    """rcscm::NumericalError (types.hpp:27-30)."""


class CudaError(RuntimeError):
    """CUDA runtime failure inside the C ABI."""


class UnsupportedError(NotImplementedError):
    """Shape / mode this build does not implement."""


def _raise(rc: int):
    if rc == C.RCSCM_OK:
        return
    msg = C.load().rcscm_gpu_last_error().decode()
    raise {C.RCSCM_INVALID_INPUT: InvalidInputError, C.RCSCM_NUMERICAL: NumericalError,
           C.RCSCM_UNSUPPORTED: UnsupportedError}.get(rc, CudaError)(msg)


def _p(a):
    return None if a is None else a.ctypes.data_as(C._dp)


def _cz(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def _mats(m):
    """(I, M, M) natural -> per-bin column-major buffer."""
    return np.ascontiguousarray(np.asarray(m, dtype=np.complex128).transpose(0, 2, 1))


def _ij(a, dtype=np.float64):
    """(I, J) -> Eigen column-major I x J buffer."""
    return np.ascontiguousarray(np.asarray(a, dtype=dtype).T)


def _from_ij(buf, I, J):
    return np.ascontiguousarray(buf.reshape(J, I).T)


@dataclass
class RcscmInputs:
    """model.hpp:16-25."""
    a: np.ndarray
    R_prime: np.ndarray
    R_prime_pinv: np.ndarray
    b: np.ndarray
    n_h: int = 0

    @property
    def num_bins(self) -> int:
        return int(self.a.shape[0])

    @property
    def mics(self) -> int:
        return int(self.a.shape[1])


@dataclass
class RcscmParams:
    """model.hpp:29-33."""
    r_h: np.ndarray
    r_u: np.ndarray
    lam: np.ndarray


@dataclass
class Hyperparams:
    """model.hpp:36-39."""
    alpha: float = 1.1
    beta: float = 1e-16


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
    params: RcscmParams
    objective: List[float] = field(default_factory=list)
    iter_seconds: List[float] = field(default_factory=list)
    trajectory: List[RcscmParams] = field(default_factory=list)


@dataclass
class ExtractionResult:
    """wiener.hpp:11-14: image (I, J, M) and dry (I, J)."""
    image: np.ndarray
    dry: np.ndarray


class _Held:
    """Keeps the numpy buffers behind a ctypes struct alive."""

    def __init__(self):
        self.refs = []

    def keep(self, a):
        self.refs.append(a)
        return a


def _c_inputs(inp: RcscmInputs, J: int, held: _Held) -> C.CInputs:
    I, M = inp.a.shape
    a = held.keep(_cz(inp.a))
    b = held.keep(_cz(inp.b))
    rp = held.keep(_mats(inp.R_prime)) if inp.R_prime is not None else None
    rpp = held.keep(_mats(inp.R_prime_pinv)) if inp.R_prime_pinv is not None else None
    return C.CInputs(I, J, M, int(inp.n_h), _p(a), _p(rp), _p(rpp), _p(b))


def _c_params_in(p: RcscmParams, held: _Held) -> C.CParams:
    rh = held.keep(_ij(p.r_h))
    ru = held.keep(_ij(p.r_u))
    lam = held.keep(np.ascontiguousarray(np.asarray(p.lam, dtype=np.float64)))
    return C.CParams(_p(rh), _p(ru), _p(lam))


class GpuContext:
    """One rcscm_gpu_ctx: one CUDA device and stream, or (devices=[...]) bins
    sharded over several devices, one stream and host thread each."""

    def __init__(self, device: int = 0, precision: str = "c128", stream: Optional[int] = None,
                 devices: Optional[List[int]] = None):
        lib = C.load()
        devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices]) if devices else None
        cfg = C.GpuConfig(int(devices[0]) if devices else int(device),
                          C.RCSCM_C128 if precision == "c128" else C.RCSCM_C64,
                          ctypes.c_void_p(stream) if stream else None, devs, len(devices) if devices else 0)
        self._devs = devs  # keep the list alive for the call
        h = ctypes.c_void_p()
        _raise(lib.rcscm_gpu_create(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        self._lib = lib

    def close(self):
        if getattr(self, "_h", None):
            self._lib.rcscm_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def launch_count(self) -> int:
        return int(self._lib.rcscm_gpu_launch_count(self._h))

    @property
    def stream(self) -> int:
        return int(self._lib.rcscm_gpu_stream(self._h) or 0)

    # ---- reference entry points ---------------------------------------------
    def build_noise_scm(self, W, A, X, n_h: int, rank_tol: float = 1e-10) -> RcscmInputs:
        X = _cz(X)
        I, J, M = X.shape
        a = np.zeros((I, M), np.complex128)
        b = np.zeros((I, M), np.complex128)
        rp = np.zeros((I, M, M), np.complex128)
        rpp = np.zeros((I, M, M), np.complex128)
        _raise(self._lib.rcscm_gpu_build_noise_scm(self._h, I, J, M, _p(X), _p(_mats(W)), _p(_mats(A)), int(n_h),
                                                   float(rank_tol), _p(a), _p(rp), _p(rpp), _p(b)))
        return RcscmInputs(a, rp.transpose(0, 2, 1).copy(), rpp.transpose(0, 2, 1).copy(), b, int(n_h))

    def init_params(self, inputs: RcscmInputs, T, V, W, A, X) -> RcscmParams:
        X = _cz(X)
        I, J, M = X.shape
        held = _Held()
        ci = _c_inputs(inputs, J, held)
        T = np.asarray(T, np.float64)
        V = np.asarray(V, np.float64)
        K = T.shape[1]
        rh = np.zeros(I * J)
        ru = np.zeros(I * J)
        lam = np.zeros(I)
        out = C.CParams(_p(rh), _p(ru), _p(lam))
        _raise(self._lib.rcscm_gpu_init_params(self._h, ctypes.byref(ci), K, _p(X), _p(_mats(W)), _p(_mats(A)),
                                               _p(_ij(T)), _p(_ij(V)), ctypes.byref(out)))
        return RcscmParams(_from_ij(rh, I, J), _from_ij(ru, I, J), lam)

    def map_objective(self, inputs: RcscmInputs, p: RcscmParams, hyper: Hyperparams, X) -> float:
        X = _cz(X)
        held = _Held()
        ci = _c_inputs(inputs, X.shape[1], held)
        cp = _c_params_in(p, held)
        h = C.CHyper(hyper.alpha, hyper.beta)
        out = ctypes.c_double()
        _raise(self._lib.rcscm_gpu_map_objective(self._h, ctypes.byref(ci), ctypes.byref(cp), ctypes.byref(h),
                                                 _p(X), ctypes.byref(out)))
        return out.value

    def _run(self, fn, inputs, params0, hyper, X, opt) -> SolverResult:
        opt = opt or SolverOptions()
        hyper = hyper or Hyperparams()
        X = _cz(X)
        I, J, M = X.shape
        held = _Held()
        ci = _c_inputs(inputs, J, held)
        cp = _c_params_in(params0, held)
        h = C.CHyper(hyper.alpha, hyper.beta)
        o = C.COpts(int(opt.iters), int(opt.compute_objective), int(opt.record_trajectory), float(opt.rel_obj_tol),
                    int(opt.threads), float(opt.eps_var), float(opt.gamma_fault))
        rh = np.zeros(I * J)
        ru = np.zeros(I * J)
        lam = np.zeros(I)
        out = C.CParams(_p(rh), _p(ru), _p(lam))
        n = max(int(opt.iters), 0)
        obj = np.zeros(n + 1)
        secs = np.zeros(max(n, 1))
        n_obj = ctypes.c_int(0)
        n_it = ctypes.c_int(0)
        traj = bool(opt.record_trajectory) and n > 0
        th = np.zeros(n * I * J) if traj else None
        tu = np.zeros(n * I * J) if traj else None
        tl = np.zeros(n * I) if traj else None
        res = C.CResult(_p(obj), ctypes.pointer(n_obj), _p(secs), ctypes.pointer(n_it), _p(th), _p(tu), _p(tl))
        _raise(fn(self._h, ctypes.byref(ci), ctypes.byref(cp), ctypes.byref(h), _p(X), ctypes.byref(o),
                  ctypes.byref(out), ctypes.byref(res)))
        result = SolverResult(RcscmParams(_from_ij(rh, I, J), _from_ij(ru, I, J), lam),
                              list(obj[: n_obj.value]), list(secs[: n_it.value]))
        if traj:
            for k in range(n_it.value):
                sl = slice(k * I * J, (k + 1) * I * J)
                result.trajectory.append(RcscmParams(_from_ij(th[sl], I, J), _from_ij(tu[sl], I, J),
                                                     tl[k * I:(k + 1) * I].copy()))
        return result

    def run_naive(self, inputs, params0, hyper, X, opt=None) -> SolverResult:
        return self._run(self._lib.rcscm_gpu_run_naive, inputs, params0, hyper, X, opt)

    def run_algorithm1(self, inputs, params0, hyper, X, opt=None) -> SolverResult:
        return self._run(self._lib.rcscm_gpu_run_algorithm1, inputs, params0, hyper, X, opt)

    def run_algorithm2(self, inputs, params0, hyper, X, opt=None) -> SolverResult:
        return self._run(self._lib.rcscm_gpu_run_algorithm2, inputs, params0, hyper, X, opt)

    def run_accel(self, stage: int, inputs, params0, hyper, X, opt=None) -> SolverResult:
        """rcscm_gpu_run_accel: stage 1 / 2 = run_algorithm1 / run_algorithm2."""
        lib, st = self._lib, int(stage)
        return self._run(lambda h, *rest: lib.rcscm_gpu_run_accel(h, st, *rest), inputs, params0, hyper, X, opt)

    def build_inputs(self, W, A, X, n_h: int, T, V, rank_tol: float = 1e-10):
        """rcscm_gpu_build_inputs: build_noise_scm then init_params in one call
        (model.hpp:58-124); returns (RcscmInputs, RcscmParams)."""
        X = _cz(X)
        I, J, M = X.shape
        T = np.asarray(T, np.float64)
        V = np.asarray(V, np.float64)
        a = np.zeros((I, M), np.complex128)
        b = np.zeros((I, M), np.complex128)
        rp = np.zeros((I, M, M), np.complex128)
        rpp = np.zeros((I, M, M), np.complex128)
        rh = np.zeros(I * J)
        ru = np.zeros(I * J)
        lam = np.zeros(I)
        out = C.CParams(_p(rh), _p(ru), _p(lam))
        _raise(self._lib.rcscm_gpu_build_inputs(self._h, I, J, M, _p(X), _p(_mats(W)), _p(_mats(A)), int(n_h),
                                                float(rank_tol), T.shape[1], _p(_ij(T)), _p(_ij(V)), _p(a), _p(rp),
                                                _p(rpp), _p(b), ctypes.byref(out)))
        inputs = RcscmInputs(a, rp.transpose(0, 2, 1).copy(), rpp.transpose(0, 2, 1).copy(), b, int(n_h))
        return inputs, RcscmParams(_from_ij(rh, I, J), _from_ij(ru, I, J), lam)

    def extract_target(self, inputs: RcscmInputs, p: RcscmParams, X) -> ExtractionResult:
        X = _cz(X)
        I, J, M = X.shape
        held = _Held()
        ci = _c_inputs(inputs, J, held)
        cp = _c_params_in(p, held)
        image = np.zeros((I, J, M), np.complex128)
        dry = np.zeros(I * J, np.complex128)
        _raise(self._lib.rcscm_gpu_extract_target(self._h, ctypes.byref(ci), ctypes.byref(cp), _p(X), _p(image),
                                                  _p(dry)))
        return ExtractionResult(image, np.ascontiguousarray(dry.reshape(J, I).T))

    def extract_noise(self, inputs: RcscmInputs, p: RcscmParams, X) -> np.ndarray:
        X = _cz(X)
        held = _Held()
        ci = _c_inputs(inputs, X.shape[1], held)
        cp = _c_params_in(p, held)
        noise = np.zeros_like(X)
        _raise(self._lib.rcscm_gpu_extract_noise(self._h, ctypes.byref(ci), ctypes.byref(cp), _p(X), _p(noise)))
        return noise

    # ---- STFT / ISTFT (stft.hpp) ---------------------------------------------
    def stft_shape(self, num_samples: int, sample_rate: float, win_ms: float = 64.0, hop_ms: float = 32.0):
        """-> (win, hop, frames, bins) (stft.hpp:37-46, :58-60)."""
        w, h = ctypes.c_int(), ctypes.c_int()
        f, b = ctypes.c_int64(), ctypes.c_int64()
        _raise(self._lib.rcscm_gpu_stft_shape(int(num_samples), float(sample_rate), float(win_ms), float(hop_ms),
                                              ctypes.byref(w), ctypes.byref(h), ctypes.byref(f), ctypes.byref(b)))
        return w.value, h.value, f.value, b.value

    def stft_analyze(self, samples, sample_rate: float = 16000.0, win_ms: float = 64.0, hop_ms: float = 32.0):
        """stft.hpp:50-88: samples (M, len) float64 -> Spectrogram X (bins, frames, M)
        complex128 with its win / hop (dict, the Spectrogram's metadata)."""
        x = np.asarray(samples, np.float64)
        if x.ndim != 2:
            raise InvalidInputError("stft_analyze: samples must be (channels, num_samples)")
        M, n = x.shape
        xt = np.ascontiguousarray(x.T)  # (ch, p) at ch + p*M
        if n == 0 or M == 0:
            _raise(self._lib.rcscm_gpu_stft_analyze(self._h, _p(xt), n, M, float(sample_rate), float(win_ms),
                                                    float(hop_ms), None))
        win, hop, J, B = self.stft_shape(n, sample_rate, win_ms, hop_ms)
        X = np.zeros((B, J, M), np.complex128)
        _raise(self._lib.rcscm_gpu_stft_analyze(self._h, _p(xt), n, M, float(sample_rate), float(win_ms),
                                                float(hop_ms), _p(X)))
        return X, {"sample_rate": float(sample_rate), "win_samples": win, "hop_samples": hop, "source_samples": n}

    def stft_synthesize(self, X, meta: dict, win_ms: float = 64.0, hop_ms: float = 32.0):
        """stft.hpp:92-129: Spectrogram X (bins, frames, M) + its metadata -> (M, len)."""
        X = _cz(X)
        I, J, M = X.shape
        sr = float(meta.get("sample_rate", 16000.0))
        win, hop = int(meta["win_samples"]), int(meta["hop_samples"])
        src = int(meta.get("source_samples", 0))
        n = src if src > 0 else J * hop - (win - hop)
        out = np.zeros((max(n, 0), M))
        _raise(self._lib.rcscm_gpu_stft_synthesize(self._h, _p(X), I, J, M, sr, win, hop, src, float(win_ms),
                                                   float(hop_ms), _p(out)))
        return np.ascontiguousarray(out.T)

    # ---- sphering + ILRMA (ilrma.hpp) ------------------------------------------
    def sphere(self, X):
        """ilrma.hpp:53-73: X (I, J, M) -> (Q (I, M, M) [r, c], whitened X (I, J, M))."""
        X = _cz(X)
        I, J, M = X.shape
        Q = np.zeros((I, M, M), np.complex128)  # [i][r + c*M] buffer
        Xw = np.zeros_like(X)
        _raise(self._lib.rcscm_gpu_sphere(self._h, I, J, M, _p(X), _p(Q), _p(Xw)))
        return np.ascontiguousarray(Q.transpose(0, 2, 1)), Xw

    def run_ilrma(self, X, K: int, iters: int, seed: int):
        """ilrma.hpp:145-240 -> (W, A (I, M, M) [r, c]; T (M, I, K); V (M, K, J))."""
        X = _cz(X)
        I, J, M = X.shape
        W = np.zeros((I, M, M), np.complex128)
        A = np.zeros((I, M, M), np.complex128)
        T = np.zeros((M, K, I)) if K > 0 else np.zeros(0)
        V = np.zeros((M, J, K)) if K > 0 else np.zeros(0)
        _raise(self._lib.rcscm_gpu_run_ilrma(self._h, I, J, M, int(K), int(iters), int(seed) & (2**64 - 1), _p(X),
                                             _p(W), _p(A), _p(T), _p(V)))
        tr = lambda m: np.ascontiguousarray(m.transpose(0, 2, 1))
        return tr(W), tr(A), tr(T), tr(V)

    # ---- cmd_extract on the device (tools/rcscm.cpp:158-221) --------------------
    def extract(self, samples, sample_rate: float = 16000.0, nmf_bases: int = 10, ilrma_iters: int = 50,
                seed: int = 0, target_index: int = -1, backend: str = "accel2", iters: int = 100,
                hyper: Optional["Hyperparams"] = None, eps_var: float = 1e-12, compute_objective: bool = True,
                rel_obj_tol: float = 0.0, win_ms: float = 64.0, hop_ms: float = 32.0, layout: str = "rows"):
        """STFT -> sphere -> ILRMA -> fold -> target index -> build_noise_scm ->
        init_params -> solver -> Wiener image / noise -> WOLA synthesis, all on the
        device. samples (M, len) -> dict(target, noise (M, len), target_index,
        objective, n_iters, iter_seconds); records.write_trace takes the last two
        as cmd_extract's trace.jsonl."""
        hyper = hyper or Hyperparams()
        # layout "rows": channel rows as numpy holds them (samples_layout 1, no
        # transposes); "interleaved": the reference's Waveform::samples order (0)
        inter = {"rows": False, "interleaved": True}[layout]
        x = np.asarray(samples, np.float64)
        M, n = x.shape
        x = np.ascontiguousarray(x.T if inter else x)
        o = C.CExtractOpts(float(sample_rate), float(win_ms), float(hop_ms), int(nmf_bases), int(ilrma_iters),
                           int(seed) & (2**64 - 1), int(target_index),
                           {"naive": 0, "accel1": 1, "accel2": 2}[backend], int(iters), hyper.alpha, hyper.beta,
                           float(eps_var), float(rel_obj_tol), int(bool(compute_objective)), 0 if inter else 1)
        obj = np.zeros(max(iters, 0) + 1)
        secs = np.zeros(max(iters, 1))
        r = C.CExtractResult(0, 0, 0, 0, _p(obj), 0, _p(secs))
        tgt = np.empty((n, M) if inter else (M, n))
        noi = np.empty((n, M) if inter else (M, n))
        _raise(self._lib.rcscm_gpu_extract(self._h, ctypes.byref(o), _p(x), n, M, _p(tgt), _p(noi), ctypes.byref(r)))
        if inter:
            tgt, noi = np.ascontiguousarray(tgt.T), np.ascontiguousarray(noi.T)
        return {"target": tgt, "noise": noi,
                "target_index": r.target_index, "objective": obj[:r.n_objective].tolist(), "n_iters": r.n_iters,
                "iter_seconds": secs[:r.n_iters].tolist(),
                "bins": r.bins, "frames": r.frames}

    # ---- device-resident session ---------------------------------------------
    def session_load(self, X, W, A, T, V, n_h: int = 0):
        """X (B, I, J, M); W, A (B, I, M, M); T (B, I, K); V (B, K, J)."""
        X = _cz(X)
        B, I, J, M = X.shape
        T = np.asarray(T, np.float64)
        K = T.shape[2]
        Wb = np.ascontiguousarray(np.asarray(W, np.complex128).transpose(0, 1, 3, 2))
        Ab = np.ascontiguousarray(np.asarray(A, np.complex128).transpose(0, 1, 3, 2))
        Tb = np.ascontiguousarray(T.transpose(0, 2, 1))
        Vb = np.ascontiguousarray(np.asarray(V, np.float64).transpose(0, 2, 1))
        _raise(self._lib.rcscm_gpu_session_load(self._h, B, I, J, M, K, int(n_h), _p(X), _p(Wb), _p(Ab), _p(Tb),
                                                _p(Vb)))
        self._shape = (B, I, J, M)

    def session_run(self, stages: int, iters: int = 0, hyper: Hyperparams = None, eps_var: float = 1e-12):
        hyper = hyper or Hyperparams()
        h = C.CHyper(hyper.alpha, hyper.beta)
        _raise(self._lib.rcscm_gpu_session_run(self._h, int(stages), int(iters), ctypes.byref(h), float(eps_var)))

    def session_check(self):
        _raise(self._lib.rcscm_gpu_session_check(self._h))

    def session_fetch_into(self, r_h: int, r_u: int, lam: int, dry: int = 0, image: int = 0):
        """Copy the session outputs into caller memory given as raw addresses
        (device pointers such as torch's data_ptr(), or host); 0 = skip.
        Layouts as session_fetch; synchronizes."""
        vp = lambda a: ctypes.cast(ctypes.c_void_p(a), C._dp) if a else None
        _raise(self._lib.rcscm_gpu_session_fetch(self._h, vp(r_h), vp(r_u), vp(lam), vp(dry), vp(image), 1))

    def session_fetch(self, want_image: bool = False):
        """-> dict of r_h, r_u (B, I, J), lam (B, I), dry (B, I, J), image (B, I, J, M)."""
        B, I, J, M = self._shape
        rh = np.zeros((B, I, J))
        ru = np.zeros((B, I, J))
        lam = np.zeros((B, I))
        dry = np.zeros((B, I, J), np.complex128)
        image = np.zeros((B, I, J, M), np.complex128) if want_image else None
        _raise(self._lib.rcscm_gpu_session_fetch(self._h, _p(rh), _p(ru), _p(lam), _p(dry), _p(image), 1))
        return {"r_h": rh, "r_u": ru, "lam": lam, "dry": dry, "image": image}


_default: Optional[GpuContext] = None


def default_context() -> GpuContext:
    global _default
    if _default is None:
        _default = GpuContext(0)
    return _default


def build_noise_scm(W, A, X, n_h, rank_tol=1e-10):
    return default_context().build_noise_scm(W, A, X, n_h, rank_tol)


def init_params(inputs, T, V, W, A, X):
    return default_context().init_params(inputs, T, V, W, A, X)


def map_objective(inputs, params, hyper, X):
    return default_context().map_objective(inputs, params, hyper, X)


def run_naive(inputs, params0, hyper, X, opt=None):
    return default_context().run_naive(inputs, params0, hyper, X, opt)


def run_algorithm1(inputs, params0, hyper, X, opt=None):
    return default_context().run_algorithm1(inputs, params0, hyper, X, opt)


def run_algorithm2(inputs, params0, hyper, X, opt=None):
    return default_context().run_algorithm2(inputs, params0, hyper, X, opt)


def extract_target(inputs, params, X):
    return default_context().extract_target(inputs, params, X)


def extract_noise(inputs, params, X):
    return default_context().extract_noise(inputs, params, X)
