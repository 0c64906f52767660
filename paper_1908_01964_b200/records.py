"""Host-side record formats around the solver: the JSON checkpoint shared by the
ILRMA and RCSCM stages, the line-delimited iteration trace, and the bench
records / speed-up report (checkpoint.hpp:18-196, metrics.hpp:14-145).

Pure host plumbing over numpy arrays -- nothing here touches the device. The
files are schema-compatible with the reference's: objects are written with
sorted keys and no whitespace (nlohmann::json's std::map order and dump()),
complex numbers as [re, im] pairs, every matrix with explicit rows / cols, and
a top-level schema_version. Non-finite doubles are written as null, as
nlohmann::json does. Array conventions follow api.py: W, A (I, M, M); T (N, I,
K); V (N, K, J); RcscmInputs.a / b (I, M), R_prime / R_prime_pinv (I, M, M);
RcscmParams.r_h / r_u (I, J), lam (I,).
"""
import json
import math
from dataclasses import dataclass, field
from typing import Dict, List, Sequence

import numpy as np

from .api import InvalidInputError, RcscmInputs, RcscmParams

SCHEMA_VERSION = 1  # checkpoint.hpp:20
SI_SDR_CAP = 300.0  # metrics.hpp:14


def _num(v: float):
    v = float(v)
    return v if math.isfinite(v) else None


def _dump(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"), allow_nan=False)


# ---- matrices (checkpoint.hpp:25-62) ------------------------------------------
def complex_matrix_to_json(m) -> dict:
    m = np.asarray(m, np.complex128)
    if m.ndim == 1:  # a VecC is an M x 1 matrix (checkpoint.hpp:96-97)
        m = m[:, None]
    return {"rows": int(m.shape[0]), "cols": int(m.shape[1]),
            "data": [[[_num(z.real), _num(z.imag)] for z in row] for row in m]}


def complex_matrix_from_json(j) -> np.ndarray:
    r, c = int(j["rows"]), int(j["cols"])
    d = j["data"]
    m = np.empty((r, c), np.complex128)
    for p in range(r):
        for q in range(c):
            m[p, q] = complex(float(d[p][q][0]), float(d[p][q][1]))
    return m


def real_matrix_to_json(m) -> dict:
    m = np.asarray(m, np.float64)
    return {"rows": int(m.shape[0]), "cols": int(m.shape[1]), "data": [[_num(v) for v in row] for row in m]}


def real_matrix_from_json(j) -> np.ndarray:
    r, c = int(j["rows"]), int(j["cols"])
    m = np.array(j["data"], np.float64).reshape(r, c)
    return m


# ---- stage objects (checkpoint.hpp:64-139) ------------------------------------
def demixing_to_json(W, A) -> dict:
    return {"W": [complex_matrix_to_json(m) for m in W], "A": [complex_matrix_to_json(m) for m in A]}


def demixing_from_json(j):
    return (np.array([complex_matrix_from_json(m) for m in j["W"]]),
            np.array([complex_matrix_from_json(m) for m in j["A"]]))


def nmf_to_json(T, V) -> dict:
    return {"T": [real_matrix_to_json(m) for m in T], "V": [real_matrix_to_json(m) for m in V]}


def nmf_from_json(j):
    return ([real_matrix_from_json(m) for m in j["T"]], [real_matrix_from_json(m) for m in j["V"]])


def inputs_to_json(inp: RcscmInputs) -> dict:
    return {"a": [complex_matrix_to_json(v) for v in inp.a],
            "R_prime": [complex_matrix_to_json(m) for m in inp.R_prime],
            "R_prime_pinv": [complex_matrix_to_json(m) for m in inp.R_prime_pinv],
            "b": [complex_matrix_to_json(v) for v in inp.b],
            "n_h": int(inp.n_h)}


def inputs_from_json(j) -> RcscmInputs:
    col0 = lambda m: complex_matrix_from_json(m)[:, 0]
    return RcscmInputs(a=np.array([col0(m) for m in j["a"]]),
                       R_prime=np.array([complex_matrix_from_json(m) for m in j["R_prime"]]),
                       R_prime_pinv=np.array([complex_matrix_from_json(m) for m in j["R_prime_pinv"]]),
                       b=np.array([col0(m) for m in j["b"]]), n_h=int(j["n_h"]))


def params_to_json(p: RcscmParams) -> dict:
    return {"r_h": real_matrix_to_json(p.r_h), "r_u": real_matrix_to_json(p.r_u),
            "lambda": [_num(v) for v in np.asarray(p.lam, np.float64)]}


def params_from_json(j) -> RcscmParams:
    return RcscmParams(r_h=real_matrix_from_json(j["r_h"]), r_u=real_matrix_from_json(j["r_u"]),
                       lam=np.array([float(v) for v in j["lambda"]], np.float64))


# ---- checkpoint file (checkpoint.hpp:141-174) ---------------------------------
@dataclass
class Checkpoint:
    W: np.ndarray
    A: np.ndarray
    T: List[np.ndarray]
    V: List[np.ndarray]
    inputs: RcscmInputs
    params: RcscmParams


def save_checkpoint(path: str, W, A, T, V, inputs: RcscmInputs, params: RcscmParams) -> None:
    """Full ILRMA + RCSCM-setup state, so the solver stage can be rerun across
    backends from bit-identical inputs (checkpoint.hpp:141-154)."""
    j = {"schema_version": SCHEMA_VERSION, "demixing": demixing_to_json(W, A), "nmf": nmf_to_json(T, V),
         "inputs": inputs_to_json(inputs), "params": params_to_json(params)}
    try:
        f = open(path, "w")
    except OSError:
        raise InvalidInputError("save_checkpoint: cannot open " + path) from None
    with f:
        f.write(_dump(j))


def load_checkpoint(path: str) -> Checkpoint:
    """checkpoint.hpp:163-174: InvalidInputError on a missing file or a schema
    version other than SCHEMA_VERSION."""
    try:
        f = open(path)
    except OSError:
        raise InvalidInputError("load_checkpoint: cannot open " + path) from None
    with f:
        j = json.load(f)
    if int(j["schema_version"]) != SCHEMA_VERSION:
        raise InvalidInputError("load_checkpoint: unsupported schema version")
    W, A = demixing_from_json(j["demixing"])
    T, V = nmf_from_json(j["nmf"])
    return Checkpoint(W, A, T, V, inputs_from_json(j["inputs"]), params_from_json(j["params"]))


# ---- iteration trace (checkpoint.hpp:176-189) ---------------------------------
def write_trace(path: str, backend: str, iter_seconds: Sequence[float], objective: Sequence[float]) -> None:
    """One JSON object per iteration: backend, iter (1-based), seconds, and the
    objective after that iteration when it was computed."""
    try:
        f = open(path, "w")
    except OSError:
        raise InvalidInputError("write_trace: cannot open " + path) from None
    with f:
        for k, s in enumerate(iter_seconds):
            line = {"backend": backend, "iter": k + 1, "seconds": _num(s)}
            if k + 1 < len(objective):
                line["objective"] = _num(objective[k + 1])
            f.write(_dump(line) + "\n")


# ---- bench records and the speed-up report (metrics.hpp:16-145) ---------------
@dataclass
class BenchRecord:
    backend: str
    mics: int = 0
    bins: int = 0
    frames: int = 0
    iter_seconds: List[float] = field(default_factory=list)
    total_seconds: float = 0.0
    objective: List[float] = field(default_factory=list)
    warmup: int = 3  # leading iterations excluded from the median

    def to_json(self) -> dict:  # checkpoint.hpp:190-195
        return {"backend": self.backend, "M": self.mics, "I": self.bins, "J": self.frames,
                "iter_seconds": [_num(s) for s in self.iter_seconds], "total_seconds": _num(self.total_seconds),
                "objective": [_num(v) for v in self.objective], "warmup": self.warmup}


def _median(v: List[float]) -> float:
    t = sorted(v)
    n = len(t)
    return t[n // 2] if n % 2 == 1 else 0.5 * (t[n // 2 - 1] + t[n // 2])


def si_sdr(estimate, reference) -> float:
    """Scale-invariant SDR in dB between single channels, capped at 300 dB for
    exact matches (metrics.hpp:16-29)."""
    e = np.asarray(estimate, np.float64).ravel()
    r = np.asarray(reference, np.float64).ravel()
    if e.size != r.size:
        raise InvalidInputError("si_sdr: length mismatch")
    ref_energy = float(r @ r)
    if ref_energy == 0.0:
        raise InvalidInputError("si_sdr: zero reference")
    alpha = float(e @ r) / ref_energy
    target_energy = alpha * alpha * ref_energy
    d = e - alpha * r
    err_energy = float(d @ d)
    if err_energy <= target_energy * 10.0 ** (-SI_SDR_CAP / 10.0):
        return SI_SDR_CAP
    return 10.0 * math.log10(target_energy / err_energy)


def median_iter_seconds(rec: BenchRecord) -> float:
    """Median per-iteration time with min(warmup, n-1) leading iterations
    skipped (metrics.hpp:43-51)."""
    skip = min(rec.warmup, max(0, len(rec.iter_seconds) - 1))
    t = list(rec.iter_seconds[skip:])
    if not t:
        raise InvalidInputError("median_iter_seconds: no timed iterations")
    return _median(t)


@dataclass
class SpeedupReport:
    median_seconds: Dict[str, float] = field(default_factory=dict)
    ratios: Dict[str, float] = field(default_factory=dict)
    exponents: Dict[str, float] = field(default_factory=dict)


def fit_exponent(mics: Sequence[int], seconds: Sequence[float]) -> float:
    """Least-squares slope of log t against log M (metrics.hpp:64-81)."""
    if len(mics) != len(seconds) or len(mics) < 2:
        raise InvalidInputError("fit_exponent: need >= 2 matched points")
    n = len(mics)
    sx = sy = sxx = sxy = 0.0
    for m, s in zip(mics, seconds):
        x, y = math.log(float(m)), math.log(s)
        sx += x
        sy += y
        sxx += x * x
        sxy += x * y
    return (n * sxy - sx * sy) / (n * sxx - sx * sx)


def speedup_report(records: Sequence[BenchRecord]) -> SpeedupReport:
    """Ratios between backends at matching (M, I, J) and per-backend complexity
    exponents over M sweeps at fixed I*J, independent of record order
    (metrics.hpp:85-143)."""
    if len(records) < 2:
        raise InvalidInputError("speedup_report: need >= 2 records")
    rep = SpeedupReport()
    medians: Dict[tuple, List[float]] = {}
    for rec in records:
        medians.setdefault((rec.backend, (rec.mics, rec.bins, rec.frames)), []).append(median_iter_seconds(rec))
    by_shape: Dict[tuple, Dict[str, float]] = {}
    for (backend, shape), meds in sorted(medians.items()):
        by_shape.setdefault(shape, {})[backend] = _median(meds)
    for shape in sorted(by_shape):
        backends = by_shape[shape]
        if len(backends) < 2:
            continue
        for na in sorted(backends):
            rep.median_seconds[na] = backends[na]
            for nb in sorted(backends):
                if na != nb:
                    rep.ratios[na + "/" + nb] = backends[na] / backends[nb]
    sweeps: Dict[tuple, Dict[int, List[float]]] = {}
    for (backend, (mics, bins, frames)), meds in sorted(medians.items()):
        for med in meds:
            sweeps.setdefault((backend, bins * frames), {}).setdefault(mics, []).append(med)
    for (backend, _), by_m in sorted(sweeps.items()):
        if len(by_m) < 2:
            continue
        ms = sorted(by_m)
        rep.exponents[backend] = fit_exponent(ms, [_median(by_m[m]) for m in ms])
    return rep
