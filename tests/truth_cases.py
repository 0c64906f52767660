"""Shared cases and error statistics of the ground-truth parity checks
(tests/test_truth.py on the CPU, tests/test_gpu_truth.py on the GPU,
tools/truth_table.py for the DESIGN table).

Each case is a BASELINE synthetic instance (paper_1908_01964_b200.synth) at a
size the binary128 truth (oracle/truth.cpp) evaluates in seconds. For one
iteration from params0 the three evaluations of the same formulas --

  truth   binary128 (oracle.truth_accel_one_iter / truth_naive_one_iter)
  oracle  the double restatement of the reference (the reference's arithmetic)
  gpu     the CUDA path through the C ABI

-- give per-field elementwise relative errors |x - truth| / max(|truth|, 1e-12)
(verify.hpp:60-68 with the truth as one side).
"""
from __future__ import annotations

import numpy as np

EPS = np.finfo(float).eps

# (cfg, I, J): every BASELINE config shape at reduced I (full J), plus full C1
CASES = [(0, 64, 320), (1, 64, 640), (2, 6, 20000), (3, 64, 320), (4, 12, 4096), (1, 1025, 640)]
NAIVE_CASES = [(0, 64, 320), (1, 64, 640), (3, 64, 320), (4, 6, 4096)]


def case_id(c):
    return f"c{c[0]}_I{c[1]}_J{c[2]}"


def instance(O, cfg, I, J):
    from paper_1908_01964_b200 import synth

    u = synth.make_config(cfg, utterances=1, I=I, J=J)[0]
    inp = O.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    return u, inp, p0


def rel_to_truth(x, t):
    x = np.asarray(x, float)
    t = np.asarray(t, float)
    return np.abs(x - t) / np.maximum(np.abs(t), 1e-12)


def field_errors(p, truth):
    """-> {field: elementwise relative error array} against the truth."""
    return {"r_h": rel_to_truth(p.r_h, truth.r_h), "r_u": rel_to_truth(p.r_u, truth.r_u),
            "lambda": rel_to_truth(p.lam, truth.lam)}


def bound_units(p, truth, B):
    """-> {field: |x - truth| / (eps * B)}: the error in units of the first-order
    rounding scale B of oracle/truth.cpp (a double evaluation of the formulas
    in any order is expected within a modest multiple of it)."""
    u = lambda x, t, b: np.abs(np.asarray(x, float) - t) / (EPS * np.maximum(b, 1e-300))
    return {"r_h": u(p.r_h, truth.r_h, B.r_h), "r_u": u(p.r_u, truth.r_u, B.r_u),
            "lambda": u(p.lam, truth.lam, B.lam)}


# Bars (units of eps * B) held by both the oracle (tests/test_truth.py) and the
# GPU (tests/test_gpu_truth.py); set from the oracle's measured maxima
# with headroom.
C_ACCEL = 8.0
C_NAIVE = 8.0
