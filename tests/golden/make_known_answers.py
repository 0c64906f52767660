"""Writes tests/golden/known_answers.json: the closed-form known answers the
reference's own tests pin the hot path with (proj/tests/*.cpp, cited per case).
The reference (C++/Eigen) cannot be built in this image (no Eigen), so these
analytic cases -- inputs and expected values exactly as the reference tests
state them -- are the golden vectors; tests/test_golden.py checks the oracle
(CPU) and the GPU path against them. Re-run to regenerate:
    python tests/golden/make_known_answers.py
"""
import json
import os

ALPHA, BETA = 1.1, 1e-16  # Hyperparams defaults (model.hpp:27-30)


def c(z):
    return [float(complex(z).real), float(complex(z).imag)]


cases = []

# test_solver_naive.cpp:44-57 -- e_step, scalar M = 1 hand evaluation:
# R^x = r_h |a|^2 + r_u (R' + lambda |b|^2) = 1 + 2 = 3,
# r^_h = 1 - 1/3 + |3/3|^2 = 5/3; one naive iteration then gives
# r_h = max((5/3 + beta)/(alpha + 2), eps) (solver_naive.hpp:333-334).
cases.append({
    "name": "naive_scalar_e_step", "ref": "proj/tests/test_solver_naive.cpp:44-57",
    "backend": "naive", "iters": 1, "I": 1, "J": 1, "M": 1,
    "a": [[c(1)]], "b": [[c(1)]], "R_prime": [[[c(0)]]], "R_prime_pinv": [[[c(0)]]],
    "X": [[[c(3)]]], "r_h": [[1.0]], "r_u": [[1.0]], "lambda": [2.0],
    "expect": {"hat_r_h": 5.0 / 3.0, "r_h": (5.0 / 3.0 + BETA) / (ALPHA + 2.0)}, "rtol": 1e-12,
})

# test_solver_accel.cpp:112-128 -- rho_first_stage scalar case, x = 0:
# R_u = R' + lambda b b^H = 2 -> rho_aa = 1/2, rho_ax = rho_xx = 0. One
# Algorithm 1 iteration from r_h = r_u = 1: gamma = 1/(1 + 1/2) = 2/3,
# r_h = (gamma + beta)/(alpha + 2), lambda = gamma |a^H b|^2 = 2/3 (s_bx = 0),
# r_u = gamma rho_aa(lambda) r_u~ / 1 = gamma (1/gamma) = 1.
g = 2.0 / 3.0
cases.append({
    "name": "accel1_scalar_rho_first_stage", "ref": "proj/tests/test_solver_accel.cpp:112-128",
    "backend": "accel1", "iters": 1, "I": 1, "J": 3, "M": 1,
    "a": [[c(1)]], "b": [[c(1)]], "R_prime": [[[c(0)]]], "R_prime_pinv": [[[c(0)]]],
    "X": [[[c(0)], [c(0)], [c(0)]]], "r_h": [[1.0, 1.0, 1.0]], "r_u": [[1.0, 1.0, 1.0]], "lambda": [2.0],
    "expect": {"rho_aa": 0.5, "r_h": (g + BETA) / (ALPHA + 2.0), "lambda": g, "r_u": 1.0}, "rtol": 1e-13,
})

# The same scalar problem through Algorithm 2 (R'^+ = 0, tau = 0): rho_aa =
# tau_aa + |s_ab|^2 / lambda = 1/2 -- the second stage must agree with the first
# (test_solver_accel.cpp:130-159, scalar instance).
cases.append({
    "name": "accel2_scalar_second_stage", "ref": "proj/tests/test_solver_accel.cpp:130-159",
    "backend": "accel2", "iters": 1, "I": 1, "J": 3, "M": 1,
    "a": [[c(1)]], "b": [[c(1)]], "R_prime": [[[c(0)]]], "R_prime_pinv": [[[c(0)]]],
    "X": [[[c(0)], [c(0)], [c(0)]]], "r_h": [[1.0, 1.0, 1.0]], "r_u": [[1.0, 1.0, 1.0]], "lambda": [2.0],
    "expect": {"r_h": (g + BETA) / (ALPHA + 2.0), "lambda": g, "r_u": 1.0}, "rtol": 1e-13,
})

# test_solver_accel.cpp:43-56 -- precompute_tau: R' = diag(2, 0), a = e0, b = e1
# -> tau_aa = 1/2; a = 3 b -> tau_aa = 0 (the pseudoinverse annihilates b).
cases.append({
    "name": "tau_aa_diag", "ref": "proj/tests/test_solver_accel.cpp:43-56",
    "R_prime_pinv": [[[c(0.5), c(0)], [c(0), c(0)]]], "a": [[c(1), c(0)]], "b": [[c(0), c(1)]],
    "expect": {"tau_aa": 0.5, "tau_aa_a_eq_3b": 0.0}, "rtol": 1e-14,
})

# test_linalg.cpp:10-24 -- hermitian_eig: diag(3, 1) -> ascending (1, 3).
cases.append({
    "name": "eig_diag", "ref": "proj/tests/test_linalg.cpp:10-24",
    "H": [[c(3), c(0)], [c(0), c(1)]], "expect": {"values": [1.0, 3.0]}, "rtol": 1e-14,
})

# test_wiener.cpp:9-15 -- r_h = 0 silences the estimate (dry = image = 0), on the
# reference's seeded instance random_instance(3, 8, 3, seed 1).
cases.append({
    "name": "wiener_rh_zero", "ref": "proj/tests/test_wiener.cpp:9-15",
    "instance": {"I": 3, "J": 8, "M": 3, "seed": 1}, "expect": {"max_abs": 0.0},
})

# test_wiener.cpp:17-29 -- noiseless limit: x = c a, r_u = 1e-14, r_h = 1 ->
# dry = c within 1e-6, on random_instance(2, 4, 3, seed 2), c = 1.5 - 0.8i.
cases.append({
    "name": "wiener_noiseless", "ref": "proj/tests/test_wiener.cpp:17-29",
    "instance": {"I": 2, "J": 4, "M": 3, "seed": 2}, "c": c(1.5 - 0.8j), "expect": {"atol": 1e-6},
})

out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "known_answers.json")
with open(out, "w") as f:
    json.dump({"hyper": {"alpha": ALPHA, "beta": BETA}, "cases": cases}, f, indent=1)
print(f"wrote {len(cases)} cases to {out}")
