"""Golden known answers (tests/golden/known_answers.json, written by
tests/golden/make_known_answers.py from the closed-form cases of the
reference's own tests, each citing its proj/tests file:line).

The oracle is checked against them on the CPU (pins the restatement); the GPU
path is checked against the same fixtures through the C ABI (gpu marker)."""
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "known_answers.json")


def _load():
    with open(GOLDEN) as f:
        return json.load(f)


def _cz(v):
    a = np.asarray(v, dtype=np.float64)
    return a[..., 0] + 1j * a[..., 1]


def _case(name):
    for c in _load()["cases"]:
        if c["name"] == name:
            return c
    raise KeyError(name)


def _problem(c):
    from paper_1908_01964_b200 import RcscmInputs, RcscmParams

    inp = RcscmInputs(_cz(c["a"]), _cz(c["R_prime"]), _cz(c["R_prime_pinv"]), _cz(c["b"]), 0)
    p = RcscmParams(np.asarray(c["r_h"], float), np.asarray(c["r_u"], float), np.asarray(c["lambda"], float))
    return inp, p, _cz(c["X"])


SOLVER_CASES = ["naive_scalar_e_step", "accel1_scalar_rho_first_stage", "accel2_scalar_second_stage"]


def _check_solver(c, got):
    e, tol = c["expect"], c["rtol"]
    for key, arr in (("r_h", got.r_h), ("r_u", got.r_u), ("lambda", got.lam)):
        if key in e:
            assert np.allclose(arr, e[key], rtol=tol, atol=0), (c["name"], key, arr, e[key])


def test_golden_file_is_current():
    """The committed fixture equals what the generator writes."""
    import subprocess
    import sys

    before = open(GOLDEN).read()
    subprocess.run([sys.executable, os.path.join(os.path.dirname(GOLDEN), "make_known_answers.py")], check=True,
                   capture_output=True)
    assert open(GOLDEN).read() == before


# ---- oracle (CPU) ---------------------------------------------------------------
@pytest.mark.parametrize("name", SOLVER_CASES)
def test_oracle_solver_known_answers(O, name):
    c = _case(name)
    inp, p, X = _problem(c)
    oi = O.Inputs(inp.a, inp.R_prime, inp.R_prime_pinv, inp.b, 0)
    op = O.Params(p.r_h, p.r_u, p.lam)
    got = O.run(c["backend"], oi, op, X, O.SolverOptions(iters=c["iters"])).params
    _check_solver(c, got)
    if "hat_r_h" in c["expect"]:
        hr, _ = O.e_step(oi, op, X)
        assert hr[0, 0] == pytest.approx(c["expect"]["hat_r_h"], rel=c["rtol"])
    if "rho_aa" in c["expect"]:
        rho_aa, rho_ax, rho_xx = O.rho_first_stage(oi, X, p.lam)
        assert rho_aa[0] == pytest.approx(c["expect"]["rho_aa"], rel=c["rtol"])
        assert np.max(np.abs(rho_ax)) == 0.0 and np.max(np.abs(rho_xx)) == 0.0


def test_oracle_tau_and_eig_known_answers(O):
    c = _case("tau_aa_diag")
    a, b, Rpp = _cz(c["a"]), _cz(c["b"]), _cz(c["R_prime_pinv"])
    X = np.ones((1, 4, 2), np.complex128)
    s = O.precompute(O.Inputs(a, None, Rpp, b, 0), X)
    assert s.tau_aa[0] == pytest.approx(c["expect"]["tau_aa"], rel=c["rtol"])
    s = O.precompute(O.Inputs(3.0 * b, None, Rpp, b, 0), X)
    assert s.tau_aa[0] == c["expect"]["tau_aa_a_eq_3b"]
    e = _case("eig_diag")
    vals, _ = O.hermitian_eig(_cz(e["H"]))
    assert np.allclose(vals, e["expect"]["values"], rtol=e["rtol"], atol=0)


def _wiener_instances(O):
    z = _case("wiener_rh_zero")
    n = _case("wiener_noiseless")
    zi = z["instance"]
    inp, p, X = O.make_verify_instance(zi["I"], zi["J"], zi["M"], zi["seed"])
    p = O.Params(np.zeros_like(p.r_h), p.r_u, p.lam)
    ni = n["instance"]
    inp2, p2, X2 = O.make_verify_instance(ni["I"], ni["J"], ni["M"], ni["seed"])
    cc = complex(*n["c"])
    X2 = np.stack([np.stack([cc * inp2.a[i] for _ in range(ni["J"])]) for i in range(ni["I"])])
    p2 = O.Params(np.ones_like(p2.r_h), np.full_like(p2.r_u, 1e-14), p2.lam)
    return (z, inp, p, X), (n, inp2, p2, X2, cc)


def test_oracle_wiener_known_answers(O):
    (z, inp, p, X), (n, inp2, p2, X2, cc) = _wiener_instances(O)
    img, dry = O.extract_target(inp, p, X)
    assert np.max(np.abs(dry)) == z["expect"]["max_abs"] and np.max(np.abs(img)) == z["expect"]["max_abs"]
    _, dry2 = O.extract_target(inp2, p2, X2)
    assert np.max(np.abs(dry2 - cc)) < n["expect"]["atol"]


# ---- GPU (C ABI) ----------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("name", SOLVER_CASES)
def test_gpu_solver_known_answers(gpu, name):
    from paper_1908_01964_b200 import Hyperparams, SolverOptions

    c = _case(name)
    inp, p, X = _problem(c)
    fn = {"naive": gpu.run_naive, "accel1": gpu.run_algorithm1, "accel2": gpu.run_algorithm2}[c["backend"]]
    got = fn(inp, p, Hyperparams(), X, SolverOptions(iters=c["iters"])).params
    _check_solver(c, got)


@pytest.mark.gpu
def test_gpu_wiener_known_answers(O, gpu):
    (z, inp, p, X), (n, inp2, p2, X2, cc) = _wiener_instances(O)
    r = gpu.extract_target(inp, p, X)
    assert np.max(np.abs(r.dry)) == z["expect"]["max_abs"] and np.max(np.abs(r.image)) == z["expect"]["max_abs"]
    r2 = gpu.extract_target(inp2, p2, X2)
    assert np.max(np.abs(r2.dry - cc)) < n["expect"]["atol"]
