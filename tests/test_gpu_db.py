"""K2d (accel_db.cuh): Algorithm 2 with two bins in flight per cluster -- a
cluster of CTAs owns a PAIR of bins, each thread 4 slots of either, the two bins
half an iteration apart so one bin's reduction / DSMEM exchange overlaps the
other's arithmetic. Selected by RCSCM_ACCEL_DB for fused cluster shapes.

Checked here: one iteration against the oracle (solver_accel.hpp:183-240; the
1e-9 bar of test_solver_accel.cpp:213-241 on the reference's seeded instances,
parity.check_params on the BASELINE recipe), the full iteration count against
k_accel, bitwise determinism, and that a bin's result does not depend on its
partner (odd bin counts, different splits: bitwise), ragged frame counts, bins
with sigma_ab = 0."""
import dataclasses

import numpy as np
import pytest

from parity import check_params, ru_condition_scale

pytestmark = pytest.mark.gpu


def _solve(gpu, monkeypatch, db, inp, p0, X, iters):
    from paper_1908_01964_b200 import Hyperparams, SolverOptions

    monkeypatch.setenv("RCSCM_ACCEL_DB", "1" if db else "0")
    return gpu.run_algorithm2(inp, p0, Hyperparams(), X, SolverOptions(iters=iters)).params


def _same(a, b):
    return np.array_equal(a.r_h, b.r_h) and np.array_equal(a.r_u, b.r_u) and np.array_equal(a.lam, b.lam)


@pytest.mark.parametrize("cfg,I,J", [(4, 7, 4096), (4, 4, 3000), (0, 5, 2500), (2, 6, 9000), (1, 3, 16384)])
def test_db_one_iteration_vs_oracle(O, gpu, monkeypatch, cfg, I, J):
    from paper_1908_01964_b200 import synth

    u = synth.make_config(cfg, utterances=1, I=I, J=J)[0]
    inp = gpu.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = gpu.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    g = _solve(gpu, monkeypatch, True, inp, p0, u.X, 1)
    assert gpu.last_accel_db, "K2d was not selected"
    o = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=1)).params
    r = check_params(g, o, S=ru_condition_scale(O, inp, p0, u.X))
    assert r["ok"], r
    # the same shape through k_accel: the two kernels differ only in their summation trees
    m = _solve(gpu, monkeypatch, False, inp, p0, u.X, 1)
    assert not gpu.last_accel_db
    assert np.max(np.abs(g.lam - m.lam) / m.lam) < 1e-12
    assert np.max(np.abs(g.r_h - m.r_h) / np.maximum(m.r_h, 1e-12)) < 1e-11


@pytest.mark.parametrize("cfg,I,J,iters", [(4, 5, 4096, 100), (0, 4, 3000, 50)])
def test_db_full_iterations_and_determinism(O, gpu, monkeypatch, cfg, I, J, iters):
    from paper_1908_01964_b200 import synth

    u = synth.make_config(cfg, utterances=1, I=I, J=J)[0]
    inp = gpu.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = gpu.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    a = _solve(gpu, monkeypatch, True, inp, p0, u.X, iters)
    b = _solve(gpu, monkeypatch, True, inp, p0, u.X, iters)
    assert _same(a, b)
    m = _solve(gpu, monkeypatch, False, inp, p0, u.X, iters)
    assert O.trajectory_distance(a, m) <= 1e-8
    # Wiener output of the final state against the oracle's full run (north star: 1e-6)
    o = O.run("accel2", inp, p0, u.X, O.SolverOptions(iters=iters)).params
    gd = gpu.extract_target(inp, a, u.X).dry
    _, od = O.extract_target(inp, o, u.X)
    floor = 1e-12 * np.sqrt(np.mean(np.abs(od) ** 2))
    assert np.max(np.abs(gd - od) / np.maximum(np.abs(od), floor)) <= 1e-6


def test_db_partner_independence(gpu, monkeypatch):
    """Bins are paired by position in the launch; any split of the bins (odd
    counts run their last bin alone) must give the same bits per bin."""
    from paper_1908_01964_b200 import RcscmInputs, RcscmParams, synth

    u = synth.make_config(4, utterances=1, I=9, J=4096)[0]
    inp = gpu.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = gpu.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    full = _solve(gpu, monkeypatch, True, inp, p0, u.X, 30)
    for cuts in ((0, 3, 9), (0, 1, 2, 9), (0, 4, 9)):
        parts = []
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            sl = slice(lo, hi)
            pi = RcscmInputs(inp.a[sl], inp.R_prime[sl], inp.R_prime_pinv[sl], inp.b[sl], 0)
            pp = RcscmParams(p0.r_h[sl], p0.r_u[sl], p0.lam[sl])
            parts.append(_solve(gpu, monkeypatch, True, pi, pp, u.X[sl], 30))
        assert np.array_equal(np.concatenate([q.r_h for q in parts]), full.r_h), cuts
        assert np.array_equal(np.concatenate([q.r_u for q in parts]), full.r_u), cuts
        assert np.array_equal(np.concatenate([q.lam for q in parts]), full.lam), cuts


def test_db_reference_instances_and_sigma_ab_zero(O, gpu, monkeypatch):
    """The reference's seeded instances (verify.hpp:22-56) at a cluster-sized J,
    two bins with b orthogonal to a (the literal lambda form) among them."""
    inp, p, X = O.make_verify_instance(6, 2600, 4, 777)
    b = inp.b.copy()
    for i in (1, 4):
        a = inp.a[i]
        v = b[i] - a * (np.vdot(a, b[i]) / np.vdot(a, a))
        b[i] = v / np.linalg.norm(v)
    inp = dataclasses.replace(inp, b=b)
    for iters in (1, 20):
        g = _solve(gpu, monkeypatch, True, inp, p, X, iters)
        assert gpu.last_accel_db
        o = O.run("accel2", inp, p, X, O.SolverOptions(iters=iters)).params
        if iters == 1:
            r = check_params(g, o)
            assert r["ok"], r
        else:
            assert O.trajectory_distance(g, o) <= 1e-8
