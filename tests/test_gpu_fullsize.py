"""BASELINE configurations at their FULL sizes on the GPU.

The oracle cannot replay a whole C3 batch or C4 utterance in a test's time, so
at full size the CUDA path is held to properties that do not depend on size,
plus an oracle spot check on a few bins / utterances of the same run:
  - determinism: the same call twice gives the same bits (the reference's
    contract, parallel.hpp:14-16, test_solver_accel.cpp:351-365);
  - shard invariance: solving the utterances / bins in two ranges gives the
    bits of the whole run (the multi-GPU partition, parallel.hpp:50-80);
  - the floors and finiteness every solver output obeys (solver_accel.hpp:139,
    :157, :174);
  - spot check: chosen utterances / bins against the oracle after the full
    iteration count, <= 1e-6 on the Wiener output (wiener.hpp:29-41).
C0 is small enough to replay whole, for both rules.
"""
import numpy as np
import pytest

from parity import output_rel_err, rel_err

pytestmark = pytest.mark.gpu

EPS = 1e-12


def _check_floors(r_h, r_u, lam):
    for name, v in (("r_h", r_h), ("r_u", r_u), ("lambda", lam)):
        assert np.all(np.isfinite(v)), name
        assert float(v.min()) >= EPS, (name, float(v.min()))


def _session_solve(gpu, X, W, A, T, V, iters):
    import paper_1908_01964_b200._capi as C

    gpu.session_load(X, W, A, T, V, 0)
    gpu.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
    # the bench step (params0, precompute fused into K2) with the Wiener output fused
    gpu.session_run(C.STAGE_RESET | C.STAGE_PRECOMPUTE | C.STAGE_ACCEL | C.STAGE_WIENER, iters)
    gpu.session_check()
    return gpu.session_fetch()


@pytest.fixture(scope="module")
def c3_batch():
    from paper_1908_01964_b200 import synth

    utts = synth.make_config(3)
    assert len(utts) == 256
    return utts, synth.stack(utts)


def test_c3_full_batch(O, gpu, c3_batch):
    """BASELINE configs[3] whole: 256 utterances x 513 x 320, M = 4, 100 iterations."""
    utts, (X, W, A, T, V) = c3_batch
    assert X.shape == (256, 513, 320, 4)
    full = _session_solve(gpu, X, W, A, T, V, 100)
    _check_floors(full["r_h"], full["r_u"], full["lam"])
    assert np.all(np.isfinite(full["dry"]))
    again = _session_solve(gpu, X, W, A, T, V, 100)
    for k in ("r_h", "r_u", "lam", "dry"):
        assert np.array_equal(full[k], again[k]), k
    del again
    # an uneven utterance split (two ranks' ranges)
    for lo, hi in ((0, 100), (100, 256)):
        part = _session_solve(gpu, X[lo:hi], W[lo:hi], A[lo:hi], T[lo:hi], V[lo:hi], 100)
        for k in ("r_h", "r_u", "lam", "dry"):
            assert np.array_equal(part[k], full[k][lo:hi]), (k, lo, hi)
        del part
    worst = {"dry": 0.0, "r_h": 0.0, "r_u": 0.0, "lambda": 0.0}
    for k in (0, 131, 255):
        u = utts[k]
        inp = O.build_noise_scm(u.W, u.A, u.X, 0)
        p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
        o = O.run("accel2_binparallel", inp, p0, u.X, O.SolverOptions(iters=100, threads=8)).params
        _, odry = O.extract_target(inp, o, u.X)
        worst["dry"] = max(worst["dry"], output_rel_err(full["dry"][k], odry))
        worst["r_h"] = max(worst["r_h"], float(rel_err(full["r_h"][k], o.r_h).max()))
        worst["r_u"] = max(worst["r_u"], float(rel_err(full["r_u"][k], o.r_u).max()))
        worst["lambda"] = max(worst["lambda"], float(rel_err(full["lam"][k], o.lam).max()))
    print("\nC3 full batch, utterances 0/131/255 after 100 iterations:", {k: f"{v:.2e}" for k, v in worst.items()})
    assert worst["dry"] <= 1e-6, worst


def _bins(O, u, sel):
    """Oracle inputs / params0 of the selected bins only (every quantity is per bin)."""
    inp = O.build_noise_scm(u.W[sel], u.A[sel], u.X[sel], 0)
    p0 = O.init_params(inp, u.T[sel], u.V, u.W[sel], u.A[sel], u.X[sel])
    return inp, p0


@pytest.mark.parametrize("cfg", [4, 2])
def test_full_utterance_bins(O, gpu, cfg):
    """BASELINE configs[4] (2049 x 4096, M = 8, 100 iterations: 2-CTA clusters) and
    configs[2] (513 x 20000, M = 2, 50 iterations: 10-CTA clusters) whole, through
    the C ABI entry points a reference caller uses."""
    from paper_1908_01964_b200 import Hyperparams, RcscmInputs, RcscmParams, SolverOptions, synth

    c = synth.CONFIGS[cfg]
    u = synth.make_config(cfg)[0]
    I, J, M = u.X.shape
    assert (I, J, M) == (c["I"], c["J"], c["M"])
    iters = c["iters"]
    inp = gpu.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = gpu.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    opt = SolverOptions(iters=iters)
    full = gpu.run_algorithm2(inp, p0, Hyperparams(), u.X, opt).params
    _check_floors(full.r_h, full.r_u, full.lam)
    again = gpu.run_algorithm2(inp, p0, Hyperparams(), u.X, opt).params
    assert np.array_equal(full.r_h, again.r_h) and np.array_equal(full.r_u, again.r_u)
    assert np.array_equal(full.lam, again.lam)
    cut = I // 3 + 1
    parts = []
    for sl in (slice(0, cut), slice(cut, I)):
        pi = RcscmInputs(inp.a[sl], inp.R_prime[sl], inp.R_prime_pinv[sl], inp.b[sl], 0)
        pp = RcscmParams(p0.r_h[sl], p0.r_u[sl], p0.lam[sl])
        parts.append(gpu.run_algorithm2(pi, pp, Hyperparams(), u.X[sl], opt).params)
    assert np.array_equal(np.concatenate([q.r_h for q in parts]), full.r_h)
    assert np.array_equal(np.concatenate([q.r_u for q in parts]), full.r_u)
    assert np.array_equal(np.concatenate([q.lam for q in parts]), full.lam)
    dry = gpu.extract_target(inp, full, u.X).dry
    assert np.all(np.isfinite(dry))
    sel = np.array([0, 1, I // 2, I - 1])
    oinp, op0 = _bins(O, u, sel)
    o = O.run("accel2_binparallel", oinp, op0, u.X[sel], O.SolverOptions(iters=iters, threads=4)).params
    _, odry = O.extract_target(oinp, o, u.X[sel])
    err = output_rel_err(dry[sel], odry)
    print(f"\nC{cfg} full, bins {list(sel)} after {iters} iterations: dry {err:.2e}, "
          f"r_h {rel_err(full.r_h[sel], o.r_h).max():.2e}, lambda {rel_err(full.lam[sel], o.lam).max():.2e}")
    assert err <= 1e-6


@pytest.mark.parametrize("rule", ["accel2", "naive"])
def test_c0_whole_against_oracle(O, gpu, rule):
    """BASELINE configs[0] whole (513 x 320, M = 2, 100 iterations), both rules,
    every bin against the oracle."""
    from paper_1908_01964_b200 import Hyperparams, SolverOptions, synth

    u = synth.make_config(0)[0]
    assert u.X.shape == (513, 320, 2)
    inp = O.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    backend = "accel2_binparallel" if rule == "accel2" else "naive"
    o = O.run(backend, inp, p0, u.X, O.SolverOptions(iters=100, threads=8)).params
    gfn = gpu.run_algorithm2 if rule == "accel2" else gpu.run_naive
    g = gfn(inp, p0, Hyperparams(), u.X, SolverOptions(iters=100)).params
    _check_floors(g.r_h, g.r_u, g.lam)
    _, odry = O.extract_target(inp, o, u.X)
    gdry = gpu.extract_target(inp, g, u.X).dry
    err = output_rel_err(gdry, odry)
    print(f"\nC0 whole, {rule}, 100 iterations: dry {err:.2e}, lambda {rel_err(g.lam, o.lam).max():.2e}")
    assert err <= 1e-6
