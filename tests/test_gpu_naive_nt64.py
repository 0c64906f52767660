"""K3's 64-thread CTA (k_naive EMU): chosen by batch size (RCSCM_NAIVE_NT64 = the
fewest bins that take it) where it pads fewer frames than the 128-thread CTA
(J = 320: 5 exact rounds instead of 3 with half of the last idle). It emulates
the 128-thread layout's lambda summation -- thread tid carries the accumulators
of threads tid and tid + 64 apart and leaves four warp partials in that layout's
order -- so every bit must equal the 128-thread result (solver_naive.hpp:319-386
per bin), or a sharded run would differ from an unsharded one."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,J", [(4, 320), (2, 320), (3, 192), (4, 576), (2, 300)])
def test_naive_nt64_bitwise(O, gpu, monkeypatch, M, J):
    from paper_1908_01964_b200 import Hyperparams, SolverOptions

    inp, p, X = O.make_verify_instance(9, J, M, 9100 + J + M)
    res = []
    for nt64 in ("1", "0"):
        monkeypatch.setenv("RCSCM_NAIVE_NT64", nt64)
        n0 = gpu.launch_count
        r = gpu.run_naive(inp, p, Hyperparams(), X, SolverOptions(iters=12, record_trajectory=True))
        assert gpu.launch_count > n0
        res.append(r)
    a, b = res
    assert np.array_equal(a.params.r_h, b.params.r_h)
    assert np.array_equal(a.params.r_u, b.params.r_u)
    assert np.array_equal(a.params.lam, b.params.lam)
    for ta, tb in zip(a.trajectory, b.trajectory):
        assert np.array_equal(ta.r_h, tb.r_h) and np.array_equal(ta.r_u, tb.r_u) and np.array_equal(ta.lam, tb.lam)
    # and against the oracle (the reference's 1e-8 cross-backend bar, acceptance.cpp:34-65)
    o = O.run("naive", inp, p, X, O.SolverOptions(iters=12)).params
    assert O.trajectory_distance(a.params, o) <= 1e-8


def test_naive_nt64_session_batch(gpu, monkeypatch):
    """BASELINE config 3's shape through the session (the bench's naive leg)."""
    from paper_1908_01964_b200 import synth
    import paper_1908_01964_b200._capi as C

    utts = synth.make_config(3, utterances=2, I=24, J=320)
    X, W, A, T, V = synth.stack(utts)
    outs = []
    for nt64 in ("1", "0"):
        monkeypatch.setenv("RCSCM_NAIVE_NT64", nt64)
        gpu.session_load(X, W, A, T, V, 0)
        gpu.session_run(C.STAGE_SETUP | C.STAGE_PRECOMPUTE)
        gpu.session_run(C.STAGE_RESET | C.STAGE_NAIVE, 15)
        gpu.session_check()
        outs.append(gpu.session_fetch())
    a, b = outs
    for k in ("r_h", "r_u", "lam"):
        assert np.array_equal(a[k], b[k]), k
