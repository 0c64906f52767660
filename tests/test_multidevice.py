"""Bins sharded over a device list inside one C-ABI context (rcscm_gpu_config
devices / num_devices): each device gets a contiguous bin range, its
inputs sliced straight from the caller's buffers and its results copied into its
(strided, for I x J col-major arrays) slice of the caller's outputs. The box has
one GPU, so the list repeats device 0: the ranges still run on separate
contexts, streams and host threads with no cross-range waits, which is what the
sharding logic needs; results must be bitwise equal to the single-device call."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _hyper():
    from paper_1908_01964_b200 import Hyperparams

    return Hyperparams()


def _opts(**kw):
    from paper_1908_01964_b200 import SolverOptions

    return SolverOptions(**kw)


def _instance(O, cfg, I, J):
    from paper_1908_01964_b200 import synth

    u = synth.make_config(cfg, utterances=1, I=I, J=J)[0]
    inp = O.build_noise_scm(u.W, u.A, u.X, 0)
    p0 = O.init_params(inp, u.T, u.V, u.W, u.A, u.X)
    return u, inp, p0


@pytest.fixture(scope="module")
def multi():
    from paper_1908_01964_b200 import GpuContext

    return {n: GpuContext(devices=[0] * n) for n in (2, 3)}


def _same(a, b):
    return all(np.array_equal(getattr(a, f), getattr(b, f)) for f in ("r_h", "r_u", "lam"))


@pytest.mark.parametrize("cfg,I,J,iters", [(1, 300, 640, 20), (0, 7, 320, 10), (4, 5, 4096, 5)])
def test_solvers_bitwise_across_device_counts(O, gpu, multi, cfg, I, J, iters):
    u, inp, p0 = _instance(O, cfg, I, J)
    for name in ("run_algorithm2", "run_naive", "run_algorithm1"):
        if name != "run_algorithm2" and J > 640:
            continue
        ref = getattr(gpu, name)(inp, p0, _hyper(), u.X, _opts(iters=iters))
        for n, ctx in multi.items():
            got = getattr(ctx, name)(inp, p0, _hyper(), u.X, _opts(iters=iters))
            assert _same(got.params, ref.params), (name, n)
            assert len(got.iter_seconds) == iters


def test_wiener_bitwise_across_device_counts(O, gpu, multi):
    u, inp, p0 = _instance(O, 1, 130, 640)
    p = gpu.run_algorithm2(inp, p0, _hyper(), u.X, _opts(iters=10)).params
    ref, noise = gpu.extract_target(inp, p, u.X), gpu.extract_noise(inp, p, u.X)
    for n, ctx in multi.items():
        got = ctx.extract_target(inp, p, u.X)
        assert np.array_equal(got.image, ref.image) and np.array_equal(got.dry, ref.dry), n
        assert np.array_equal(ctx.extract_noise(inp, p, u.X), noise), n


def test_more_devices_than_bins_and_errors(O, gpu, multi):
    from paper_1908_01964_b200 import NumericalError, RcscmParams, UnsupportedError

    inp, p, X = O.make_verify_instance(2, 8, 2, 31)  # 2 bins over 3 devices: one range empty
    ref = gpu.run_algorithm2(inp, p, _hyper(), X, _opts(iters=3)).params
    assert _same(multi[3].run_algorithm2(inp, p, _hyper(), X, _opts(iters=3)).params, ref)
    with pytest.raises(UnsupportedError, match="one device"):
        multi[2].run_algorithm2(inp, p, _hyper(), X, _opts(iters=3, compute_objective=True))
    # a singular slot in the second range reports its global bin (test_gpu_parity::test_errors)
    inp, p, X = O.make_verify_instance(6, 4, 2, 19)
    rh, ru = p.r_h.copy(), p.r_u.copy()
    rh[4, 1] = ru[4, 1] = 0.0
    with pytest.raises(NumericalError, match="e_step: singular covariance at bin 4, frame 1"):
        multi[2].run_naive(inp, RcscmParams(rh, ru, p.lam), _hyper(), X, _opts(iters=1))
