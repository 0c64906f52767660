"""cmd_extract's pipeline on the device (rcscm_gpu_extract, tools/rcscm.cpp:158-221):
STFT -> sphere -> ILRMA -> fold -> target selection -> build_noise_scm ->
init_params -> solver -> Wiener image / noise -> WOLA synthesis, against the same
chain of oracle steps (numpy for the fold and select_target_index)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
SR = 16000.0


def _mixture(M, n, seed):
    """Two amplitude-modulated noise sources, instantaneously mixed, plus a
    small sensor-noise floor (keeps every bin energised, test_ilrma.cpp:133-137)."""
    r = np.random.default_rng(seed)
    t = np.arange(n) / SR
    s1 = r.standard_normal(n) * (1.0 + np.sin(2 * np.pi * 3.0 * t))
    s2 = r.standard_normal(n) * (1.0 + np.cos(2 * np.pi * 5.0 * t))
    mix = r.standard_normal((M, 2))
    return mix @ np.stack([s1, s2]) + 0.01 * r.standard_normal((M, n))


def _oracle_extract(O, x, K, ilrma_iters, seed, iters, backend="accel2"):
    X, win, hop = O.stft_analyze(x, SR, 64.0, 32.0)
    Q, Xw = O.sphere(X)
    Wi, _, T, V = O.run_ilrma(Xw, K, ilrma_iters, seed)
    W = Wi @ Q
    A = np.linalg.inv(W)
    I, J, M = X.shape
    power = np.zeros(M)
    for i in range(I):
        y = W[i] @ X[i].T
        power += np.sum(np.abs(y) ** 2, axis=1) * np.sum(np.abs(A[i]) ** 2, axis=0)
    n_h = int(np.argmax(power))
    inp = O.build_noise_scm(W, A, X, n_h)
    p0 = O.init_params(inp, T[n_h], V[n_h], W, A, X)
    res = O.run(backend, inp, p0, X, O.SolverOptions(iters=iters, compute_objective=True))
    img, _ = O.extract_target(inp, res.params, X)
    noise = O.extract_noise(inp, res.params, X)
    tw = O.stft_synthesize(img, SR, 64.0, 32.0, win, hop, x.shape[1])
    nw = O.stft_synthesize(noise, SR, 64.0, 32.0, win, hop, x.shape[1])
    return tw, nw, n_h, res.objective


@pytest.mark.parametrize("M,n,K,ilrma_iters,iters", [(2, 16000, 4, 3, 20), (3, 12000, 2, 2, 10)])
def test_gpu_extract_matches_oracle(O, gpu, M, n, K, ilrma_iters, iters):
    x = _mixture(M, n, 5 + M)
    g = gpu.extract(x, SR, nmf_bases=K, ilrma_iters=ilrma_iters, seed=3, iters=iters)
    tw, nw, n_h, obj = _oracle_extract(O, x, K, ilrma_iters, 3, iters)
    # rounding-noise response of the oracle chain (ILRMA amplifies it)
    xp = x * (1 + 1e-15 * np.random.default_rng(1).standard_normal(x.shape))
    tp, _, _, objp = _oracle_extract(O, xp, K, ilrma_iters, 3, iters)
    sens = float(np.max(np.abs(tp - tw)) / np.max(np.abs(tw)))
    bar = max(1e-7, 50.0 * sens)
    assert g["target_index"] == n_h
    assert g["target"].shape == tw.shape == (M, n)
    assert float(np.max(np.abs(g["target"] - tw)) / np.max(np.abs(tw))) <= bar
    assert float(np.max(np.abs(g["noise"] - nw)) / np.max(np.abs(nw))) <= bar
    assert len(g["objective"]) == iters + 1
    assert len(g["iter_seconds"]) == g["n_iters"] == iters and min(g["iter_seconds"]) > 0
    dobj = max(abs(a - b) for a, b in zip(obj, objp))
    assert np.allclose(g["objective"], obj, rtol=max(1e-8, 50 * dobj / max(abs(obj[-1]), 1e-300)), atol=0)
    # x = target image + noise (wiener.hpp:46-53) survives the linear synthesis
    inner = slice(1024, n - 1024)
    assert np.max(np.abs(g["target"][:, inner] + g["noise"][:, inner] - x[:, inner])) <= 1e-8 * np.max(np.abs(x))


def test_gpu_extract_backends_agree(gpu):
    """naive / Algorithm 1 / Algorithm 2 give the same extraction (the reference's
    cross-backend bar, acceptance.cpp:34-65, carried to the waveform)."""
    x = _mixture(2, 12000, 9)
    outs = {b: gpu.extract(x, SR, nmf_bases=2, ilrma_iters=2, seed=1, iters=10, backend=b,
                           compute_objective=False) for b in ("accel2", "accel1", "naive")}
    ref = outs["accel2"]["target"]
    for b in ("accel1", "naive"):
        assert outs[b]["target_index"] == outs["accel2"]["target_index"]
        assert float(np.max(np.abs(outs[b]["target"] - ref)) / np.max(np.abs(ref))) <= 1e-7, b


def test_gpu_extract_layouts_bitwise(gpu):
    """samples_layout 0 (the reference's Waveform::samples, M x len col-major) and
    1 (channel rows) run the same arithmetic: bitwise equal outputs."""
    x = _mixture(3, 9000, 4)
    a = gpu.extract(x, SR, nmf_bases=2, ilrma_iters=2, seed=1, iters=5)
    b = gpu.extract(x, SR, nmf_bases=2, ilrma_iters=2, seed=1, iters=5, layout="interleaved")
    assert np.array_equal(a["target"], b["target"]) and np.array_equal(a["noise"], b["noise"])
    assert a["objective"] == b["objective"]
