"""STFT analysis / WOLA synthesis (stft.hpp): the oracle restatement pinned by
the reference's own test cases (proj/tests/test_stft.cpp), and the GPU path
(cuFFT + our framing / layout / overlap-add kernels, through the C ABI)
against the oracle and the same cases. White noise is numpy-seeded (the
reference's mt19937 draws are not reproduced; the checks are seed-free)."""
import numpy as np
import pytest

SR = 16000.0


def _noise(M, n, seed):
    return np.random.default_rng(seed).standard_normal((M, n))


def _interior_rms_error(a, b, win):
    """test_stft.cpp:25-31: relative RMS error excluding one window at each edge."""
    n = a.shape[1] - 2 * win
    assert n > 0
    da, db = a[:, win:win + n], b[:, win:win + n]
    return float(np.linalg.norm(da - db) / np.linalg.norm(db))


# ---- oracle pinned by the reference cases ----------------------------------------
def test_oracle_shape_and_params(O):
    """test_stft.cpp:35-44 (J = ceil((139200 + 512) / 512) = 273) and :73-80."""
    win, hop = O.stft_params(SR, 64.0, 32.0)
    assert (win, hop) == (1024, 512)
    assert (139200 + (win - hop) + hop - 1) // hop == 273
    with pytest.raises(O.InvalidInputError):
        O.stft_params(SR, 32.0, 64.0)
    with pytest.raises(O.InvalidInputError):
        O.stft_analyze(np.zeros((1, 0)), SR, 64.0, 32.0)


def test_oracle_dc_and_impulse(O):
    """test_stft.cpp:46-71: DC lands in bins 0/1 on interior frames; an impulse at
    a frame centre has flat magnitude w[win/2]."""
    X, win, hop = O.stft_analyze(np.ones((1, 8000)), SR, 64.0, 32.0)
    e = np.sum(np.abs(X[:, 1:15, 0]) ** 2, axis=1)
    assert e[0] > 0 and e[1] < e[0] and e[2:].sum() < 1e-20 * e[0]
    x = np.zeros((1, 8000))
    frame = 4
    x[0, frame * hop - (win - hop) + win // 2] = 1.0
    X, _, _ = O.stft_analyze(x, SR, 64.0, 32.0)
    assert np.allclose(np.abs(X[:, frame, 0]), O.hamming_window(win)[win // 2], rtol=1e-10, atol=0)


def test_oracle_round_trip_and_linearity(O):
    """test_stft.cpp:82-97 (round trip < 1e-8 interior), :99-108 (zero spectrum),
    :110-124 (linearity < 1e-10)."""
    w = _noise(2, 48000, 3)
    X, win, hop = O.stft_analyze(w, SR, 64.0, 32.0)
    r = O.stft_synthesize(X, SR, 64.0, 32.0, win, hop, w.shape[1])
    assert r.shape == w.shape and _interior_rms_error(r, w, 1024) < 1e-8
    t = np.arange(32000)
    s = np.sin(2 * np.pi * 440.0 * t / SR)[None, :]
    X, win, hop = O.stft_analyze(s, SR, 64.0, 32.0)
    assert _interior_rms_error(O.stft_synthesize(X, SR, 64.0, 32.0, win, hop, 32000), s, 1024) < 1e-8
    z = O.stft_synthesize(np.zeros_like(X), SR, 64.0, 32.0, win, hop, 32000)
    assert np.max(np.abs(z)) == 0.0
    with pytest.raises(O.InvalidInputError):
        O.stft_synthesize(X, SR, 32.0, 16.0, win, hop, 32000)
    w1, w2 = _noise(1, 16000, 5), _noise(1, 16000, 6)
    s1, s2, sm = (O.stft_analyze(v, SR, 64.0, 32.0)[0] for v in (w1, w2, 2 * w1 - 3 * w2))
    assert np.sqrt(np.sum(np.abs(sm - 2 * s1 + 3 * s2) ** 2) / np.sum(np.abs(sm) ** 2)) < 1e-10


# ---- GPU ------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("M,n,win_ms,hop_ms", [(4, 139200, 64.0, 32.0), (2, 8000, 64.0, 32.0), (3, 5000, 64.0, 16.0),
                                               (1, 3001, 20.0, 10.0)])
def test_gpu_stft_matches_oracle(O, gpu, M, n, win_ms, hop_ms):
    """GPU analysis and synthesis against the oracle: <= 1e-12 relative (max-abs
    over the max magnitude) on the spectrogram and the resynthesised waveform;
    shapes as test_stft.cpp:35-44."""
    w = _noise(M, n, 11 + M)
    X, meta = gpu.stft_analyze(w, SR, win_ms, hop_ms)
    Xo, win, hop = O.stft_analyze(w, SR, win_ms, hop_ms)
    assert X.shape == Xo.shape and (meta["win_samples"], meta["hop_samples"]) == (win, hop)
    assert np.max(np.abs(X - Xo)) <= 1e-12 * np.max(np.abs(Xo))
    if (M, n) == (4, 139200):
        assert X.shape == (513, 273, 4)
    # synthesis of a modified spectrum (nonzero imaginary DC/Nyquist parts are discarded as the reference's inverse does)
    Y = X * (0.5 + 0.25j)
    r = gpu.stft_synthesize(Y, meta, win_ms, hop_ms)
    ro = O.stft_synthesize(Y, SR, win_ms, hop_ms, win, hop, n)
    assert r.shape == ro.shape == (M, n)
    assert np.max(np.abs(r - ro)) <= 1e-12 * np.max(np.abs(ro))
    rt = gpu.stft_synthesize(X, meta, win_ms, hop_ms)
    assert _interior_rms_error(rt, w, win) < 1e-8


@pytest.mark.gpu
def test_gpu_stft_reference_cases(gpu):
    """test_stft.cpp:46-71 (DC, impulse), :99-108 (zero spectrum, mismatch), :73-80 (empty)."""
    from paper_1908_01964_b200 import InvalidInputError

    X, meta = gpu.stft_analyze(np.ones((1, 8000)), SR)
    e = np.sum(np.abs(X[:, 1:15, 0]) ** 2, axis=1)
    assert e[0] > 0 and e[1] < e[0] and e[2:].sum() < 1e-20 * e[0]
    x = np.zeros((1, 8000))
    x[0, 4 * 512 - 512 + 512] = 1.0
    X, meta = gpu.stft_analyze(x, SR)
    assert np.allclose(np.abs(X[:, 4, 0]), 0.54 - 0.46 * np.cos(np.pi), rtol=1e-10, atol=0)
    z = gpu.stft_synthesize(np.zeros_like(X), meta)
    assert z.shape == (1, 8000) and np.max(np.abs(z)) == 0.0
    with pytest.raises(InvalidInputError, match="window/hop do not match analysis"):
        gpu.stft_synthesize(X, meta, 32.0, 16.0)
    with pytest.raises(InvalidInputError, match="empty waveform"):
        gpu.stft_analyze(np.zeros((1, 0)), SR)
    with pytest.raises(InvalidInputError, match="win_ms > hop_ms"):
        gpu.stft_analyze(np.ones((1, 100)), SR, 32.0, 64.0)
