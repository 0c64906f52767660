"""Checkpoint / trace / bench-record formats (records.py), ported from the
reference's test_checkpoint.cpp and test_metrics.cpp. Host only."""
import json

import numpy as np
import pytest

from paper_1908_01964_b200 import InvalidInputError, RcscmInputs, RcscmParams
from paper_1908_01964_b200 import records as R


def _cm(r, rows, cols):
    return r.standard_normal((rows, cols)) + 1j * r.standard_normal((rows, cols))


def _instance(I, J, M, seed):
    r = np.random.default_rng(seed)
    G = np.array([_cm(r, M, M - 1) for _ in range(I)])
    inp = RcscmInputs(a=_cm(r, I, M), R_prime=G @ G.conj().transpose(0, 2, 1),
                      R_prime_pinv=_cm(r, I * M, M).reshape(I, M, M), b=_cm(r, I, M), n_h=1)
    p = RcscmParams(r_h=0.1 + np.abs(r.standard_normal((I, J))), r_u=0.1 + np.abs(r.standard_normal((I, J))),
                    lam=0.1 + np.abs(r.standard_normal(I)))
    return inp, p


def test_checkpoint_round_trip_exact(tmp_path):
    """test_checkpoint.cpp:12-50: every field survives save/load bit for bit."""
    inp, p = _instance(3, 6, 3, 1)
    r = np.random.default_rng(2)
    W = np.array([_cm(r, 3, 3) for _ in range(3)])
    A = np.linalg.inv(W)
    T = [np.abs(r.uniform(-1, 1, (3, 4))) for _ in range(3)]
    V = [np.abs(r.uniform(-1, 1, (4, 6))) for _ in range(3)]
    path = str(tmp_path / "ck.json")
    R.save_checkpoint(path, W, A, T, V, inp, p)
    ck = R.load_checkpoint(path)
    assert np.array_equal(ck.W, W) and np.array_equal(ck.A, A)
    for n in range(3):
        assert np.array_equal(ck.T[n], T[n]) and np.array_equal(ck.V[n], V[n])
    for f in ("a", "R_prime", "R_prime_pinv", "b"):
        assert np.array_equal(getattr(ck.inputs, f), getattr(inp, f)), f
    assert ck.inputs.n_h == inp.n_h
    assert np.array_equal(ck.params.r_h, p.r_h) and np.array_equal(ck.params.r_u, p.r_u)
    assert np.array_equal(ck.params.lam, p.lam)
    # top-level layout: sorted keys, compact (nlohmann::json dump order)
    text = open(path).read()
    assert text.startswith('{"demixing":{"A":[{"cols":3,"data":[[[')
    assert set(json.loads(text)) == {"schema_version", "demixing", "nmf", "inputs", "params"}


def test_checkpoint_schema_version_validated(tmp_path):
    """test_checkpoint.cpp:52-74, plus a missing file."""
    inp, p = _instance(1, 2, 2, 3)
    path = str(tmp_path / "schema.json")
    R.save_checkpoint(path, np.eye(2)[None], np.eye(2)[None], [np.ones((1, 2))] * 2, [np.ones((2, 2))] * 2, inp, p)
    j = json.load(open(path))
    j["schema_version"] = 999
    json.dump(j, open(path, "w"))
    with pytest.raises(InvalidInputError, match="schema"):
        R.load_checkpoint(path)
    with pytest.raises(InvalidInputError, match="cannot open"):
        R.load_checkpoint(str(tmp_path / "absent.json"))


def test_complex_serialization_shape():
    """test_checkpoint.cpp:76-89: [re, im] pairs with explicit shape."""
    m = _cm(np.random.default_rng(4), 2, 3)
    j = R.complex_matrix_to_json(m)
    assert j["rows"] == 2 and j["cols"] == 3
    assert len(j["data"]) == 2 and len(j["data"][0]) == 3 and len(j["data"][0][0]) == 2
    assert np.array_equal(R.complex_matrix_from_json(j), m)
    # a vector is an M x 1 matrix
    assert R.complex_matrix_to_json(m[0])["cols"] == 1


def test_write_trace(tmp_path):
    """test_checkpoint.cpp:91-106: one record per iteration, 1-based; the
    objective after iteration k is objective[k]."""
    path = str(tmp_path / "trace.jsonl")
    R.write_trace(path, "accel2", [0.1, 0.2], [-5.0, -4.0, -3.0])
    lines = [json.loads(s) for s in open(path).read().splitlines()]
    assert [ln["iter"] for ln in lines] == [1, 2]
    assert all(ln["backend"] == "accel2" for ln in lines)
    assert [ln["objective"] for ln in lines] == [-4.0, -3.0]
    assert [ln["seconds"] for ln in lines] == [0.1, 0.2]
    R.write_trace(path, "naive", [0.1, 0.2], [])
    assert all("objective" not in json.loads(s) for s in open(path).read().splitlines())


def _row(n, seed):
    return np.random.default_rng(seed).standard_normal(n)


def _fake(backend, mics, t, bins=64, frames=1024):
    return R.BenchRecord(backend, mics, bins, frames, [t] * 10, 10 * t)


def test_si_sdr():
    """test_metrics.cpp:33-56."""
    ref = _row(1000, 1)
    assert R.si_sdr(ref, ref) == R.SI_SDR_CAP
    assert R.si_sdr(2.0 * ref, ref) == R.SI_SDR_CAP
    assert R.si_sdr(-ref, ref) == R.SI_SDR_CAP
    ref = _row(2000, 2)
    noise = _row(2000, 3)
    noise -= (noise @ ref) / (ref @ ref) * ref
    noise *= np.linalg.norm(ref) / np.linalg.norm(noise)
    assert abs(R.si_sdr(ref + noise, ref)) <= 1e-9
    ref = _row(100, 4)
    with pytest.raises(InvalidInputError):
        R.si_sdr(_row(99, 5), ref)
    with pytest.raises(InvalidInputError):
        R.si_sdr(ref, np.zeros(100))


def test_median_and_speedup_report():
    """test_metrics.cpp:58-100."""
    rec = _fake("naive", 4, 1.0)
    rec.iter_seconds = [100.0, 100.0, 100.0, 2.0, 2.0, 2.0, 2.0]
    assert R.median_iter_seconds(rec) == 2.0
    rep = R.speedup_report([_fake("naive", 4, 1e-3), _fake("accel2", 4, 1e-3)])
    assert rep.ratios["naive/accel2"] == pytest.approx(1.0)
    recs = [_fake("naive", m, 1e-5 * m ** 3) for m in (2, 4, 8, 16)] + [_fake("accel2", m, 1e-5) for m in (2, 4, 8, 16)]
    rep = R.speedup_report(recs)
    assert rep.exponents["naive"] == pytest.approx(3.0, rel=0.01)
    assert rep.exponents["accel2"] == pytest.approx(0.0, abs=0.01)
    recs = []
    for m in (2, 4, 8):
        recs += [_fake("naive", m, 1e-4 * m ** 3), _fake("accel1", m, 1e-4 * m ** 2)]
    fwd = R.speedup_report(recs)
    rev = R.speedup_report(recs[::-1])
    assert fwd == rev
    assert R.fit_exponent([2, 4, 8], [4.0, 16.0, 64.0]) == pytest.approx(2.0)
    with pytest.raises(InvalidInputError):
        R.fit_exponent([2], [4.0])
    with pytest.raises(InvalidInputError):
        R.fit_exponent([2, 4], [4.0])
    with pytest.raises(InvalidInputError):
        R.speedup_report([rec])
