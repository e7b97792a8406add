"""The oracle's restatement of proj/core/src/metrics.cpp pinned against the reference's own
known-answer tests (proj/tests/test_metrics.cpp) and its golden spectrum_bound output
(tests/golden/inputs.npz c2_delta, written by the compiled reference: make_golden.py)."""
import numpy as np
import pytest

import cases
from oracle import ffcz_oracle as O


def test_psnr_kats():
    # test_metrics.cpp:12-24
    a, b = np.array([0.0, 1.0]), np.array([0.5, 1.0])
    assert O.psnr(a, b) == pytest.approx(20.0 * np.log10(1.0 / np.sqrt(0.125)))
    assert np.isinf(O.psnr(a, a))
    flat = np.array([3.0, 3.0])
    assert np.isinf(O.psnr(flat, flat))
    with pytest.raises(O.UndefinedMetric):
        O.psnr(flat, np.array([3.0, 3.5]))


def test_ssnr_rfe_kats():
    # test_metrics.cpp:26-41
    X = np.array([2.0 + 0j, 0.0])
    Y = np.array([2.0 + 0j, 0.2])
    assert O.ssnr(X, Y) == pytest.approx(20.0)
    assert np.isinf(O.ssnr(X, X))
    r = O.rfe(np.array([0.4 + 0j, -1j]), np.array([4.0 + 0j, 2j]))
    assert r[0] == pytest.approx(0.1) and r[1] == pytest.approx(0.25)


def test_power_spectrum_kats():
    # test_metrics.cpp:43-73
    k, p, c, fb, mean = O.power_spectrum(np.array([1.0, 2.0, 0.5, 1.5]))
    assert list(c) == [1, 2, 1] and not fb and mean == pytest.approx(1.25)
    X = np.fft.fft(np.array([-0.2, 0.6, -0.6, 0.2]))
    assert p[0] == pytest.approx(abs(X[0]) ** 2, rel=1e-9, abs=1e-15)
    assert p[1] == pytest.approx(abs(X[1]) ** 2 + abs(X[3]) ** 2, rel=1e-9)
    assert p[2] == pytest.approx(abs(X[2]) ** 2, rel=1e-9)
    k, p, c, fb, mean = O.power_spectrum(np.array([1.0, -1.0, 0.5, -0.5]))
    X = np.fft.fft(np.array([1.0, -1.0, 0.5, -0.5]))
    assert fb and p[1] == pytest.approx(abs(X[1]) ** 2 + abs(X[3]) ** 2, rel=1e-9)
    _, _, c, _, _ = O.power_spectrum(cases.noise((8, 8, 8), 3))
    assert int(c.sum()) == 512


def test_spectrum_bound_matches_reference_golden():
    inp = cases.load_inputs()
    if "c2_orig" not in inp:
        pytest.skip("golden inputs absent")
    o = inp["c2_orig"].astype(np.float64)
    mine = O.spectrum_bound_to_freq_bounds(np.fft.fftn(o), 1e-3)
    ref = inp["c2_delta"]
    assert np.all(np.abs(mine - ref) <= 1e-12 * ref.max() + 1e-9 * np.abs(ref))
    # the power-preserving property (test_metrics.cpp:78-101)
    X = np.fft.fftn(o).ravel()
    d = mine.ravel()
    ok = np.abs(X) >= 1e-9
    worst = np.hypot(np.abs(X.real) + d, np.abs(X.imag) + d)
    assert np.all(worst[ok] ** 2 <= (1 + 1e-3) * np.abs(X[ok]) ** 2 * (1 + 1e-12))
