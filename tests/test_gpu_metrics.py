"""Device metrics (csrc/metrics.cu) against the oracle's restatement of
proj/core/src/metrics.cpp, the reference's golden spectrum_bound output, and acceptance
criterion 5 (power-spectrum ribbon, proj/tests/acceptance.cpp:170-200)."""
import numpy as np
import pytest

import cases
from oracle import ffcz_oracle as O

pytestmark = pytest.mark.gpu

SHAPES = [(4,), (17,), (16, 16), (12, 10, 9), (32, 32, 32), (64, 48, 40), (100, 120)]


@pytest.fixture(scope="module")
def ffcz():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2601_01596_b200 as P
    return P


def _close(a, b, rel=1e-12):
    return np.all(np.abs(a - b) <= rel * np.max(np.abs(b)) + 1e-9 * np.abs(b))


def test_spectrum_bound_golden(ffcz):
    inp = cases.load_inputs()
    o = inp["c2_orig"]
    for x in (o, o.astype(np.float64)):  # f32 buffer and widened
        d = ffcz.spectrum_bound_to_freq_bounds(x, 1e-3)
        assert _close(d, inp["c2_delta"])


@pytest.mark.parametrize("shape", SHAPES, ids=[str(s) for s in SHAPES])
def test_spectrum_bound_vs_oracle(ffcz, shape):
    x = cases.noise(shape, 11)
    d = ffcz.spectrum_bound_to_freq_bounds(x, 1e-3)
    ref = O.spectrum_bound_to_freq_bounds(np.fft.fftn(x), 1e-3)
    assert _close(d, ref)
    # mirrored components carry identical bounds (test_metrics.cpp:93-95), exactly
    m = O.mirror_index_grid(x.shape)
    assert np.array_equal(d.ravel(), d.ravel()[m])


def test_spectrum_bound_errors_and_floor(ffcz):
    with pytest.raises(ffcz.ValidationError, match="rho"):
        ffcz.spectrum_bound_to_freq_bounds(np.ones(8), -1.0)
    with pytest.raises(ffcz.ValidationError):
        ffcz.spectrum_bound_to_freq_bounds(np.ones(8), float("nan"))
    z = ffcz.spectrum_bound_to_freq_bounds(np.zeros(4), 1e-3)
    assert np.all(z > 0.0)


@pytest.mark.parametrize("shape", SHAPES, ids=[str(s) for s in SHAPES])
def test_metrics_vs_oracle(ffcz, shape):
    o = cases.noise(shape, 21)
    r = o + np.random.default_rng(22).uniform(-1e-3, 1e-3, shape)
    m = ffcz.metrics(o, r)
    p, s, mr, ms = O.metrics(o, r)
    assert m.psnr_db == pytest.approx(p, rel=1e-12)
    assert m.ssnr_db == pytest.approx(s, rel=1e-10)
    assert m.max_rfe == pytest.approx(mr, rel=1e-10)
    assert m.max_spatial == ms  # exact: max of the same FP64 differences


def test_metrics_edge_cases(ffcz):
    o = cases.noise((8, 8), 5)
    m = ffcz.metrics(o, o)
    assert np.isinf(m.psnr_db) and np.isinf(m.ssnr_db) and m.max_rfe == 0.0 and m.max_spatial == 0.0
    flat = np.full(8, 3.0)
    with pytest.raises(ffcz.UndefinedMetricError, match="psnr"):
        ffcz.metrics(flat, flat + np.linspace(0, 1e-3, 8))
    with pytest.raises(ffcz.UndefinedMetricError, match="ssnr"):
        ffcz.metrics(np.zeros(8), np.zeros(8))
    with pytest.raises(ffcz.ValidationError):
        ffcz.metrics(np.zeros(8), np.zeros(9))


PS_SHAPES = SHAPES + [(8, 8, 8), (8192,)]  # (8192,): 4097 shells, past the shared-memory bins


@pytest.mark.parametrize("shape", PS_SHAPES, ids=[str(s) for s in PS_SHAPES])
def test_power_spectrum_vs_oracle(ffcz, shape):
    x = cases.noise(shape, 31) + 2.0
    ps = ffcz.power_spectrum(x)
    k, p, c, fb, mean = O.power_spectrum(x)
    assert np.array_equal(ps.counts, c)  # bit-exact
    assert int(ps.counts.sum()) == x.size
    assert ps.mean_fallback == fb and ps.mean == pytest.approx(mean, rel=1e-13)
    assert np.all(np.abs(ps.power - p) <= 1e-12 * p.max())


def test_power_spectrum_kats(ffcz):
    # test_metrics.cpp:43-73
    ps = ffcz.power_spectrum(np.array([1.0, 2.0, 0.5, 1.5]))
    assert list(ps.counts) == [1, 2, 1] and not ps.mean_fallback
    assert ps.mean == pytest.approx(1.25)
    X = np.fft.fft(np.array([-0.2, 0.6, -0.6, 0.2]))
    assert ps.power[1] == pytest.approx(abs(X[1]) ** 2 + abs(X[3]) ** 2, rel=1e-9)
    ps = ffcz.power_spectrum(np.array([1.0, -1.0, 0.5, -0.5]))
    assert ps.mean_fallback


def test_device_tensors(ffcz):
    import torch
    x = torch.from_numpy(cases.noise((32, 32, 32), 41)).cuda()
    d = ffcz.spectrum_bound_to_freq_bounds(x, 1e-3)
    assert d.is_cuda and d.dtype == torch.float64
    ref = ffcz.spectrum_bound_to_freq_bounds(x.cpu().numpy(), 1e-3)
    assert np.array_equal(d.cpu().numpy(), ref)
    m = ffcz.metrics(x, x + 1e-4)
    assert m.max_spatial == pytest.approx(1e-4, rel=1e-9)
    ps = ffcz.power_spectrum(x.float())
    assert int(ps.counts.sum()) == 32 ** 3


def test_power_spectrum_ribbon(ffcz):
    """Acceptance criterion 5 (acceptance.cpp:170-200) on the golden 32^3 config-2 field made
    zero-mean (power_spectrum's mean-removal branch, metrics.cpp:21-30, so that each field's own
    mean normalisation does not enter): with the device rho bound every shell b >= 1 of the
    corrected field's power spectrum stays within rho of the original's, and the device shell
    sums agree with the oracle's."""
    case = next(c for c in cases.all_cases() if c.name == "config2_rho32")
    rho = 1e-3
    mu = float(np.mean(case.original))
    o, d = case.original - mu, case.decompressed - mu
    D = ffcz.spectrum_bound_to_freq_bounds(o, rho)
    r = ffcz.correct(o, d, ffcz.DualBounds(case.E, D, D), 16, 1000, "f64")
    assert r.report.converged and r.verify_ok
    corrected = ffcz.apply_archive(r.archive_bytes, d)
    p0 = ffcz.power_spectrum(o)
    p1 = ffcz.power_spectrum(corrected)
    assert p0.mean_fallback and p1.mean_fallback
    sel = p0.power[1:] > 0
    worst = np.max(np.abs(p1.power[1:][sel] - p0.power[1:][sel]) / p0.power[1:][sel])
    assert worst <= rho, worst
    _, q1, c1, _, _ = O.power_spectrum(corrected)
    assert np.array_equal(p1.counts, c1)
    assert np.all(np.abs(p1.power - q1) <= 1e-12 * q1.max())
