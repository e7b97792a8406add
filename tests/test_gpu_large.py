"""Lines longer than the shared-memory passes hold (csrc/fft_large.cuh): global-memory mixed-radix
Stockham passes, Bluestein for prime factors above 64, packed real rows.  FFTW takes any extent
(transform.cpp:20-50); SPEC.md:84 / PAPER.md:104 name an EEG-like 31,000-sample 1-D signal.

* forward_dft / inverse_dft against numpy's FFT (rel 1e-12) on 1-D rows above 8192 (power of
  two, mixed radix incl. 31, a prime -> Bluestein, odd), 2-D column axes above 4096 and a
  column axis with a large prime factor;
* correct() on 1-D signals of 31,000 and 20,011 (prime) samples and an 8192 x 64 field against
  the UNMODIFIED reference run here on the same inputs (oracle/_ref): iterations, converged,
  active counts, verify result and flags identical, int32 codes identical, both bounds exact on
  the FP64 corrected field."""
import numpy as np
import pytest

import cases
from oracle import ref_binding as ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ffcz():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2601_01596_b200 as P
    return P


SHAPES = [(16384,), (31000,), (20011,), (24000,), (30030,), (8192, 64), (6400 * 2, 8),
          (4099 * 4, 4), (12, 9000, 3)]


@pytest.mark.parametrize("shape", SHAPES, ids=[str(s) for s in SHAPES])
def test_long_line_dft(ffcz, shape):
    x = cases.noise(shape, 7)
    X = ffcz.forward_dft(x)
    want = np.fft.fftn(x)
    assert np.max(np.abs(X - want)) / np.max(np.abs(want)) < 1e-12
    back = ffcz.inverse_dft(X)
    assert np.max(np.abs(back - x)) < 1e-11 * max(1.0, float(np.max(np.abs(x))))


def _signal(n, seed):
    """EEG-like: a few oscillations + 1/f noise, FP32; uniform base error within 0.99 E."""
    rng = np.random.default_rng(seed)
    t = np.arange(n) / 256.0
    x = (np.sin(2 * np.pi * 10 * t) + 0.5 * np.sin(2 * np.pi * 22 * t + 1.0)
         + np.cumsum(rng.standard_normal(n)) * 0.02)
    orig = x.astype(np.float32).astype(np.float64)
    E = 1e-3 * float(orig.max() - orig.min())
    dec = (orig + rng.uniform(-0.99 * E, 0.99 * E, orig.shape)).astype(np.float32).astype(np.float64)
    return orig, dec, E


@pytest.mark.parametrize("shape,c", [((31000,), 0.8), ((20011,), 1.0), ((8192, 64), 0.8)])
def test_long_line_correct_matches_reference(ffcz, shape, c):
    if len(shape) == 1:
        orig, dec, E = _signal(shape[0], shape[0])
    else:
        orig = cases.noise(shape, 3).astype(np.float32).astype(np.float64)
        E = 1e-3 * float(orig.max() - orig.min())
        rng = np.random.default_rng(4)
        dec = (orig + rng.uniform(-0.99 * E, 0.99 * E, shape)).astype(np.float32).astype(np.float64)
    D = c * float(np.mean(np.abs(np.fft.fftn(dec - orig))))
    mine = ffcz.correct(orig.astype(np.float32), dec.astype(np.float32), ffcz.DualBounds(E, D),
                        16, 1000, "f32")
    r = ref.correct(orig, dec, E, D, None, 16, 1000, "f32")
    assert (mine.report.iterations, mine.report.converged, mine.report.active_spatial,
            mine.report.active_frequency) == (r.report.iterations, r.report.converged,
                                              r.report.active_spatial, r.report.active_frequency)
    assert mine.verify_ok == r.verify_ok
    a, b = ref.archive_edits(mine.archive_bytes), ref.archive_edits(r.archive)
    assert np.array_equal(a.spatial_flags, b.spatial_flags)
    assert np.array_equal(a.frequency_flags, b.frequency_flags)
    assert np.array_equal(a.spatial_codes, b.spatial_codes)
    assert np.array_equal(a.frequency_codes, b.frequency_codes)
    if r.report.converged:
        corr = mine.corrected
        assert float(np.max(np.abs(corr - orig) - E)) <= 0.0
        assert cases.freq_excess_per_component(orig, corr, np.full(shape, D), None) <= 1e-15


def test_8192_square_correct_self_verified(ffcz):
    """8192^2 (SPEC.md:84 sizes; the column axis exceeds the shared-memory passes): the FP64
    corrected field satisfies both bounds exactly under numpy's FFT, and the engine's verify
    agrees (the reference would take minutes on the host here)."""
    n = 8192
    rng = np.random.default_rng(81)
    orig = rng.standard_normal((n, n)).astype(np.float32).astype(np.float64)
    E = 1e-3 * float(orig.max() - orig.min())
    dec = (orig + rng.uniform(-0.99 * E, 0.99 * E, orig.shape)).astype(np.float32).astype(np.float64)
    D = 0.8 * float(np.mean(np.abs(np.fft.rfft2(dec - orig))))
    r = ffcz.correct(orig.astype(np.float32), dec.astype(np.float32), ffcz.DualBounds(E, D), 16,
                     1000, "f32", want_archive=False)
    assert r.report.converged and r.verify_ok
    corr = r.corrected
    assert float(np.max(np.abs(corr - orig) - E)) <= 0.0
    assert cases.freq_excess_per_component(orig, corr, D, None) <= 1e-15
