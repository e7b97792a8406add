"""Mixed-radix passes (csrc/fft_mixed.cuh) for extents that are not powers of two: transforms
against numpy's FFT (and the brute-force DFT oracle, test_transform.cpp:25-33's bar), and the
projection loop / correct() on such shapes against the numpy oracle."""
import numpy as np
import pytest

import cases
from oracle import ffcz_oracle as O

pytestmark = pytest.mark.gpu

# radix-2/3/4/5/7 products, generic primes (11, 13, 17, 97), a prime row (97), a 6000-point row
# (packed: two 3001-point ping-pong buffers) and a 7000-point row
SHAPES = [(2,), (3,), (6,), (2, 3), (420,), (143,), (97,), (2310,), (6000,), (7000,), (100, 120), (250, 96), (60, 50, 48),
          (27, 25, 49), (11, 13, 17), (125, 36, 30), (3, 5, 7)]


@pytest.fixture(scope="module")
def ffcz():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2601_01596_b200 as P
    return P


@pytest.mark.parametrize("shape", SHAPES, ids=[str(s) for s in SHAPES])
def test_mixed_radix_dft(ffcz, shape):
    x = cases.noise(shape, 300 + len(shape))
    X = ffcz.forward_dft(x)
    ref = np.fft.fftn(x)
    assert np.max(np.abs(X - ref)) / np.max(np.abs(ref)) < 1e-13
    if x.size <= 4096:
        bf = O.brute_force_dft(x)
        assert np.max(np.abs(X - bf)) / np.max(np.abs(bf)) < 1e-9
    back = ffcz.inverse_dft(X)
    assert np.max(np.abs(back - x)) < 1e-12


@pytest.mark.parametrize("shape", [(30, 36, 40), (96, 100), (45, 27, 50)],
                         ids=["30x36x40", "96x100", "45x27x50"])
def test_mixed_radix_projection_vs_oracle(ffcz, shape):
    o = cases.noise(shape, 41)
    E = 0.01
    d = o + np.random.default_rng(42).uniform(-0.99, 0.99, shape) * E
    D = 0.7 * cases.mean_abs_delta0(o, d)
    b = O.shrink_bounds(O.DualBounds(E, D), 16)
    eps0 = d - o
    slack = 1.0 / (1.0 - 2.0**-16) - 1.0 + 2.0**-20
    S0, F0, e0, r0 = O.alternating_projection(eps0, b, 1000, slack)
    S, F, e, r = ffcz.alternating_projection(eps0, ffcz.DualBounds(b.spatial, b.freq_re), 1000,
                                             slack)
    assert (r.iterations, r.active_spatial, r.active_frequency, r.converged) == \
           (r0.iterations, r0.active_spatial, r0.active_frequency, r0.converged)
    assert np.array_equal(S != 0, S0 != 0)
    assert np.max(np.abs(e - e0)) <= 1e-9 * np.max(np.abs(e0))
    # correct(): both bounds hold exactly on the FP64 corrected field, checked by the oracle
    res = ffcz.correct(o, d, ffcz.DualBounds(E, D), 16, 1000)
    assert res.report.iterations == r0.iterations and res.verify_ok
    ok, ms, mf = O.verify_bounds(o, res.corrected, O.DualBounds(E, D))
    assert ms == 0.0 and mf <= 1e-12 * D
    # the mixed FP32 -> FP64 policy on the same shape (FP32 mixed-radix passes)
    rm = ffcz.correct(o, d, ffcz.DualBounds(E, D), 16, 1000, policy="mixed")
    assert rm.report.converged and rm.verify_ok
