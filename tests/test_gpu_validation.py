"""Engine-side validation through the C-ABI (GPU): DualBounds' invariants on raw arrays
(bounds.cpp:10-59: entries > 0 and finite, Hermitian-consistent Re/Im lanes) checked on the host
or device copy, and a malformed archive rejected by apply_archive BEFORE any device scatter
(archive.cpp:205-208), leaving the context usable."""
import numpy as np
import pytest

import cases
from oracle import ffcz_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2601_01596_b200 as P
    return P


def _case():
    shape = (8, 12, 10)
    o = cases.noise(shape, 41)
    E = 0.05
    d = cases.uniform_perturb(o, E, 42, precision="f64")
    D = np.full(shape, 0.7 * cases.mean_abs_delta0(o, d))
    return o, d, E, D


@pytest.mark.parametrize("where", ["host", "device"])
def test_asymmetric_per_component_bounds_rejected(P, where):
    import torch
    o, d, E, D = _case()
    bad = D.copy()
    bad[1, 2, 3] *= 1.5          # its mirror (7, 10, 7) keeps the old value
    if where == "device":
        o, d = torch.tensor(o, device="cuda"), torch.tensor(d, device="cuda")
        bad = torch.tensor(bad, device="cuda")
    with pytest.raises(P.ValidationError, match="not Hermitian-consistent"):
        P.correct(o, d, P.DualBounds(E, bad))


@pytest.mark.parametrize("where", ["host", "device"])
def test_nonpositive_bounds_rejected(P, where):
    import torch
    o, d, E, D = _case()
    bad = D.copy()
    bad[0, 0, 0] = 0.0
    Epp = np.full(o.shape, E)
    Epp[3, 3, 3] = np.nan
    if where == "device":
        o, d = torch.tensor(o, device="cuda"), torch.tensor(d, device="cuda")
        bad, Epp, D = (torch.tensor(x, device="cuda") for x in (bad, Epp, D))
    with pytest.raises(P.ValidationError, match="strictly positive"):
        P.correct(o, d, P.DualBounds(E, bad))
    with pytest.raises(P.ValidationError, match="strictly positive"):
        P.correct(o, d, P.DualBounds(Epp, D))


def test_symmetric_bounds_validated_once(P):
    o, d, E, D = _case()
    b = P.DualBounds(E, D)
    r1 = P.correct(o, d, b, want_archive=False)
    assert b._validated_for is not None          # later calls skip the check
    r2 = P.correct(o, d, b, want_archive=False)
    assert r1.report == r2.report or r1.report.iterations == r2.report.iterations
    assert np.array_equal(r1.frequency_codes, r2.frequency_codes)


def _archive(P):
    o, d, E, D = _case()
    r = P.correct(o, d, P.DualBounds(E, float(D.flat[0])))
    return o, d, r


def test_padding_bits_ignored_like_bitvector(P):
    # 5 x 7 x 9 = 315 samples and 5 x 7 x 5 = 175 half-grid components: both flag streams end in
    # a partial byte.  The reference's BitVector ignores bits >= nbits, so setting every padding
    # bit must not change the decoded field.
    o = cases.noise((5, 7, 9), 43)
    d = cases.uniform_perturb(o, 0.05, 44, precision="f64")
    r = P.correct(o, d, P.DualBounds(0.05, 0.6 * cases.mean_abs_delta0(o, d)))
    a = O.read_archive(r.archive_bytes)
    ref = P.apply_archive(r.archive_bytes, d)
    sf = np.packbits(a.spatial_flags, bitorder="little")
    ff = np.packbits(a.frequency_flags, bitorder="little")
    sf[-1] |= np.uint8((0xFF << (a.spatial_flags.size % 8)) & 0xFF)
    ff[-1] |= np.uint8((0xFF << (a.frequency_flags.size % 8)) & 0xFF)
    out = P.apply_archive(O.write_archive_raw_flags(a, sf.tobytes(), ff.tobytes(), level=1), d)
    assert np.array_equal(out, ref)


def test_flag_count_mismatch_is_format_error_and_context_survives(P):
    o, d, r = _archive(P)
    a = O.read_archive(r.archive_bytes)
    ff = np.packbits(a.frequency_flags, bitorder="little")
    # one extra frequency flag without a matching code
    idx = int(np.flatnonzero(~a.frequency_flags)[0])
    ff2 = np.packbits(np.where(np.arange(a.frequency_flags.size) == idx, True, a.frequency_flags),
                      bitorder="little")
    data = O.write_archive_raw_flags(a, np.packbits(a.spatial_flags, bitorder="little").tobytes(),
                                     ff2.tobytes(), level=1)
    with pytest.raises(P.FormatError, match="edit count mismatch"):
        P.apply_archive(data, d)
    # the context is still healthy: a valid archive decodes
    good = P.apply_archive(r.archive_bytes, d)
    assert np.all(np.isfinite(good))
    del ff
