"""Device decoder: ffcz_cuda_apply_archive = ffcz::apply_edits(decompressed, read_archive(bytes))
(archive.cpp:137-273).  Checked on the reference's OWN archives (tests/golden/archives.npz,
written by the compiled reference) and on the engine's archives, against the numpy oracle's
apply_edits and the engine's corrected field; corrupt / mismatched inputs raise like the
reference (format_error / validation_error)."""
import os

import numpy as np
import pytest

import cases
from oracle import ffcz_oracle as O

pytestmark = pytest.mark.gpu

ARCH = dict(np.load(os.path.join(cases.GOLDEN, "archives.npz")))
CASES = {c.name: c for c in cases.all_cases()}
REF_NAMES = [n for n in ARCH if n in CASES]


@pytest.fixture(scope="module")
def ffcz():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2601_01596_b200 as P
    return P


def _close(a, b):
    scale = max(1.0, float(np.max(np.abs(b))))
    assert np.max(np.abs(a - b)) <= 1e-12 * scale, np.max(np.abs(a - b))


@pytest.mark.parametrize("name", REF_NAMES)
def test_apply_reference_archive(ffcz, name):
    case = CASES[name]
    data = ARCH[name].tobytes()
    want = O.apply_edits(case.decompressed, O.read_archive(data))
    got = ffcz.apply_archive(data, case.decompressed)
    assert got.shape == case.decompressed.shape
    _close(got, want)


@pytest.mark.parametrize("name", ["config1_c0.4", "config2_rho32", "config3_frame256",
                                  "config4_comb32", "per_point_2d", "odd_12x10x9"])
def test_apply_engine_archive(ffcz, name):
    case = CASES[name]
    b = ffcz.DualBounds(case.E, case.Dre, case.Dim)
    r = ffcz.correct(case.original, case.decompressed, b, case.m, case.max_iters, case.precision)
    got = ffcz.apply_archive(r.archive_bytes, case.decompressed)
    _close(got, r.corrected)
    _close(got, O.apply_edits(case.decompressed, O.read_archive(r.archive_bytes)))
    r0 = ffcz.correct(case.original, case.decompressed, b, case.m, case.max_iters,
                      case.precision, device_encode=True, zlib_level=0)
    _close(ffcz.apply_archive(r0.archive_bytes, case.decompressed), r.corrected)


def test_apply_device_input(ffcz):
    import torch
    case = CASES["config1_c1.0"]
    data = ARCH["config1_c1.0"].tobytes()
    d32 = case.decompressed.astype(np.float32)
    host = ffcz.apply_archive(data, d32)
    dev = ffcz.apply_archive(data, torch.from_numpy(d32).cuda()).cpu().numpy()
    assert np.array_equal(host, dev)


def test_apply_errors(ffcz):
    case = CASES["config1_c1.0"]
    data = bytearray(ARCH["config1_c1.0"].tobytes())
    bad = bytes(data[:10]) + bytes([data[10] ^ 1]) + bytes(data[11:])   # header CRC mismatch
    with pytest.raises(ffcz.FormatError):
        ffcz.apply_archive(bad, case.decompressed)
    with pytest.raises(ffcz.FormatError):
        ffcz.apply_archive(bytes(data[:-5]), case.decompressed)        # truncated
    with pytest.raises(ffcz.ValidationError):
        ffcz.apply_archive(bytes(data), case.decompressed[:, :, :-1].copy())
