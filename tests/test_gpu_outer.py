"""Device outer stage and device-assembled archives (csrc/deflate.cu, csrc/archive_dev.cu).

* outer_compress_device: the u64 raw size + zlib framing of streams.cpp:21-32, produced on the
  GPU, must decode with zlib (the reference's outer_decompress is zlib uncompress,
  streams.cpp:34-48) to the input bytes, for every block shape the encoder distinguishes: empty,
  tiny, runs of every length around the 258-byte match limit, incompressible (stored blocks),
  sizes around the 32 KiB block boundary.
* crc32c_device: equal to the host CRC-32C (archive.cpp:61-71) at every length around the 8 KiB
  segment and 256-byte lane boundaries.
* archives written with the default FFCZ_OUTER_DEVICE mode: the UNMODIFIED reference's
  read_archive (oracle/_ref) decodes them to exactly the edits of the zlib-9 archive (flags, int32
  codes, escapes), for global and per-component bounds held on the host and on the device (the
  header CRC over the bound arrays is then computed on the GPU)."""
import zlib

import numpy as np
import pytest

import cases
from oracle import ffcz_oracle as O
from oracle import ref_binding as ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ffcz():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2601_01596_b200 as P
    return P


def _runs(rng, n, lens):
    out, v = [], 0
    while sum(map(len, out)) < n:
        L = int(rng.choice(lens))
        v = (v + 1 + int(rng.integers(0, 254))) & 0xFF
        out.append(bytes([v]) * L)
    return b"".join(out)[:n]


def _payloads():
    rng = np.random.default_rng(5)
    yield "empty", b""
    yield "one", b"\x07"
    yield "two_same", b"\xff\xff"
    yield "four_same", b"\x90\x90\x90\x90"
    yield "ones_100k", b"\xff" * 100000
    yield "zeros_chunk", b"\x00" * 32768
    yield "zeros_chunk_plus1", b"\x00" * 32769
    for L in (1, 2, 3, 4, 5, 258, 259, 260, 261, 262, 516, 517, 518, 519):
        yield f"run_{L}", (b"\xa5" * L + b"\x11") * 37
    yield "runs_mixed", _runs(rng, 300001, [1, 2, 3, 4, 7, 100, 258, 259, 260, 1000, 5000])
    yield "random_200k", rng.integers(0, 256, 200000, dtype=np.uint8).tobytes()
    yield "literals_high", bytes(range(144, 256)) * 300
    sparse = np.zeros(250000, dtype=np.uint8)
    sparse[rng.integers(0, sparse.size, 3000)] = rng.integers(1, 256, 3000, dtype=np.uint8)
    yield "sparse_bits", sparse.tobytes()


PAYLOADS = list(_payloads())


@pytest.mark.parametrize("name,data", PAYLOADS, ids=[p[0] for p in PAYLOADS])
def test_outer_compress_round_trip(ffcz, name, data):
    out = ffcz.ffcz.outer_compress_device(data)
    assert int.from_bytes(out[:8], "little") == len(data)
    assert zlib.decompress(out[8:]) == data
    assert O.outer_decompress(out) == data
    # never worse than stored blocks (5 bytes per 32 KiB block + framing)
    nblk = (len(data) + 32767) // 32768
    assert len(out) <= 8 + 2 + len(data) + 5 * nblk + 6
    if name.startswith(("ones", "zeros")):
        assert len(out) < 64 + len(data) // 100


@pytest.mark.parametrize("n", [0, 1, 3, 255, 256, 257, 8191, 8192, 8193, 3 * 8192 + 77, 1 << 20,
                               (1 << 20) + 12345])
def test_crc32c_device(ffcz, n):
    rng = np.random.default_rng(n)
    data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
    want = ffcz.ffcz.capi.load().ffcz_cuda_crc32c(data, len(data))
    assert ffcz.ffcz.crc32c_device(data) == want == O.crc32c(data)


def test_crc32c_device_tensor(ffcz):
    import torch
    x = torch.arange(1 << 18, dtype=torch.float64, device="cuda") * 1.37
    want = O.crc32c(x.cpu().numpy().tobytes())
    assert ffcz.ffcz.crc32c_device(x) == want


_NAMES = ("config1_c1.0", "config1_c0.4", "config2_rho32", "config3_frame256", "config4_comb32",
          "m8_32cube", "accept_05", "odd_12x10x9", "per_point_2d", "overflow_m24")
CASES = [c for c in cases.all_cases() if c.name in _NAMES]


def _same_edits(a, b):
    assert np.array_equal(a.spatial_flags, b.spatial_flags)
    assert np.array_equal(a.frequency_flags, b.frequency_flags)
    assert np.array_equal(a.spatial_codes, b.spatial_codes)
    assert np.array_equal(a.frequency_codes, b.frequency_codes)
    assert np.array_equal(a.escape_index, b.escape_index)
    assert np.array_equal(a.escape_frequency, b.escape_frequency)
    assert a.converged == b.converged


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_device_archive_decodes_to_reference_edits(ffcz, case):
    b = ffcz.DualBounds(case.E, case.Dre, case.Dim)
    z9 = ffcz.correct(case.original, case.decompressed, b, case.m, case.max_iters, case.precision,
                      zlib_level=9)
    dev = ffcz.correct(case.original, case.decompressed, b, case.m, case.max_iters,
                       case.precision)
    assert dev.timings_ms["t_archive_ms"] >= 0.0
    _same_edits(ref.archive_edits(dev.archive_bytes), ref.archive_edits(z9.archive_bytes))
    a, h = O.read_archive(dev.archive_bytes), O.read_archive(z9.archive_bytes)
    assert np.array_equal(a.frequency_codes, h.frequency_codes)
    # the reference's decoder reproduces the corrected field from either archive
    c_dev = ref.apply_archive(dev.archive_bytes, case.decompressed, case.precision)
    c_z9 = ref.apply_archive(z9.archive_bytes, case.decompressed, case.precision)
    assert np.array_equal(c_dev, c_z9)


@pytest.mark.parametrize("name", ["config2_rho32", "per_point_2d", "overflow_m24"])
def test_device_archive_device_bounds(ffcz, name):
    """Bounds resident on the device: the header CRC over the bound arrays runs on the GPU."""
    import torch
    case = next(c for c in CASES if c.name == name)
    t = lambda a: None if a is None else (a if np.isscalar(a) else
                                         torch.as_tensor(np.asarray(a, dtype=np.float64)).cuda())
    dt = torch.float32 if case.precision == "f32" else torch.float64
    o = torch.as_tensor(case.original).to(dt).cuda()
    d = torch.as_tensor(case.decompressed).to(dt).cuda()
    bd = ffcz.DualBounds(t(case.E), t(case.Dre), t(case.Dim))
    dev = ffcz.correct(o, d, bd, case.m, case.max_iters, case.precision)
    hb = ffcz.DualBounds(case.E, case.Dre, case.Dim)
    z9 = ffcz.correct(case.original, case.decompressed, hb, case.m, case.max_iters,
                      case.precision, zlib_level=9)
    _same_edits(ref.archive_edits(dev.archive_bytes), ref.archive_edits(z9.archive_bytes))
    # header bytes (bounds included) identical: only the stream framing differs
    hd, hz = O.read_archive(dev.archive_bytes), O.read_archive(z9.archive_bytes)
    assert hd.converged == hz.converged
