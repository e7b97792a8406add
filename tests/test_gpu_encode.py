"""Device edit encoding (csrc/encode.cu): the zigzag + blockwise canonical Huffman payload must be
byte-identical to the reference's huffman::encode (huffman.cpp:156-251, streams.cpp:13-15; the
oracle's restatement is pinned to the reference's archives), and archives written with it must be
byte-identical to the host-encoded ones at zlib level 9 and decodable at level 0 (stored)."""
import json
import os

import numpy as np
import pytest

import cases
from oracle import ffcz_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ffcz():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2601_01596_b200 as P
    return P


def _codes(kind, n, seed):
    rng = np.random.default_rng(seed)
    if kind == "laplace":
        return np.round(rng.laplace(0, 40, n)).astype(np.int32)
    if kind == "wide":
        return rng.integers(-2 ** 31, 2 ** 31 - 1, n, dtype=np.int64).astype(np.int32)
    if kind == "const":
        return np.full(n, -7, dtype=np.int32)
    if kind == "two":
        return rng.choice(np.array([0, 1], dtype=np.int32), n, p=[0.999, 0.001])
    if kind == "fib":   # skewed counts -> long codes
        w = np.array([int(1.6 ** k) + 1 for k in range(22)])
        return np.repeat(np.arange(22, dtype=np.int32) - 11, w)[:n]
    raise ValueError(kind)


@pytest.mark.parametrize("kind,n", [("laplace", 0), ("laplace", 1), ("laplace", 5),
                                    ("laplace", 65536), ("laplace", 65537), ("laplace", 300001),
                                    ("wide", 70000), ("const", 131072), ("two", 140000),
                                    ("fib", 50000)])
def test_huffman_payload_matches_reference(ffcz, kind, n):
    c = _codes(kind, n, 1234 + n)
    got = ffcz.ffcz.huffman_encode_device(c)
    want = O.huffman_encode(O.zigzag(c))
    assert got == want
    assert np.array_equal(O.unzigzag(O.huffman_decode(got)).astype(np.int32), c)


@pytest.mark.parametrize("mode", ["global"])
@pytest.mark.parametrize("kind,n", [("laplace", 300001), ("wide", 70000), ("fib", 50000),
                                    ("two", 140000)])
def test_huffman_table_paths(ffcz, monkeypatch, mode, kind, n):
    """The global-memory fallback of the code-length kernel (encode.cu block_table_global)
    gives the reference's payload too."""
    monkeypatch.setenv("FFCZ_HUFFMAN_TABLES", mode)
    c = _codes(kind, n, 99 + n)
    assert ffcz.ffcz.huffman_encode_device(c) == O.huffman_encode(O.zigzag(c))


_NAMES = ("config1_c1.0", "config1_c0.4", "config2_rho32", "config3_frame256", "config4_comb32",
          "m8_32cube", "accept_05", "odd_12x10x9")
CASES = [c for c in cases.all_cases() if c.name in _NAMES]


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_device_encoded_archive(ffcz, case):
    b = ffcz.DualBounds(case.E, case.Dre, case.Dim)
    host = ffcz.correct(case.original, case.decompressed, b, case.m, case.max_iters, case.precision,
                        zlib_level=9)
    dev9 = ffcz.correct(case.original, case.decompressed, b, case.m, case.max_iters,
                        case.precision, device_encode=True, zlib_level=9)
    assert dev9.archive_bytes == host.archive_bytes
    dev0 = ffcz.correct(case.original, case.decompressed, b, case.m, case.max_iters,
                        case.precision, device_encode=True, zlib_level=0)
    a, h = O.read_archive(dev0.archive_bytes), O.read_archive(host.archive_bytes)
    assert np.array_equal(a.spatial_flags, h.spatial_flags)
    assert np.array_equal(a.frequency_flags, h.frequency_flags)
    assert np.array_equal(a.spatial_codes, h.spatial_codes)
    assert np.array_equal(a.frequency_codes, h.frequency_codes)
    assert len(a.escapes) == len(h.escapes)
