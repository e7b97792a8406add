"""CPU restatement (numpy) of the reference FFCz correction path.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may import
this module, and only as the checker.  The product path (paper_2601_01596_b200) never imports it.

Every function restates one reference function (paths relative to /root/reference/proj/core):
the FFT is numpy's pocketfft c2c in FP64 standing in for FFTW (src/transform.cpp:20-50), the
rest is the same double arithmetic in the same order.  The restatement is pinned against the
reference itself: tests/golden/*.json are outputs of the unmodified reference compiled by
oracle/Makefile (script: tests/golden/make_golden.py), and tests/test_oracle.py checks this
module against them.
"""
from __future__ import annotations

import heapq
import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------------------------
# errors (include/ffcz/errors.hpp:9-48)


class FfczError(RuntimeError):
    pass


class ValidationError(FfczError):
    pass


class SymmetryError(FfczError):
    pass


class FormatError(FfczError):
    pass


# ---------------------------------------------------------------------------------------------
# bounds (include/ffcz/bounds.hpp:11-47, src/bounds.cpp)


@dataclass
class DualBounds:
    """E global or per point; Delta global or per component (Re, Im lanes, FULL spectrum)."""

    spatial: float | np.ndarray
    freq_re: float | np.ndarray
    freq_im: float | np.ndarray | None = None

    def __post_init__(self):
        if self.freq_im is None:
            self.freq_im = self.freq_re

    @property
    def spatial_per_point(self) -> bool:
        return isinstance(self.spatial, np.ndarray)

    @property
    def freq_per_component(self) -> bool:
        return isinstance(self.freq_re, np.ndarray)

    def E(self, shape):
        return np.broadcast_to(np.asarray(self.spatial, dtype=np.float64), shape)

    def Dre(self, shape):
        return np.broadcast_to(np.asarray(self.freq_re, dtype=np.float64), shape)

    def Dim(self, shape):
        return np.broadcast_to(np.asarray(self.freq_im, dtype=np.float64), shape)


def shrink_bounds(b: DualBounds, m: int) -> DualBounds:
    """src/bounds.cpp:74-85: every entry times (1 - 2^-m)."""
    if m < 1 or m > 24:
        raise ValidationError("shrink_bounds requires 1 <= m <= 24")
    f = 1.0 - 2.0 ** (-m)

    def s(v):
        return v * f if isinstance(v, np.ndarray) else float(v) * f

    return DualBounds(s(b.spatial), s(b.freq_re), s(b.freq_im))


# ---------------------------------------------------------------------------------------------
# transform (src/transform.cpp)


def forward_dft(x: np.ndarray) -> np.ndarray:
    """src/transform.cpp:45-50: unnormalised full c2c DFT of a real field (FP64)."""
    return np.fft.fftn(np.asarray(x, dtype=np.complex128))


def inverse_dft_complex(X: np.ndarray) -> np.ndarray:
    """src/transform.cpp:52-58: c2c inverse with 1/N."""
    return np.fft.ifftn(X)


def imaginary_residue_tolerance(precision: str, scale: float) -> float:
    """src/transform.cpp:60-62"""
    return (1e-6 if precision == "f32" else 1e-10) * scale


def inverse_dft(X: np.ndarray, precision: str = "f64") -> np.ndarray:
    """src/transform.cpp:64-80: inverse with the imaginary-residue gate."""
    c = inverse_dft_complex(X)
    max_re = float(np.max(np.abs(c.real))) if c.size else 0.0
    max_im = float(np.max(np.abs(c.imag))) if c.size else 0.0
    tol = imaginary_residue_tolerance(precision, max(max_re, 1e-300))
    if max_im > tol:
        raise SymmetryError(f"inverse_dft: imaginary residue {max_im} exceeds tolerance")
    return c.real.copy()


def brute_force_dft(x: np.ndarray) -> np.ndarray:
    """src/transform.cpp:82-103: O(N^2) summation (<= 4096 samples)."""
    x = np.asarray(x, dtype=np.float64)
    if x.size > 4096:
        raise ValidationError("brute_force_dft is a test oracle capped at 4096 samples")
    dims = x.shape
    coords = np.stack(np.unravel_index(np.arange(x.size), dims), axis=1).astype(np.float64)
    phase = np.zeros((x.size, x.size))
    for a, d in enumerate(dims):
        phase += np.outer(coords[:, a], coords[:, a]) / d
    return (np.exp(-2j * np.pi * phase) @ x.ravel()).reshape(dims)


def mirror_index_grid(dims) -> np.ndarray:
    """src/field.cpp:41-50: flat index of (dims - k) mod dims, for every k."""
    idx = [(-np.arange(d)) % d for d in dims]
    grids = np.meshgrid(*idx, indexing="ij")
    return np.ravel_multi_index(grids, dims).ravel()


# ---------------------------------------------------------------------------------------------
# projection (src/projection.cpp)


@dataclass
class ProjectionReport:
    iterations: int = 0
    active_spatial: int = 0
    active_frequency: int = 0
    converged: bool = False
    residual_f: float = 0.0
    residual_s: float = 0.0


def check_convergence(delta, Dre, Dim):
    """src/projection.cpp:29-52 -> (satisfied, violations, max_excess)."""
    peak = max(float(np.max(np.abs(delta.real))), float(np.max(np.abs(delta.imag))))
    tol = 1e-11 * peak
    ex = np.maximum(np.abs(delta.real) - Dre, np.abs(delta.imag) - Dim)
    bad = ex > tol
    nv = int(np.count_nonzero(bad))
    return nv == 0, nv, float(np.max(ex[bad])) if nv else 0.0


def _clamp(v, b):
    # std::clamp(v, -b, b) (projection.cpp:14-16)
    return np.where(v < -b, -b, np.where(b < v, b, v))


def project_onto_fcube(delta, Dre, Dim):
    """src/projection.cpp:54-66 -> (clipped, displacement)."""
    c = _clamp(delta.real, Dre) + 1j * _clamp(delta.imag, Dim)
    return c, c - delta


def project_onto_scube(eps, E):
    """src/projection.cpp:68-79 -> (clipped, displacement)."""
    c = _clamp(eps, E)
    return c, c - eps


def alternating_projection(eps0, bw: DualBounds, max_iters, slack=2.0 ** -20, precision="f64"):
    """src/projection.cpp:81-142 -> (S dense, F dense FULL spectrum, final eps, report)."""
    if max_iters < 1:
        raise ValidationError("alternating_projection: max_iters must be >= 1")
    eps0 = np.asarray(eps0, dtype=np.float64)
    shape = eps0.shape
    E, Dre, Dim = bw.E(shape), bw.Dre(shape), bw.Dim(shape)
    bad = np.flatnonzero(np.abs(eps0) > E * (1.0 + slack))
    if bad.size:
        raise ValidationError(
            f"alternating_projection: epsilon0 violates the spatial bound at index {bad[0]}")
    S = np.zeros(shape)
    F = np.zeros(shape, dtype=np.complex128)
    eps = eps0.copy()
    rep = ProjectionReport()
    passes = 0
    while True:
        delta = forward_dft(eps)
        ok, _, max_ex = check_convergence(delta, Dre, Dim)
        if ok:
            rep.converged, rep.residual_f = True, 0.0
            break
        if passes >= max_iters:
            rep.converged, rep.residual_f = False, max_ex
            break
        clipped, disp = project_onto_fcube(delta, Dre, Dim)
        F += disp
        eps = inverse_dft(clipped, precision)
        eps, sdisp = project_onto_scube(eps, E)
        S += sdisp
        passes += 1
    rep.iterations = max(passes, 1)
    rep.residual_s = float(max(0.0, np.max(np.abs(eps) - E)))
    rep.active_spatial = int(np.count_nonzero(S))
    rep.active_frequency = int(np.count_nonzero((F.real != 0) | (F.imag != 0)))
    return S, F, eps, rep


# ---------------------------------------------------------------------------------------------
# edit set (src/editset.cpp)


def half_dims(dims):
    """src/editset.cpp:9-13"""
    return tuple(dims[:-1]) + (dims[-1] // 2 + 1,)


def half_to_full_grid(dims) -> np.ndarray:
    """src/editset.cpp:19-23 for every half index."""
    h = half_dims(dims)
    coords = np.unravel_index(np.arange(int(np.prod(h))), h)
    return np.ravel_multi_index(coords, dims)


def llround(x: np.ndarray) -> np.ndarray:
    """std::llround: half away from zero."""
    return np.where(x >= 0, np.floor(x + 0.5), np.ceil(x - 0.5))


def _llround_exact(x: np.ndarray) -> np.ndarray:
    # floor(x + 0.5) can misround when x + 0.5 is inexact (|x| near 2^52 or x = 0.49999999999999994);
    # use the exact definition: r = trunc(x); r +/- 1 when |x - r| >= 0.5
    t = np.trunc(x)
    frac = np.abs(x - t)
    return np.where(frac >= 0.5, t + np.sign(x), t)


def quantize_value(v, step):
    """src/editset.cpp:76-84 (vectorised): llround(v / step) in int32 range."""
    v = np.asarray(v, dtype=np.float64)
    if not np.all(np.isfinite(v)):
        raise ValidationError("quantize: non-finite edit value")
    q = _llround_exact(v / step)
    if np.any(q > 2147483647) or np.any(q < -2147483648):
        raise ValidationError("quantize: index exceeds 32-bit range")
    return q.astype(np.int32)


def step_of(bound, m):
    """src/editset.cpp:31-41: ldexp(2*bound, -m)"""
    return np.ldexp(2.0 * np.asarray(bound, dtype=np.float64), -m)


# ---------------------------------------------------------------------------------------------
# streams + huffman (src/streams.cpp, src/huffman.cpp)


def zigzag(v: np.ndarray) -> np.ndarray:
    """src/streams.cpp:13-15"""
    v = np.asarray(v, dtype=np.int32).astype(np.int64)
    return (((v << 1) ^ (v >> 31)) & 0xFFFFFFFF).astype(np.uint32)


def unzigzag(u: np.ndarray) -> np.ndarray:
    """src/streams.cpp:17-19"""
    u = np.asarray(u, dtype=np.uint32).astype(np.int64)
    return ((u >> 1) ^ (-(u & 1))).astype(np.int32)


def _code_lengths(syms, counts):
    """src/huffman.cpp:74-120: pair the two lightest subtrees, tie-break (weight, min symbol)."""
    n = len(syms)
    if n == 1:
        return [1]
    left, right = [-1] * n, [-1] * n
    heap = [(int(counts[i]), int(syms[i]), i) for i in range(n)]
    heapq.heapify(heap)
    while len(heap) > 1:
        wa, ta, a = heapq.heappop(heap)
        wb, tb, b = heapq.heappop(heap)
        left.append(a)
        right.append(b)
        heapq.heappush(heap, (wa + wb, min(ta, tb), len(left) - 1))
    lens = [0] * n
    stack = [(heap[0][2], 0)]
    while stack:
        i, d = stack.pop()
        if left[i] < 0:
            lens[i] = d
        else:
            stack.append((left[i], d + 1))
            stack.append((right[i], d + 1))
    return lens


def _canonical(syms, lens):
    """src/huffman.cpp:124-154 -> [(symbol, length, code)] in canonical order."""
    order = sorted(range(len(syms)), key=lambda i: (lens[i], int(syms[i])))
    out, code, prev = [], 0, 0
    for i in order:
        code <<= lens[i] - prev
        out.append((int(syms[i]), lens[i], code))
        code += 1
        prev = lens[i]
    return out


def huffman_encode(symbols: np.ndarray) -> bytes:
    """src/huffman.cpp:156-251 (encode side)."""
    symbols = np.asarray(symbols, dtype=np.uint32)
    out = bytearray(struct.pack("<Q", symbols.size))
    for s0 in range(0, symbols.size, 1 << 16):
        blk = symbols[s0:s0 + (1 << 16)]
        syms, counts = np.unique(blk, return_counts=True)
        table = _canonical(syms, _code_lengths(syms, counts))
        out += struct.pack("<II", blk.size, len(table))
        for s, ln, _ in table:
            out += struct.pack("<IB", s, ln)
        lut = {s: (c, ln) for s, ln, c in table}
        bits = "".join(format(lut[int(v)][0], f"0{lut[int(v)][1]}b") for v in blk)
        nbits = len(bits)
        bits += "0" * (-nbits % 8)
        out += struct.pack("<Q", nbits)
        out += int(bits, 2).to_bytes(len(bits) // 8, "big") if bits else b""
    return bytes(out)


def huffman_decode(data: bytes) -> np.ndarray:
    """src/huffman.cpp:156-262 (decode side)."""
    off = 0

    def rd(fmt):
        nonlocal off
        sz = struct.calcsize(fmt)
        if off + sz > len(data):
            raise FormatError("huffman: truncated stream")
        v = struct.unpack_from(fmt, data, off)
        off += sz
        return v

    (total,) = rd("<Q")
    out = []
    while len(out) < total:
        n, distinct = rd("<II")
        if distinct == 0 or distinct > n:
            raise FormatError("huffman: bad table size")
        syms, lens = [], []
        for _ in range(distinct):
            s, ln = rd("<IB")
            if ln == 0 or ln > 32:
                raise FormatError("huffman: bad code length")
            syms.append(s)
            lens.append(ln)
        table = _canonical(syms, lens)
        lut = {(ln, c): s for s, ln, c in table}
        (nbits,) = rd("<Q")
        nbytes = (nbits + 7) // 8
        if off + nbytes > len(data):
            raise FormatError("huffman: truncated bitstream")
        bits = bin(int.from_bytes(data[off:off + nbytes], "big"))[2:].zfill(nbytes * 8)[:nbits]
        off += nbytes
        pos, maxlen = 0, max(lens)
        for _ in range(n):
            code, ln = 0, 0
            while True:
                if ln >= maxlen or pos >= nbits:
                    raise FormatError("huffman: invalid code")
                code = (code << 1) | (bits[pos] == "1")
                pos += 1
                ln += 1
                if (ln, code) in lut:
                    out.append(lut[(ln, code)])
                    break
    if len(out) != total or off != len(data):
        raise FormatError("huffman: stream length mismatch")
    return np.asarray(out, dtype=np.uint32)


def outer_compress(raw: bytes, level: int = 9) -> bytes:
    """src/streams.cpp:21-32: u64 raw size + zlib compress2."""
    return struct.pack("<Q", len(raw)) + zlib.compress(raw, level)


def outer_decompress(frame: bytes) -> bytes:
    """src/streams.cpp:34-46"""
    if len(frame) < 8:
        raise FormatError("outer frame truncated")
    (n,) = struct.unpack_from("<Q", frame)
    if n == 0:
        return b""
    try:
        raw = zlib.decompress(frame[8:])
    except zlib.error as e:
        raise FormatError("outer_decompress failed: corrupt frame") from e
    if len(raw) != n:
        raise FormatError("outer_decompress failed: corrupt frame")
    return raw


def pack_flags(flags: np.ndarray) -> bytes:
    """include/ffcz/bitvector.hpp: LSB-first bytes."""
    return np.packbits(np.asarray(flags, dtype=bool), bitorder="little").tobytes()


def unpack_flags(b: bytes, nbits: int) -> np.ndarray:
    return np.unpackbits(np.frombuffer(b, dtype=np.uint8), bitorder="little")[:nbits].astype(bool)


def crc32c(data: bytes) -> int:
    """src/archive.cpp:16-21, 61-71 (poly 0x82F63B78)."""
    table = []
    for i in range(256):
        c = i
        for _ in range(8):
            c = (c >> 1) ^ (0x82F63B78 if c & 1 else 0)
        table.append(c)
    crc = 0xFFFFFFFF
    for b in data:
        crc = (crc >> 8) ^ table[(crc ^ b) & 0xFF]
    return crc ^ 0xFFFFFFFF


# ---------------------------------------------------------------------------------------------
# archive (src/archive.cpp, docs/FORMAT.md)


@dataclass
class Escape:
    frequency: bool
    index: int
    re: float
    im: float = 0.0


@dataclass
class Archive:
    dims: tuple
    precision: str
    converged: bool
    bounds: DualBounds
    m: int
    spatial_flags: np.ndarray
    frequency_flags: np.ndarray
    spatial_codes: np.ndarray
    frequency_codes: np.ndarray
    escapes: list = field(default_factory=list)


def write_archive(a: Archive, level: int = 9) -> bytes:
    """src/archive.cpp:73-135."""
    return write_archive_raw_flags(a, pack_flags(a.spatial_flags), pack_flags(a.frequency_flags),
                                   level)


def write_archive_raw_flags(a: Archive, sflag_bytes: bytes, fflag_bytes: bytes,
                            level: int = 9) -> bytes:
    """write_archive with the flag streams given as raw bytes (test hook for malformed or
    padding-bit archives); the header counts stay the flags' own counts (a.spatial_flags /
    a.frequency_flags)."""
    sf = outer_compress(bytes(sflag_bytes), level)
    si = outer_compress(huffman_encode(zigzag(a.spatial_codes)), level)
    ff = outer_compress(bytes(fflag_bytes), level)
    fi = outer_compress(huffman_encode(zigzag(a.frequency_codes)), level)
    w = bytearray(b"FFCZ") + struct.pack("<HB", 1, len(a.dims))
    for d in a.dims:
        w += struct.pack("<Q", d)
    tags = (1 if a.bounds.spatial_per_point else 0) | (2 if a.bounds.freq_per_component else 0) | (
        4 if a.converged else 0)
    w += struct.pack("<BB", 0 if a.precision == "f32" else 1, tags)
    if a.bounds.spatial_per_point:
        w += np.asarray(a.bounds.spatial, dtype="<f8").ravel().tobytes()
    else:
        w += struct.pack("<d", a.bounds.spatial)
    if a.bounds.freq_per_component:
        w += np.asarray(a.bounds.freq_re, dtype="<f8").ravel().tobytes()
        w += np.asarray(a.bounds.freq_im, dtype="<f8").ravel().tobytes()
    else:
        w += struct.pack("<d", a.bounds.freq_re)
    w += struct.pack("<B", a.m)
    w += struct.pack("<7Q", int(np.count_nonzero(a.spatial_flags)),
                     int(np.count_nonzero(a.frequency_flags)), len(sf), len(ff), len(si), len(fi),
                     len(a.escapes))
    w += struct.pack("<I", crc32c(bytes(w)))
    w += sf + ff + si + fi
    for e in a.escapes:
        w += struct.pack("<Qd", e.index | ((1 << 63) if e.frequency else 0), e.re)
        if e.frequency:
            w += struct.pack("<d", e.im)
    return bytes(w)


def read_archive(data: bytes) -> Archive:
    """src/archive.cpp:137-225 (codes kept as integers; dequantise with dequantize())."""
    off = 0

    def rd(fmt):
        nonlocal off
        sz = struct.calcsize(fmt)
        if off + sz > len(data):
            raise FormatError("archive truncated")
        v = struct.unpack_from(fmt, data, off)
        off += sz
        return v

    if data[:4] != b"FFCZ" or len(data) < 4:
        raise FormatError("read_archive: bad magic")
    off = 4
    (ver,) = rd("<H")
    if ver != 1:
        raise FormatError("read_archive: unsupported version")
    (ndim,) = rd("<B")
    if ndim < 1 or ndim > 3:
        raise FormatError("read_archive: bad dimensionality")
    dims = tuple(rd("<Q")[0] for _ in range(ndim))
    if any(d == 0 for d in dims):
        raise FormatError("read_archive: zero extent")
    N = int(np.prod(dims))
    prec, tags = rd("<BB")
    if prec > 1:
        raise FormatError("read_archive: bad precision tag")

    def doubles(n):
        nonlocal off
        if off + 8 * n > len(data):
            raise FormatError("archive truncated")
        v = np.frombuffer(data, dtype="<f8", count=n, offset=off).copy()
        off += 8 * n
        return v

    E = doubles(N).reshape(dims) if tags & 1 else rd("<d")[0]
    if tags & 2:
        dre, dim_ = doubles(N).reshape(dims), doubles(N).reshape(dims)
    else:
        dre = dim_ = rd("<d")[0]
    (m,) = rd("<B")
    if m < 1 or m > 24:
        raise FormatError("read_archive: bad quantization width")
    n_s, n_f, lsf, lff, lsi, lfi, n_esc = rd("<7Q")
    hlen = off
    (crc,) = rd("<I")
    if crc32c(data[:hlen]) != crc:
        raise FormatError("read_archive: header checksum mismatch")

    def take(n):
        nonlocal off
        if off + n > len(data):
            raise FormatError("archive truncated")
        b = data[off:off + n]
        off += n
        return b

    sf, ff, si, fi = take(lsf), take(lff), take(lsi), take(lfi)
    hn = int(np.prod(half_dims(dims)))
    sflags_raw = outer_decompress(sf)
    fflags_raw = outer_decompress(ff)
    if len(sflags_raw) != (N + 7) // 8 or len(fflags_raw) != (hn + 7) // 8:
        raise FormatError("decode_streams: flag payload length mismatch")
    sflags, fflags = unpack_flags(sflags_raw, N), unpack_flags(fflags_raw, hn)
    scodes = unzigzag(huffman_decode(outer_decompress(si)))
    fcodes = unzigzag(huffman_decode(outer_decompress(fi)))
    if np.count_nonzero(sflags) != n_s or scodes.size != n_s:
        raise FormatError("read_archive: spatial edit count mismatch")
    if np.count_nonzero(fflags) != n_f or fcodes.size != 2 * n_f:
        raise FormatError("read_archive: frequency edit count mismatch")
    escapes = []
    for _ in range(n_esc):
        (packed,) = rd("<Q")
        isf = bool(packed >> 63)
        idx = packed & ~(1 << 63)
        (re,) = rd("<d")
        im = rd("<d")[0] if isf else 0.0
        if idx >= (hn if isf else N):
            raise FormatError("read_archive: escape index out of range")
        escapes.append(Escape(isf, idx, re, im))
    if off != len(data):
        raise FormatError("read_archive: trailing bytes")
    return Archive(dims, "f32" if prec == 0 else "f64", bool(tags & 4), DualBounds(E, dre, dim_), m,
                   sflags, fflags, scodes, fcodes, escapes)


def dequantize(a: Archive):
    """Decoder view (src/archive.cpp:206-211, 227-260): dense spatial (N) and half frequency."""
    dims = a.dims
    N = int(np.prod(dims))
    hn = int(np.prod(half_dims(dims)))
    spat = np.zeros(N)
    sidx = np.flatnonzero(a.spatial_flags)
    spat[sidx] = a.spatial_codes.astype(np.float64) * step_of(a.bounds.E(dims).ravel()[sidx], a.m)
    half = np.zeros(hn, dtype=np.complex128)
    fidx = np.flatnonzero(a.frequency_flags)
    full_k = half_to_full_grid(dims)[fidx]
    sre = step_of(a.bounds.Dre(dims).ravel()[full_k], a.m)
    sim = step_of(a.bounds.Dim(dims).ravel()[full_k], a.m)
    half[fidx] = a.frequency_codes[0::2].astype(np.float64) * sre + 1j * (
        a.frequency_codes[1::2].astype(np.float64) * sim)
    for e in a.escapes:
        if e.frequency:
            half[e.index] = complex(e.re, e.im)
        else:
            spat[e.index] = e.re
    return spat.reshape(dims), half


def expand_half(dims, half: np.ndarray) -> np.ndarray:
    """src/archive.cpp:251-258: half -> full spectrum by conjugate mirror."""
    N = int(np.prod(dims))
    full = np.zeros(N, dtype=np.complex128)
    h2f = half_to_full_grid(dims)
    full[h2f] = half
    inhalf = np.zeros(N, dtype=bool)
    inhalf[h2f] = True
    mir = mirror_index_grid(dims)
    k = np.flatnonzero(~inhalf)
    full_of_mirror = full[mir[k]]
    full[k] = np.conj(full_of_mirror)
    return full.reshape(dims)


def apply_edits(decompressed: np.ndarray, a: Archive) -> np.ndarray:
    """src/archive.cpp:262-273"""
    spat, half = dequantize(a)
    fpart = inverse_dft(expand_half(a.dims, half), a.precision)
    return decompressed + spat + fpart


def verify_bounds(original, corrected, b: DualBounds):
    """src/archive.cpp:275-297 -> (ok, max_spatial_excess, max_freq_excess)."""
    shape = original.shape
    eps = corrected - original
    ex = np.abs(eps) - b.E(shape)
    ms = float(np.max(ex[ex > 0])) if np.any(ex > 0) else 0.0
    d = forward_dft(eps)
    exf = np.maximum(np.abs(d.real) - b.Dre(shape), np.abs(d.imag) - b.Dim(shape))
    mf = float(np.max(exf[exf > 0])) if np.any(exf > 0) else 0.0
    return ms == 0.0 and mf == 0.0, ms, mf


# ---------------------------------------------------------------------------------------------
# pipeline (src/pipeline.cpp)


@dataclass
class CorrectionResult:
    archive_bytes: bytes
    report: ProjectionReport
    escape_count: int
    verify_ok: bool
    verify_max_spatial_excess: float
    verify_max_freq_excess: float
    archive: Archive
    corrected: np.ndarray
    escape_rounds: int


def correct(original, decompressed, b: DualBounds, m: int = 16, max_iters: int = 1000,
            precision: str = "f64", level: int = 9) -> CorrectionResult:
    """src/pipeline.cpp:26-178."""
    original = np.asarray(original, dtype=np.float64)
    decompressed = np.asarray(decompressed, dtype=np.float64)
    dims = original.shape
    N = original.size
    eps0 = decompressed - original                                        # :31
    E0 = b.E(dims)
    bad = np.flatnonzero(np.abs(eps0) > E0 * (1.0 + 2.0 ** -20))           # :33-37
    if bad.size:
        raise ValidationError(
            "correct: decompressed data violates the declared spatial bound at index "
            f"{bad[0]}")
    working = shrink_bounds(b, m)                                          # :39
    slack = 1.0 / (1.0 - 2.0 ** -m) - 1.0 + 2.0 ** -20                     # :42
    S, F, final_eps, rep = alternating_projection(eps0, working, max_iters, slack, precision)

    # compaction + restrict_to_half (:46-50)
    h2f = half_to_full_grid(dims)
    Fh = F.ravel()[h2f]
    Sflat = S.ravel()
    sflags = Sflat != 0.0
    fflags = (Fh.real != 0.0) | (Fh.imag != 0.0)
    esc = {}  # (bool, index) -> complex, ordered like std::map at the end
    # overflow escapes (:57-88)
    kmax = 2147483520.0
    sstep = step_of(E0.ravel(), m)
    sidx = np.flatnonzero(sflags)
    ovf = np.abs(Sflat[sidx]) / sstep[sidx] > kmax
    for i in sidx[ovf]:
        esc[(False, int(i))] = complex(Sflat[i], 0.0)
    sflags[sidx[ovf]] = False
    Dre0, Dim0 = b.Dre(dims).ravel(), b.Dim(dims).ravel()
    fidx = np.flatnonzero(fflags)
    fre_step = step_of(Dre0[h2f[fidx]], m)
    fim_step = step_of(Dim0[h2f[fidx]], m)
    fovf = (np.abs(Fh[fidx].real) / fre_step > kmax) | (np.abs(Fh[fidx].imag) / fim_step > kmax)
    for i in fidx[fovf]:
        esc[(True, int(i))] = complex(Fh[i])
    fflags[fidx[fovf]] = False
    # quantize -> dequantize (decoder view, :91-106)
    sidx = np.flatnonzero(sflags)
    scodes = quantize_value(Sflat[sidx], sstep[sidx])
    spat_dq = np.zeros(N)
    spat_dq[sidx] = scodes.astype(np.float64) * sstep[sidx]
    fidx = np.flatnonzero(fflags)
    sre, sim = step_of(Dre0[h2f[fidx]], m), step_of(Dim0[h2f[fidx]], m)
    cre = quantize_value(Fh[fidx].real, sre)
    cim = quantize_value(Fh[fidx].imag, sim)
    fcodes = np.empty(2 * fidx.size, dtype=np.int32)
    fcodes[0::2], fcodes[1::2] = cre, cim
    freq_dq = np.zeros(h2f.size, dtype=np.complex128)
    freq_dq[fidx] = cre.astype(np.float64) * sre + 1j * (cim.astype(np.float64) * sim)

    rounds = 0
    if rep.converged:                                                      # :111-163
        delta_star = forward_dft(final_eps).ravel()
        hn = h2f.size
        mir = mirror_index_grid(dims)
        full_to_half = np.full(N, -1, dtype=np.int64)
        full_to_half[h2f] = np.arange(hn)
        hmir = full_to_half[mir[h2f]]
        for _ in range(32):
            rounds += 1
            spat_cur = spat_dq.copy()
            freq_cur = freq_dq.copy()
            for (isf, i), v in esc.items():
                if isf:
                    freq_cur[i] = v
                else:
                    spat_cur[i] = v.real
            fsp = inverse_dft_complex(expand_half(dims, freq_cur)).real.ravel()
            eps_tilde = eps0.ravel() + spat_cur + fsp
            dt = forward_dft(eps_tilde.reshape(dims)).ravel()
            clean = True
            dth = dt[h2f]
            viol = (np.abs(dth.real) > Dre0[h2f]) | (np.abs(dth.imag) > Dim0[h2f])
            for h in np.flatnonzero(viol):
                clean = False
                k = h2f[h]
                rep_v = freq_cur[h] + (delta_star[k] - dt[k])
                esc[(True, int(h))] = rep_v
                hm = hmir[h]
                if hm >= 0 and hm != h:
                    esc[(True, int(hm))] = np.conj(rep_v)
            sv = np.flatnonzero(np.abs(eps_tilde) > E0.ravel())
            for n in sv:
                clean = False
                esc[(False, int(n))] = complex(spat_cur[n] + (final_eps.ravel()[n] - eps_tilde[n]))
            if clean:
                break
    escapes = [Escape(isf, i, v.real, v.imag if isf else 0.0) for (isf, i), v in sorted(esc.items())]
    arch = Archive(dims, precision, rep.converged, b, m, sflags, fflags, scodes, fcodes, escapes)
    data = write_archive(arch, level)
    corrected = apply_edits(decompressed, read_archive(data))
    ok, ms, mf = verify_bounds(original, corrected, b)
    return CorrectionResult(data, rep, len(escapes), ok, ms, mf, arch, corrected, rounds)


# ---------------------------------------------------------------------------------------------
# helpers for the BASELINE configs


class UndefinedMetric(ValueError):
    """errors.hpp undefined_metric_error."""


def power_spectrum(field: np.ndarray):
    """src/metrics.cpp:11-62 -> (k_bins, power, counts, mean_fallback, mean)."""
    x = np.asarray(field, dtype=np.float64)
    mean = float(np.sum(x)) / x.size
    max_abs = float(np.max(np.abs(x)))
    fallback = abs(mean) <= 1e-12 * max_abs                       # metrics.cpp:21-24
    fl = (x - mean) if fallback else (x - mean) / mean
    X = forward_dft(fl)
    max_bin = int(np.floor(np.sqrt(sum(float(d // 2) ** 2 for d in x.shape)) + 0.5))
    r2 = np.zeros(x.shape)
    for a, d in enumerate(x.shape):
        c = np.arange(d, dtype=np.float64)
        c[np.arange(d) > d // 2] -= d                                # metrics.cpp:48-52
        sh = [1] * x.ndim
        sh[a] = d
        r2 = r2 + (c * c).reshape(sh)
    bins = np.floor(np.sqrt(r2) + 0.5).astype(np.int64).ravel()      # llround, non-negative
    power = np.bincount(bins, weights=np.abs(X.ravel()) ** 2, minlength=max_bin + 1)
    counts = np.bincount(bins, minlength=max_bin + 1).astype(np.uint64)
    return np.arange(max_bin + 1), power, counts, fallback, mean


def psnr(original: np.ndarray, reconstructed: np.ndarray) -> float:
    """src/metrics.cpp:64-79."""
    o = np.asarray(original, dtype=np.float64)
    d = np.asarray(reconstructed, dtype=np.float64) - o
    se = float(np.sum(d * d))
    if se == 0.0:
        return float("inf")
    lo, hi = float(o.min()), float(o.max())
    if hi == lo:
        raise UndefinedMetric("psnr: constant original has no defined range")
    return 20.0 * np.log10((hi - lo) / np.sqrt(se / o.size))


def ssnr(X: np.ndarray, Y: np.ndarray) -> float:
    """src/metrics.cpp:81-93 on FULL spectra."""
    signal = float(np.sum(np.abs(X) ** 2))
    noise = float(np.sum(np.abs(X - Y) ** 2))
    if signal == 0.0:
        raise UndefinedMetric("ssnr: zero-energy original spectrum")
    return float("inf") if noise == 0.0 else 10.0 * np.log10(signal / noise)


def rfe(delta: np.ndarray, X: np.ndarray) -> np.ndarray:
    """src/metrics.cpp:95-105."""
    mx = float(np.max(np.abs(X)))
    if mx == 0.0:
        raise UndefinedMetric("rfe: all-zero original spectrum")
    return np.abs(delta) / mx


def metrics(original: np.ndarray, reconstructed: np.ndarray):
    """What `ffcz metrics` reports (proj/tools/ffcz.cpp:246-256): psnr, ssnr, max rfe, max |eps|."""
    o = np.asarray(original, dtype=np.float64)
    r = np.asarray(reconstructed, dtype=np.float64)
    X, Y = forward_dft(o), forward_dft(r)
    eps = r - o
    p = psnr(o, r)
    s = ssnr(X, Y)
    m = float(np.max(rfe(forward_dft(eps), X)))
    return p, s, m, float(np.max(np.abs(eps)))


def spectrum_bound_to_freq_bounds(X: np.ndarray, rho: float) -> np.ndarray:
    """src/metrics.cpp:107-128 -> per-component Delta (Re lane == Im lane)."""
    mag = np.abs(X)
    floor = max(1e-12 * float(mag.max()), 1e-300)
    scale = (np.sqrt(1.0 + rho) - 1.0) / np.sqrt(2.0)
    mirror = mirror_index_grid(X.shape)
    mm = np.minimum(mag.ravel(), mag.ravel()[mirror]).reshape(X.shape)
    return np.maximum(mm * scale, floor)
