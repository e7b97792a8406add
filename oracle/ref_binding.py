"""ctypes binding to oracle/_ref/libffcz_ref.so (the UNMODIFIED CPU reference + FFTW-API shim,
built by oracle/Makefile).  TEST INFRASTRUCTURE ONLY: used by tests/golden/make_golden.py,
tests/test_oracle.py and bench.py's reference / cpu_baseline legs.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# FFT provider behind the reference's fftw_* calls (oracle/Makefile): "mkl" = MKL DFTI
# (shim/fftw_mkl.cpp, FFTW-class speed; the default when built), "radix2" = the dependency-free
# stand-in (shim/fftw_shim.cpp).  FFCZ_REF_FFT selects; the choice is reported by fft_backend().
_LIBS = {"radix2": os.path.join(HERE, "_ref", "libffcz_ref.so"),
         "mkl": os.path.join(HERE, "_ref", "libffcz_ref_mkl.so")}


def fft_backend() -> str:
    want = os.environ.get("FFCZ_REF_FFT", "")
    if want in _LIBS:
        return want
    return "mkl" if os.path.exists(_LIBS["mkl"]) else "radix2"


LIB_PATH = _LIBS[fft_backend()]

_ERRS = {1: "ValidationError", 2: "SymmetryError", 3: "FormatError", 4: "IoError", 5: "Error",
         6: "Exception"}


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_ERRS.get(code, code)}: {msg}")
        self.code = code
        self.kind = _ERRS.get(code, str(code))


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("active_spatial", C.c_uint64),
                ("active_frequency", C.c_uint64), ("converged", C.c_int32),
                ("residual_f", C.c_double), ("residual_s", C.c_double),
                ("wall_time_s", C.c_double)]


class _CorrectOut(C.Structure):
    _fields_ = [("report", _Report), ("escape_count", C.c_uint64), ("verify_ok", C.c_int32),
                ("verify_max_spatial_excess", C.c_double), ("verify_max_freq_excess", C.c_double),
                ("archive", C.POINTER(C.c_uint8)), ("archive_len", C.c_uint64),
                ("correct_wall_s", C.c_double)]


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{LIB_PATH} missing: run `make -C oracle` where /root/reference exists")
        _lib = C.CDLL(LIB_PATH)
        _lib.ffcz_ref_last_error.restype = C.c_char_p
    return _lib


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ffcz_ref_last_error().decode())


def _dims(shape):
    return (C.c_uint64 * 3)(*shape, *([0] * (3 - len(shape))))


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _bounds_args(shape, E, Dre, Dim):
    e_arr = _f64(E).ravel() if isinstance(E, np.ndarray) else None
    re_arr = _f64(Dre).ravel() if isinstance(Dre, np.ndarray) else None
    im_arr = _f64(Dim if Dim is not None else Dre).ravel() if isinstance(Dre, np.ndarray) else None
    args = [C.c_int(1 if e_arr is not None else 0), C.c_double(0.0 if e_arr is not None else float(E)),
            _dp(e_arr), C.c_int(1 if re_arr is not None else 0),
            C.c_double(0.0 if re_arr is not None else float(Dre)), _dp(re_arr), _dp(im_arr)]
    return args, (e_arr, re_arr, im_arr)


@dataclass
class RefReport:
    iterations: int
    active_spatial: int
    active_frequency: int
    converged: bool
    residual_f: float
    residual_s: float
    wall_time_s: float


def _rep(r):
    return RefReport(int(r.iterations), int(r.active_spatial), int(r.active_frequency),
                     bool(r.converged), float(r.residual_f), float(r.residual_s),
                     float(r.wall_time_s))


@dataclass
class RefCorrect:
    report: RefReport
    escape_count: int
    verify_ok: bool
    verify_max_spatial_excess: float
    verify_max_freq_excess: float
    archive: bytes
    correct_wall_s: float


def correct(original, decompressed, E, Dre, Dim=None, m=16, max_iters=1000, precision="f64"):
    """ffcz::correct (pipeline.hpp:22-24) of the reference."""
    o, d = _f64(original), _f64(decompressed)
    bargs, keep = _bounds_args(o.shape, E, Dre, Dim)
    out = _CorrectOut()
    rc = lib().ffcz_ref_correct(C.c_int(o.ndim), _dims(o.shape), C.c_int(0 if precision == "f32" else 1),
                                _dp(o.ravel()), _dp(d.ravel()), *bargs, C.c_int(m),
                                C.c_uint64(max_iters), C.byref(out))
    _check(rc)
    # (C.string_at takes an int size: a 512^3 rho-mode archive is 2.8 GB)
    data = np.ctypeslib.as_array(out.archive, shape=(max(1, int(out.archive_len)),))[
        : int(out.archive_len)].tobytes() if out.archive_len else b""
    lib().ffcz_ref_free(out.archive)
    return RefCorrect(_rep(out.report), int(out.escape_count), bool(out.verify_ok),
                      float(out.verify_max_spatial_excess), float(out.verify_max_freq_excess), data,
                      float(out.correct_wall_s))


def alternating_projection(eps0, E, Dre, Dim=None, max_iters=1000, slack=2.0 ** -20,
                           precision="f64"):
    """ffcz::alternating_projection (projection.hpp:65-70) -> (S, F full, eps, report)."""
    e = _f64(eps0)
    bargs, keep = _bounds_args(e.shape, E, Dre, Dim)
    S = np.zeros(e.shape)
    F = np.zeros(e.shape, dtype=np.complex128)
    eps = np.zeros(e.shape)
    rep = _Report()
    rc = lib().ffcz_ref_alternating_projection(
        C.c_int(e.ndim), _dims(e.shape), C.c_int(0 if precision == "f32" else 1), _dp(e.ravel()),
        *bargs, C.c_uint64(max_iters), C.c_double(slack), _dp(S),
        F.ctypes.data_as(C.POINTER(C.c_double)), _dp(eps), C.byref(rep))
    _check(rc)
    return S, F, eps, _rep(rep)


def forward_dft(x):
    x = _f64(x)
    out = np.zeros(x.shape, dtype=np.complex128)
    _check(lib().ffcz_ref_forward_dft(C.c_int(x.ndim), _dims(x.shape), _dp(x.ravel()),
                                      out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def brute_force_dft(x):
    x = _f64(x)
    out = np.zeros(x.shape, dtype=np.complex128)
    _check(lib().ffcz_ref_brute_force_dft(C.c_int(x.ndim), _dims(x.shape), _dp(x.ravel()),
                                          out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


def apply_archive(data: bytes, decompressed, precision="f64"):
    d = _f64(decompressed)
    out = np.zeros(d.shape)
    buf = (C.c_uint8 * len(data)).from_buffer_copy(data)
    _check(lib().ffcz_ref_apply_archive(buf, C.c_uint64(len(data)), C.c_int(d.ndim), _dims(d.shape),
                                        C.c_int(0 if precision == "f32" else 1), _dp(d.ravel()),
                                        _dp(out)))
    return out


def synth_field(kind: int, shape, seed: int, param: float):
    out = np.zeros(shape)
    _check(lib().ffcz_ref_synth_field(C.c_int(kind), C.c_int(len(shape)), _dims(shape),
                                      C.c_uint64(seed), C.c_double(param), _dp(out)))
    return out


def rho_bounds(original, rho):
    o = _f64(original)
    out = np.zeros(o.shape)
    _check(lib().ffcz_ref_rho_bounds(C.c_int(o.ndim), _dims(o.shape), _dp(o.ravel()),
                                     C.c_double(rho), _dp(out)))
    return out


class _ArchiveEdits(C.Structure):
    _fields_ = [("spatial_flags", C.POINTER(C.c_uint8)), ("spatial_flag_bytes", C.c_uint64),
                ("frequency_flags", C.POINTER(C.c_uint8)), ("frequency_flag_bytes", C.c_uint64),
                ("spatial_codes", C.POINTER(C.c_int32)), ("n_spatial", C.c_uint64),
                ("frequency_codes", C.POINTER(C.c_int32)), ("n_frequency", C.c_uint64),
                ("escape_index", C.POINTER(C.c_uint64)), ("escape_freq", C.POINTER(C.c_int32)),
                ("n_escapes", C.c_uint64), ("converged", C.c_int32)]


@dataclass
class RefEdits:
    spatial_flags: np.ndarray     # packed LSB-first bytes, as the archive carries them
    frequency_flags: np.ndarray
    spatial_codes: np.ndarray     # int32
    frequency_codes: np.ndarray   # int32, interleaved Re, Im
    escape_index: np.ndarray      # uint64, the reference's std::map order
    escape_frequency: np.ndarray  # int32 (1 = frequency entry)
    converged: bool


def archive_edits(data: bytes) -> RefEdits:
    """The reference's read_archive (archive.cpp:137-225) of `data` as flag bytes / int32 codes /
    escape indices (codes re-quantised exactly from the dequantised values)."""
    buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data if data else b"\0")
    out = _ArchiveEdits()
    _check(lib().ffcz_ref_archive_edits(buf, C.c_uint64(len(data)), C.byref(out)))

    def take(p, n, dt):
        a = np.ctypeslib.as_array(p, shape=(max(1, n),))[:n].astype(dt, copy=True)
        lib().ffcz_ref_free(C.cast(p, C.c_void_p))
        return a

    return RefEdits(take(out.spatial_flags, out.spatial_flag_bytes, np.uint8),
                    take(out.frequency_flags, out.frequency_flag_bytes, np.uint8),
                    take(out.spatial_codes, out.n_spatial, np.int32),
                    take(out.frequency_codes, 2 * out.n_frequency, np.int32),
                    take(out.escape_index, out.n_escapes, np.uint64),
                    take(out.escape_freq, out.n_escapes, np.int32), bool(out.converged))
