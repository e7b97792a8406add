"""Python host mirror of the reference's public API for the correction path, running on the B200
engine through the C-ABI (include/ffcz_cuda.h).

Same names, argument meaning and error behaviour as the reference C++ API:
  correct(original, decompressed, bounds, m=16, max_iters=1000)   pipeline.hpp:22-24
  alternating_projection(eps0, bounds_working, max_iters, slack)  projection.hpp:65-70
  forward_dft(x), inverse_dft(X, precision)                       transform.hpp:7-17
Errors raise ValidationError / SymmetryError / FormatError like the reference's exception
classes (errors.hpp:9-48).  There is no CPU fallback: without a GPU or the built library the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _capi as capi

# zlib_level value of correct(): the archive's streams are encoded on the device
# (include/ffcz_cuda.h FFCZ_OUTER_DEVICE)
OUTER_DEVICE = -1


class FfczError(RuntimeError):
    pass


class ValidationError(FfczError):
    pass


class SymmetryError(FfczError):
    pass


class FormatError(FfczError):
    pass


class IoError(FfczError):
    pass


class CudaError(FfczError):
    pass


class UnsupportedError(FfczError):
    pass


class UndefinedMetricError(FfczError):
    """ffcz::undefined_metric_error (errors.hpp): psnr / ssnr / rfe without a defined value."""


_STATUS = {capi.FFCZ_UNDEFINED_METRIC: UndefinedMetricError, capi.FFCZ_VALIDATION_ERROR: ValidationError, capi.FFCZ_SYMMETRY_ERROR: SymmetryError,
           capi.FFCZ_FORMAT_ERROR: FormatError, capi.FFCZ_IO_ERROR: IoError,
           capi.FFCZ_CUDA_ERROR: CudaError, capi.FFCZ_UNSUPPORTED: UnsupportedError,
           capi.FFCZ_OUT_OF_MEMORY: CudaError}


def _check(rc):
    if rc != capi.FFCZ_OK:
        raise _STATUS.get(rc, FfczError)(capi.load().ffcz_cuda_last_error().decode())


class Context:
    """One engine context (device + stream); calls on a context serialise."""

    def __init__(self, device: int = 0, stream: int | None = None):
        lib = capi.load()
        h = C.c_void_p()
        _check(lib.ffcz_cuda_create(C.byref(h), device, C.c_void_p(stream or 0)))
        self.handle = h
        self.device = device

    def close(self):
        if self.handle:
            capi.load().ffcz_cuda_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default = {}
_lock = threading.Lock()


def default_context(device: int = 0) -> Context:
    with _lock:
        if device not in _default:
            _default[device] = Context(device)
        return _default[device]


# ---------------------------------------------------------------------------------------------


@dataclass
class DualBounds:
    """ffcz::DualBounds (bounds.hpp:11-47): E global or per point; Delta global or per component
    over the FULL spectrum (Re lane, Im lane)."""

    spatial: float | np.ndarray
    freq_re: float | np.ndarray
    freq_im: float | np.ndarray | None = None
    # the field shape these arrays were validated for (DualBounds' invariants: entries > 0 and
    # finite, Hermitian-consistent lanes, bounds.cpp:10-59).  The reference checks them once,
    # when a DualBounds is built; here the engine checks them on the first call that uses the
    # arrays and later calls pass FFCZ_BOUNDS_VALIDATED.  Arrays are treated as immutable
    # afterwards, like the reference's vectors.
    _validated_for: tuple | None = field(default=None, repr=False, compare=False)

    def _arrays(self):
        return tuple(id(a) for a in (self.spatial, self.freq_re, self.freq_im)
                     if a is not None and not isinstance(a, (float, int, np.floating)))

    @staticmethod
    def global_(e: float, delta: float) -> "DualBounds":
        return DualBounds(float(e), float(delta))


@dataclass
class ProjectionReport:
    iterations: int
    active_spatial: int
    active_frequency: int
    converged: bool
    residual_f: float
    residual_s: float
    wall_time_s: float


# numpy image of ffcz_cuda_escape (include/ffcz_cuda.h)
ESCAPE_DTYPE = np.dtype([("frequency", "<i4"), ("_pad", "<i4"), ("index", "<u8"), ("re", "<f8"),
                         ("im", "<f8")])


@dataclass
class EscapeEntry:
    frequency: bool
    index: int
    re: float
    im: float


@dataclass
class CorrectionResult:
    """ffcz::CorrectionResult (pipeline.hpp:11-16) plus the device products."""

    archive_bytes: bytes | None
    report: ProjectionReport
    escape_count: int
    verify_ok: bool
    verify_max_spatial_excess: float
    verify_max_freq_excess: float
    spatial_flags: np.ndarray | None
    frequency_flags: np.ndarray | None
    spatial_codes: np.ndarray | None
    frequency_codes: np.ndarray | None
    escapes: np.ndarray | None          # structured: frequency, index, re, im (EscapeEntry order)
    corrected: np.ndarray | None
    escape_rounds: int
    timings_ms: dict
    kernel_launches: int
    iterations_fp32: int = 0     # mixed policy: clip passes run by the FP32 phase
    iterations_fp64: int = 0     # clip passes run in FP64


class _ResultHolder:
    """Owns one ffcz_cuda_result; releases its library buffers exactly once."""

    def __init__(self):
        self.res = capi.Result()
        self.live = True

    def free(self):
        if self.live:
            capi.load().ffcz_cuda_result_free(C.byref(self.res))
            self.live = False

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _is_torch(x):
    return type(x).__module__.startswith("torch")


def _order_after_torch(*tensors):
    """Device tensors handed to the engine were produced on torch's current stream; the engine
    runs on its context's own stream, so wait for torch's work on them first."""
    for t in tensors:
        if t is not None and _is_torch(t) and t.is_cuda:
            import torch
            torch.cuda.current_stream(t.device).synchronize()
            return


def _field_desc(shape, dtype_code, precision):
    d = capi.FieldDesc()
    d.ndim = len(shape)
    for i, s in enumerate(shape):
        d.dims[i] = int(s)
    d.dtype = dtype_code
    d.precision = capi.FFCZ_PRECISION_F32 if precision == "f32" else capi.FFCZ_PRECISION_F64
    return d


class _Marshal:
    """Keeps host arrays alive and produces pointers (host numpy or device torch)."""

    def __init__(self):
        self.keep = []

    def ptr(self, a, dtype=np.float64, on_dev=None, what="array"):
        """Pointer to `a` as a contiguous `dtype` buffer.  Torch tensors must already have that
        dtype (a float32 tensor is never reinterpreted as float64) and live where the call's
        inputs live (on_dev); numpy arrays are converted (a copy when needed)."""
        if a is None:
            return None
        if _is_torch(a):
            import torch
            want = torch.float64 if dtype == np.float64 else torch.float32
            if a.dtype != want:
                raise ValidationError(f"{what}: expected a {want} tensor, got {a.dtype}")
            if on_dev is not None and bool(a.is_cuda) != bool(on_dev):
                raise ValidationError(f"{what}: must be a {'CUDA' if on_dev else 'host'} array "
                                      "like the fields")
            if not a.is_cuda:
                return self.ptr(a.numpy(), dtype, on_dev, what)
            a = a.contiguous()
            self.keep.append(a)
            return C.c_void_p(a.data_ptr())
        if on_dev:
            raise ValidationError(f"{what}: must be a CUDA tensor like the fields")
        arr = np.ascontiguousarray(a, dtype=dtype)
        self.keep.append(arr)
        return C.c_void_p(arr.ctypes.data)


def _numel(a) -> int:
    return int(a.numel()) if _is_torch(a) else int(np.size(a))


def _bounds_desc(b: DualBounds, m: _Marshal, shape=None, on_dev=None):
    """ffcz_bounds_desc of `b`; with `shape`, DualBounds::validate_for (bounds.cpp:65-71): array
    bounds must cover every sample / the full spectrum (the engine reads N doubles from each)."""
    bd = capi.BoundsDesc()
    total = int(np.prod(shape)) if shape is not None else None
    sp = b.spatial
    if isinstance(sp, (float, int, np.floating)):
        bd.spatial_per_point, bd.spatial_global = 0, float(sp)
    else:
        if total is not None and _numel(sp) != total:
            raise ValidationError("per-point spatial bound length does not match field size")
        bd.spatial_per_point = 1
        bd.spatial_values = m.ptr(sp, np.float64, on_dev, "per-point spatial bound")
    re = b.freq_re
    im = b.freq_im if b.freq_im is not None else b.freq_re
    if isinstance(re, (float, int, np.floating)):
        bd.freq_per_component, bd.freq_global = 0, float(re)
    else:
        if isinstance(im, (float, int, np.floating)):
            raise ValidationError("per-component frequency bounds need both Re and Im lanes")
        if total is not None and (_numel(re) != total or _numel(im) != total):
            raise ValidationError("per-component frequency bound length does not match field size")
        bd.freq_per_component = 1
        bd.freq_re = m.ptr(re, np.float64, on_dev, "per-component frequency bound (Re)")
        bd.freq_im = bd.freq_re if im is re else m.ptr(im, np.float64, on_dev,
                                                         "per-component frequency bound (Im)")
    return bd


def _options(on_dev, want_archive, want_edits, want_corrected, fused, zlib_level,
             device_encode=False, policy="fp64", tau=1e-4, repair_order="decoder",
             f_update="rebuild"):
    lib = capi.load()
    opt = capi.Options()
    lib.ffcz_cuda_default_options(C.byref(opt))
    flags = 0
    if repair_order not in ("decoder", "reference"):
        raise ValidationError(f"unknown repair order {repair_order!r}")
    if f_update not in ("rebuild", "accumulate"):
        raise ValidationError(f"unknown F update {f_update!r}")
    if repair_order == "reference":
        flags |= capi.FFCZ_REPAIR_REFERENCE_ORDER
    if f_update == "accumulate":
        flags |= capi.FFCZ_F_ACCUMULATE
    if on_dev:
        flags |= capi.FFCZ_INPUTS_ON_DEVICE
    if want_archive:
        flags |= capi.FFCZ_WANT_ARCHIVE
    if want_edits:
        flags |= capi.FFCZ_WANT_EDITS
    if want_corrected:
        flags |= capi.FFCZ_WANT_CORRECTED
    if not fused:
        flags |= capi.FFCZ_FORCE_UNFUSED
    if device_encode:
        flags |= capi.FFCZ_DEVICE_ENCODE
    opt.flags = flags
    if policy not in ("fp64", "mixed"):
        raise ValidationError(f"unknown precision policy {policy!r}")
    opt.policy = 1 if policy == "mixed" else 0
    opt.tau_switch = float(tau)
    opt.zlib_level = zlib_level
    return opt


def _convert(holder, shape, want_archive, want_edits, want_corrected, copy):
    """ffcz_cuda_result -> CorrectionResult (views of the pinned buffers when copy=False)."""
    res = holder.res
    N = int(np.prod(shape))
    r = res.report
    rep = ProjectionReport(int(r.iterations), int(r.active_spatial), int(r.active_frequency),
                           bool(r.converged), float(r.residual_f), float(r.residual_s),
                           float(r.wall_time_s))

    def arr(p, n, dtype):
        if not p or n == 0:
            return np.zeros(0, dtype=dtype)
        a = np.ctypeslib.as_array(p, shape=(n,))
        return (a.copy() if copy else a).view(dtype)

    edits = want_edits or want_archive
    sflags = fflags = scodes = fcodes = None
    escapes = None
    if edits:
        sflags = arr(res.spatial_flags, int(res.spatial_flag_bytes), np.uint8)
        fflags = arr(res.frequency_flags, int(res.frequency_flag_bytes), np.uint8)
        scodes = arr(res.spatial_codes, int(res.n_spatial), np.int32)
        fcodes = arr(res.frequency_codes, 2 * int(res.n_frequency), np.int32)
        ne = int(res.escape_count)
        if ne and res.escapes:
            raw = np.ctypeslib.as_array(C.cast(res.escapes, C.POINTER(C.c_uint8)),
                                        shape=(ne * C.sizeof(capi.Escape),))
            escapes = raw.view(ESCAPE_DTYPE)
            if copy:
                escapes = escapes.copy()
        else:
            escapes = np.zeros(0, dtype=ESCAPE_DTYPE)
    corrected = None
    if want_corrected:
        corrected = np.ctypeslib.as_array(res.corrected, shape=(N,)).reshape(shape)
        if copy:
            corrected = corrected.copy()
    data = None
    if want_archive:   # (C.string_at takes an int size: archives can exceed 2 GiB)
        if not res.archive_len:
            data = b""
        else:
            view = np.ctypeslib.as_array(res.archive, shape=(int(res.archive_len),))
            data = view.tobytes() if copy else view  # copy=False: a uint8 view of the pinned bytes
    timings = {k: float(getattr(res, k)) for k in ("t_feasible_ms", "t_loop_ms", "t_gate_ms",
                                                   "t_h2d_ms", "t_d2h_ms", "t_archive_ms")}
    out = CorrectionResult(data, rep, int(res.escape_count), bool(res.verify_ok),
                           float(res.verify_max_spatial_excess),
                           float(res.verify_max_freq_excess), sflags, fflags, scodes, fcodes,
                           escapes, corrected, int(res.escape_rounds), timings,
                           int(res.kernel_launches), int(res.iterations_fp32),
                           int(res.iterations_fp64))
    if copy:
        holder.free()
    else:
        out._holder = holder  # keeps the pinned buffers alive with the views
    return out


def _field_of(original, decompressed):
    """(on_dev, is32, shape, original, decompressed) of numpy / CUDA torch inputs, with the
    reference's compute_error check (projection.cpp:20-22): same dims and sample type."""
    if _is_torch(original) != _is_torch(decompressed):
        raise ValidationError("compute_error: original and decompressed must both be host arrays "
                              "or both CUDA tensors")
    on_dev = _is_torch(original)
    if on_dev:
        import torch
        if not (original.is_cuda and decompressed.is_cuda):
            original, decompressed = original.cpu().numpy(), decompressed.cpu().numpy()
            return _field_of(original, decompressed)
        if original.dtype not in (torch.float32, torch.float64):
            raise ValidationError(f"fields must be float32 or float64, got {original.dtype}")
        if tuple(original.shape) != tuple(decompressed.shape) or \
                original.dtype != decompressed.dtype:
            raise ValidationError("compute_error: dims/precision mismatch")
        is32 = original.dtype == torch.float32
        shape = tuple(original.shape)
        original, decompressed = original.contiguous(), decompressed.contiguous()
    else:
        original = np.asarray(original)
        decompressed = np.asarray(decompressed)
        if original.shape != decompressed.shape or original.dtype != decompressed.dtype:
            raise ValidationError("compute_error: dims/precision mismatch")
        is32 = original.dtype == np.float32
        shape = original.shape
    if not 1 <= len(shape) <= 3 or any(int(n) == 0 for n in shape):
        raise ValidationError("field must have 1 to 3 non-empty axes")
    return on_dev, is32, shape, original, decompressed


def correct(original, decompressed, bounds: DualBounds, m: int = 16, max_iters: int = 1000,
            precision: str | None = None, *, want_archive: bool = True, want_edits: bool = True,
            want_corrected: bool = True, zlib_level: int = OUTER_DEVICE, fused: bool = True,
            copy: bool = True, device_encode: bool = False, policy: str = "fp64",
            tau: float = 1e-4, repair_order: str = "decoder", f_update: str = "rebuild",
            ctx: Context | None = None) -> CorrectionResult:
    """ffcz::correct (pipeline.cpp:26-178) on the GPU.

    original / decompressed: numpy arrays (host; float32 or float64) or CUDA torch tensors (then
    every bound array must be a CUDA tensor too).  precision: the ScalarField precision tag
    written into the archive ("f32" / "f64"; default from the input dtype).  copy=False returns
    views of the library's pinned result buffers, valid while the returned object is alive.
    zlib_level: OUTER_DEVICE (default) assembles the archive from streams encoded on the GPU
    (Huffman payloads identical to huffman.cpp, deflate blocks written on the device, readable by
    the reference's read_archive); 0..9 runs the outer zlib stage on the host at that level (9 =
    the reference's own bytes).  device_encode: with a host zlib level, the Huffman stage on the
    GPU (same payload bytes).
    policy: "fp64" (reference control flow in FP64, default) or "mixed" (FP32 passes while
    max_excess / peak > tau, then FP64; iterations within +-1 of the reference).
    repair_order: "decoder" (default: repair the decoder's own view) or
    "reference" (check eps_tilde each round + a separate verify, pipeline.cpp:134-160 — the
    reference's escape lists).  f_update: "rebuild" (default: F rebuilt once at the gate) or
    "accumulate" (F += displacement in every clip, projection.cpp:117-119).
    """
    lib = capi.load()
    on_dev, is32, shape, original, decompressed = _field_of(original, decompressed)
    if precision is None:
        precision = "f32" if is32 else "f64"
    dt = np.float32 if is32 else np.float64
    mar = _Marshal()
    fd = _field_desc(shape, capi.FFCZ_F32 if is32 else capi.FFCZ_F64, precision)
    bd = _bounds_desc(bounds, mar, shape, on_dev)
    opt = _options(on_dev, want_archive, want_edits, want_corrected, fused, zlib_level,
                   device_encode, policy, tau, repair_order, f_update)
    ctx = ctx or default_context()   # after the argument checks (they need no device)
    key = (tuple(shape), bool(on_dev), bounds._arrays())
    if bounds._validated_for == key:
        opt.flags |= capi.FFCZ_BOUNDS_VALIDATED
    if on_dev:
        _order_after_torch(original, decompressed, bounds.spatial, bounds.freq_re, bounds.freq_im)
    holder = _ResultHolder()
    rc = lib.ffcz_cuda_correct(ctx.handle, C.byref(fd), mar.ptr(original, dt),
                               mar.ptr(decompressed, dt), C.byref(bd), int(m), int(max_iters),
                               C.byref(opt), C.byref(holder.res))
    try:
        _check(rc)
    except Exception:
        holder.free()
        raise
    bounds._validated_for = key
    return _convert(holder, shape, want_archive, want_edits, want_corrected, copy)


def correct_batch(original, decompressed, bounds, m: int = 16, max_iters: int = 1000,
                  precision: str | None = None, *, lanes: int = 8, want_archive: bool = True,
                  want_edits: bool = True, want_corrected: bool = True,
                  zlib_level: int = OUTER_DEVICE,
                  fused: bool = True, copy: bool = True, policy: str = "fp64", tau: float = 1e-4,
                  repair_order: str = "decoder", f_update: str = "rebuild",
                  ctx: Context | None = None) -> list[CorrectionResult]:
    """Independent ffcz::correct() of every frame of a batch (BASELINE config 3).

    original / decompressed: arrays of shape (frames, *frame_shape), numpy or CUDA torch.
    bounds: one DualBounds per frame (a single DualBounds is used for every frame).  Returns one
    CorrectionResult per frame, identical to correct() on that frame alone.
    """
    ctx = ctx or default_context()
    lib = capi.load()
    on_dev, is32, shape, original, decompressed = _field_of(original, decompressed)
    nf, frame = int(shape[0]), tuple(shape[1:])
    if precision is None:
        precision = "f32" if is32 else "f64"
    dt = np.float32 if is32 else np.float64
    if isinstance(bounds, DualBounds):
        bounds = [bounds] * nf
    if len(bounds) != nf:
        raise ValidationError(f"correct_batch: {len(bounds)} bounds for {nf} frames")
    mar = _Marshal()
    fd = _field_desc(frame, capi.FFCZ_F32 if is32 else capi.FFCZ_F64, precision)
    bds = (capi.BoundsDesc * max(1, nf))()
    for i, b in enumerate(bounds):
        bds[i] = _bounds_desc(b, mar, frame, on_dev)
    opt = _options(on_dev, want_archive, want_edits, want_corrected, fused, zlib_level,
                   False, policy, tau, repair_order, f_update)
    if on_dev:
        _order_after_torch(original, decompressed)
    res = (capi.Result * max(1, nf))()
    rc = lib.ffcz_cuda_correct_batch(ctx.handle, C.byref(fd), nf, mar.ptr(original, dt),
                                     mar.ptr(decompressed, dt), bds, int(m), int(max_iters),
                                     C.byref(opt), int(lanes), res)
    _check(rc)
    outs = []
    for i in range(nf):
        h = _ResultHolder()
        C.memmove(C.byref(h.res), C.byref(res[i]), C.sizeof(capi.Result))
        outs.append(_convert(h, frame, want_archive, want_edits, want_corrected, copy))
    return outs


def alternating_projection(eps0, bounds_working: DualBounds, max_iters: int,
                           precondition_slack: float = 2.0 ** -20, *, fused: bool = True,
                           ctx: Context | None = None):
    """ffcz::alternating_projection (projection.cpp:81-142) on the GPU.

    Returns (spatial_edits, frequency_edits FULL spectrum complex, final_epsilon, report)."""
    ctx = ctx or default_context()
    lib = capi.load()
    eps0 = np.ascontiguousarray(eps0, dtype=np.float64)
    shape = eps0.shape
    mar = _Marshal()
    fd = _field_desc(shape, capi.FFCZ_F64, "f64")
    bd = _bounds_desc(bounds_working, mar, shape, False)
    opt = capi.Options()
    lib.ffcz_cuda_default_options(C.byref(opt))
    opt.flags = 0 if fused else capi.FFCZ_FORCE_UNFUSED
    S = np.zeros(shape)
    F = np.zeros(shape, dtype=np.complex128)
    eps = np.zeros(shape)
    rep = capi.Report()
    _check(lib.ffcz_cuda_alternating_projection(
        ctx.handle, C.byref(fd), C.c_void_p(eps0.ctypes.data), C.byref(bd), int(max_iters),
        float(precondition_slack), C.byref(opt), C.c_void_p(S.ctypes.data),
        C.c_void_p(F.ctypes.data), C.c_void_p(eps.ctypes.data), C.byref(rep)))
    report = ProjectionReport(int(rep.iterations), int(rep.active_spatial),
                              int(rep.active_frequency), bool(rep.converged),
                              float(rep.residual_f), float(rep.residual_s), float(rep.wall_time_s))
    return S, F, eps, report


def forward_dft(x, *, ctx: Context | None = None) -> np.ndarray:
    """ffcz::forward_dft (transform.cpp:45-50): unnormalised FP64 DFT, FULL spectrum."""
    ctx = ctx or default_context()
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(x.shape, dtype=np.complex128)
    fd = _field_desc(x.shape, capi.FFCZ_F64, "f64")
    _check(capi.load().ffcz_cuda_forward_dft(ctx.handle, C.byref(fd), C.c_void_p(x.ctypes.data),
                                             C.c_void_p(out.ctypes.data)))
    return out


def _metric_input(x):
    """(pointer holder, shape, dtype code, on_device) for a numpy array or a CUDA tensor."""
    if _is_torch(x):
        import torch
        if not x.is_cuda:
            x = x.numpy()
        else:
            x = x.contiguous()
            if x.dtype not in (torch.float32, torch.float64):
                x = x.to(torch.float64)
            return x, tuple(x.shape), capi.FFCZ_F32 if x.dtype == torch.float32 else capi.FFCZ_F64, 1
    a = np.asarray(x)
    a = np.ascontiguousarray(a, dtype=np.float32 if a.dtype == np.float32 else np.float64)
    return a, a.shape, capi.FFCZ_F32 if a.dtype == np.float32 else capi.FFCZ_F64, 0


def _vp(a):
    return C.c_void_p(a.data_ptr() if _is_torch(a) else a.ctypes.data)


def spectrum_bound_to_freq_bounds(original, rho: float, *, ctx: Context | None = None):
    """ffcz::spectrum_bound_to_freq_bounds(forward_dft(original), rho) (metrics.cpp:107-128) on
    the device: the FULL-spectrum per-component Delta (Re lane == Im lane), shaped like the field.
    A CUDA tensor in gives a CUDA float64 tensor out."""
    ctx = ctx or default_context()
    x, shape, dt, dev = _metric_input(original)
    if dev:
        import torch
        _order_after_torch(x)
        out = torch.empty(shape, dtype=torch.float64, device=x.device)
    else:
        out = np.empty(shape, dtype=np.float64)
    fd = _field_desc(shape, dt, "f64")
    _check(capi.load().ffcz_cuda_spectrum_bound(ctx.handle, C.byref(fd), _vp(x), dev, float(rho),
                                                _vp(out)))
    return out


@dataclass
class Metrics:
    """The values `ffcz metrics` prints (proj/tools/ffcz.cpp:246-278)."""
    psnr_db: float
    ssnr_db: float
    max_rfe: float
    max_spatial: float


def metrics(original, reconstructed, *, ctx: Context | None = None) -> Metrics:
    """psnr, ssnr of the spectra, max relative frequency error and max |eps| (metrics.cpp),
    computed on the device.  Raises UndefinedMetricError where the reference throws."""
    ctx = ctx or default_context()
    x, shape, dt, dev = _metric_input(original)
    y, shape2, dt2, dev2 = _metric_input(reconstructed)
    if shape != shape2:
        raise ValidationError("metrics: dims mismatch")
    if dt != dt2 or dev != dev2:
        raise ValidationError("metrics: both fields must have the same dtype and location")
    _order_after_torch(x, y)
    fd = _field_desc(shape, dt, "f64")
    m = capi.MetricsOut()
    _check(capi.load().ffcz_cuda_metrics(ctx.handle, C.byref(fd), _vp(x), _vp(y), dev,
                                         C.byref(m)))
    return Metrics(m.psnr_db, m.ssnr_db, m.max_rfe, m.max_spatial)


@dataclass
class PowerSpectrum:
    """ffcz::PowerSpectrum (metrics.hpp:12-18)."""
    k_bins: np.ndarray
    power: np.ndarray
    counts: np.ndarray
    mean_fallback: bool
    mean: float


def power_spectrum(field, *, ctx: Context | None = None) -> PowerSpectrum:
    """ffcz::power_spectrum (metrics.cpp:11-62) on the device."""
    ctx = ctx or default_context()
    x, shape, dt, dev = _metric_input(field)
    _order_after_torch(x)
    fd = _field_desc(shape, dt, "f64")
    lib = capi.load()
    nb = C.c_uint64()
    _check(lib.ffcz_cuda_power_spectrum(ctx.handle, C.byref(fd), _vp(x), dev, 0, None, None,
                                        C.byref(nb), None, None))
    power = np.zeros(nb.value, dtype=np.float64)
    counts = np.zeros(nb.value, dtype=np.uint64)
    mean = C.c_double()
    fb = C.c_int()
    _check(lib.ffcz_cuda_power_spectrum(ctx.handle, C.byref(fd), _vp(x), dev, nb.value,
                                        C.c_void_p(power.ctypes.data),
                                        C.c_void_p(counts.ctypes.data), C.byref(nb),
                                        C.byref(mean), C.byref(fb)))
    return PowerSpectrum(np.arange(nb.value, dtype=np.uint64), power, counts, bool(fb.value),
                         float(mean.value))


def inverse_dft(X, precision: str = "f64", *, ctx: Context | None = None) -> np.ndarray:
    """ffcz::inverse_dft (transform.cpp:64-80): 1/N inverse with the imaginary-residue gate."""
    ctx = ctx or default_context()
    X = np.ascontiguousarray(X, dtype=np.complex128)
    out = np.zeros(X.shape)
    fd = _field_desc(X.shape, capi.FFCZ_F64, "f64")
    _check(capi.load().ffcz_cuda_inverse_dft(
        ctx.handle, C.byref(fd), C.c_void_p(X.ctypes.data),
        capi.FFCZ_PRECISION_F32 if precision == "f32" else capi.FFCZ_PRECISION_F64,
        C.c_void_p(out.ctypes.data)))
    return out


def r2c_device(x, out, *, ctx: Context | None = None):
    """Half-spectrum R2C on CUDA torch tensors (float32/float64): out[..., :n/2+1] complex."""
    import torch
    ctx = ctx or default_context()
    fd = _field_desc(tuple(x.shape), capi.FFCZ_F32 if x.dtype == torch.float32 else capi.FFCZ_F64,
                     "f64")
    _order_after_torch(x, out)
    _check(capi.load().ffcz_cuda_r2c_device(ctx.handle, C.byref(fd), C.c_void_p(x.data_ptr()),
                                            C.c_void_p(out.data_ptr())))


def c2r_device(half, x, *, ctx: Context | None = None):
    """1/N-normalised C2R on CUDA torch tensors."""
    import torch
    ctx = ctx or default_context()
    fd = _field_desc(tuple(x.shape), capi.FFCZ_F32 if x.dtype == torch.float32 else capi.FFCZ_F64,
                     "f64")
    _order_after_torch(half, x)
    _check(capi.load().ffcz_cuda_c2r_device(ctx.handle, C.byref(fd), C.c_void_p(half.data_ptr()),
                                            C.c_void_p(x.data_ptr())))


def huffman_encode_device(codes, *, ctx: Context | None = None) -> bytes:
    """The device Huffman encoder on int32 codes (test hook): huffman::encode's payload of
    zigzag(codes) (huffman.cpp:156-251, streams.cpp:13-15)."""
    ctx = ctx or default_context()
    lib = capi.load()
    c = np.ascontiguousarray(codes, dtype=np.int32)
    n = C.c_uint64()
    _check(lib.ffcz_cuda_huffman_encode(ctx.handle, C.c_void_p(c.ctypes.data), c.size, None, 0,
                                        C.byref(n)))
    out = np.zeros(max(1, n.value), dtype=np.uint8)
    _check(lib.ffcz_cuda_huffman_encode(ctx.handle, C.c_void_p(c.ctypes.data), c.size,
                                        C.c_void_p(out.ctypes.data), n.value, C.byref(n)))
    return out[: n.value].tobytes()


def outer_compress_device(data, *, ctx: Context | None = None) -> bytes:
    """The device outer stage (deflate.cu) on host bytes: outer_compress's framing
    (streams.cpp:21-32: u64 raw size + zlib stream), decodable by zlib / outer_decompress."""
    ctx = ctx or default_context()
    lib = capi.load()
    b = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else \
        np.ascontiguousarray(data, dtype=np.uint8).reshape(-1)
    n = C.c_uint64()
    ptr = C.c_void_p(b.ctypes.data) if b.size else None
    _check(lib.ffcz_cuda_outer_compress(ctx.handle, ptr, b.size, None, 0, C.byref(n)))
    out = np.zeros(max(1, n.value), dtype=np.uint8)
    _check(lib.ffcz_cuda_outer_compress(ctx.handle, ptr, b.size, C.c_void_p(out.ctypes.data),
                                        n.value, C.byref(n)))
    return out[: n.value].tobytes()


def crc32c_device(data, *, ctx: Context | None = None) -> int:
    """CRC-32C (archive.cpp:61-71) computed on the device; data: bytes / numpy (host) or a CUDA
    torch tensor (device)."""
    ctx = ctx or default_context()
    lib = capi.load()
    out = C.c_uint32()
    if _is_torch(data):
        _check(lib.ffcz_cuda_crc32c_device(ctx.handle, C.c_void_p(data.data_ptr()),
                                           data.numel() * data.element_size(), 1, C.byref(out)))
        return out.value
    b = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else \
        np.ascontiguousarray(data).view(np.uint8).reshape(-1)
    ptr = C.c_void_p(b.ctypes.data) if b.size else None
    _check(lib.ffcz_cuda_crc32c_device(ctx.handle, ptr, b.size, 0, C.byref(out)))
    return out.value


def apply_archive(archive: bytes, decompressed, *, ctx: Context | None = None):
    """ffcz::apply_edits(decompressed, ffcz::read_archive(archive)) (archive.cpp:137-273) on the
    GPU: the FP64 corrected field (numpy for host input, CUDA torch tensor for device input)."""
    ctx = ctx or default_context()
    lib = capi.load()
    on_dev = _is_torch(decompressed)
    if on_dev:
        import torch
        is32 = decompressed.dtype == torch.float32
        shape = tuple(decompressed.shape)
        out = torch.empty(shape, dtype=torch.float64, device=decompressed.device)
        _order_after_torch(decompressed)
        dptr, optr = C.c_void_p(decompressed.data_ptr()), C.c_void_p(out.data_ptr())
        keep = (decompressed,)
    else:
        d = np.asarray(decompressed)
        is32 = d.dtype == np.float32
        d = np.ascontiguousarray(d, dtype=np.float32 if is32 else np.float64)
        shape = d.shape
        out = np.empty(shape, dtype=np.float64)
        dptr, optr = C.c_void_p(d.ctypes.data), C.c_void_p(out.ctypes.data)
        keep = (d,)
    fd = _field_desc(shape, capi.FFCZ_F32 if is32 else capi.FFCZ_F64, "f64")
    buf = np.frombuffer(archive, dtype=np.uint8)
    _check(lib.ffcz_cuda_apply_archive(ctx.handle, C.c_void_p(buf.ctypes.data), buf.size,
                                       C.byref(fd), dptr,
                                       capi.FFCZ_INPUTS_ON_DEVICE if on_dev else 0, optr))
    del keep
    return out
