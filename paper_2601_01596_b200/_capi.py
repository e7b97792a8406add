"""ctypes mirror of include/ffcz_cuda.h (the C-ABI of libffcz_cuda.so).

The library is built in-tree (paper_2601_01596_b200/libffcz_cuda.so) by __graft_entry__.build()
or `make -C paper_2601_01596_b200/csrc`.  There is no fallback: if the shared object is missing,
loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FFCZ_CUDA_LIB") or os.path.join(HERE, "libffcz_cuda.so")

FFCZ_OK = 0
FFCZ_VALIDATION_ERROR = 1
FFCZ_SYMMETRY_ERROR = 2
FFCZ_FORMAT_ERROR = 3
FFCZ_IO_ERROR = 4
FFCZ_CUDA_ERROR = 5
FFCZ_UNSUPPORTED = 6
FFCZ_OUT_OF_MEMORY = 7
FFCZ_UNDEFINED_METRIC = 8

FFCZ_F32, FFCZ_F64 = 0, 1
FFCZ_PRECISION_F32, FFCZ_PRECISION_F64 = 0, 1
FFCZ_POLICY_FP64, FFCZ_POLICY_MIXED = 0, 1

FFCZ_INPUTS_ON_DEVICE = 1 << 0
FFCZ_WANT_ARCHIVE = 1 << 1
FFCZ_WANT_EDITS = 1 << 2
FFCZ_WANT_CORRECTED = 1 << 3
FFCZ_DEVICE_ENCODE = 1 << 5
FFCZ_FORCE_UNFUSED = 1 << 4
FFCZ_BOUNDS_VALIDATED = 1 << 6
FFCZ_REPAIR_REFERENCE_ORDER = 1 << 7
FFCZ_F_ACCUMULATE = 1 << 8

# every symbol include/ffcz_cuda.h declares
EXPORTS = [
    "ffcz_cuda_create", "ffcz_cuda_destroy", "ffcz_cuda_last_error", "ffcz_cuda_abi_version",
    "ffcz_cuda_default_options", "ffcz_cuda_correct", "ffcz_cuda_correct_batch",
    "ffcz_cuda_result_free",
    "ffcz_cuda_alternating_projection", "ffcz_cuda_forward_dft", "ffcz_cuda_inverse_dft",
    "ffcz_cuda_r2c_device", "ffcz_cuda_c2r_device", "ffcz_cuda_crc32c",
    "ffcz_cuda_profile_enable", "ffcz_cuda_profile_read", "ffcz_cuda_bench_passes",
    "ffcz_cuda_slab", "ffcz_cuda_slab_pitch", "ffcz_cuda_huffman_encode",
    "ffcz_cuda_apply_archive", "ffcz_cuda_spectrum_bound", "ffcz_cuda_metrics",
    "ffcz_cuda_power_spectrum", "ffcz_cuda_outer_compress", "ffcz_cuda_crc32c_device",
    "ffcz_cuda_ipc_handle", "ffcz_cuda_ipc_open", "ffcz_cuda_ipc_close",
    "ffcz_cuda_launch_count",
]


class FieldDesc(C.Structure):
    _fields_ = [("ndim", C.c_int32), ("dims", C.c_uint64 * 3), ("dtype", C.c_int32),
                ("precision", C.c_int32)]


class MetricsOut(C.Structure):
    _fields_ = [("psnr_db", C.c_double), ("ssnr_db", C.c_double), ("max_rfe", C.c_double),
                ("max_spatial", C.c_double)]


class BoundsDesc(C.Structure):
    _fields_ = [("spatial_per_point", C.c_int32), ("spatial_global", C.c_double),
                ("spatial_values", C.c_void_p), ("freq_per_component", C.c_int32),
                ("freq_global", C.c_double), ("freq_re", C.c_void_p), ("freq_im", C.c_void_p)]


class Options(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("policy", C.c_int32), ("tau_switch", C.c_double),
                ("zlib_level", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_uint64), ("active_spatial", C.c_uint64),
                ("active_frequency", C.c_uint64), ("converged", C.c_int32),
                ("residual_f", C.c_double), ("residual_s", C.c_double),
                ("wall_time_s", C.c_double)]


class Escape(C.Structure):
    _fields_ = [("frequency", C.c_int32), ("index", C.c_uint64), ("re", C.c_double),
                ("im", C.c_double)]


class Result(C.Structure):
    _fields_ = [
        ("report", Report), ("iterations_fp32", C.c_uint64), ("iterations_fp64", C.c_uint64),
        ("escape_rounds", C.c_uint64), ("escape_count", C.c_uint64), ("verify_ok", C.c_int32),
        ("verify_max_spatial_excess", C.c_double), ("verify_max_freq_excess", C.c_double),
        ("n_spatial", C.c_uint64), ("n_frequency", C.c_uint64),
        ("spatial_flags", C.POINTER(C.c_uint8)), ("spatial_flag_bytes", C.c_uint64),
        ("frequency_flags", C.POINTER(C.c_uint8)), ("frequency_flag_bytes", C.c_uint64),
        ("spatial_codes", C.POINTER(C.c_int32)), ("frequency_codes", C.POINTER(C.c_int32)),
        ("escapes", C.POINTER(Escape)), ("corrected", C.POINTER(C.c_double)),
        ("archive", C.POINTER(C.c_uint8)), ("archive_len", C.c_uint64),
        ("t_feasible_ms", C.c_double), ("t_loop_ms", C.c_double), ("t_gate_ms", C.c_double),
        ("t_h2d_ms", C.c_double), ("t_d2h_ms", C.c_double), ("t_archive_ms", C.c_double),
        ("kernel_launches", C.c_uint64),
    ]


class KernelStat(C.Structure):
    _fields_ = [("name", C.c_char * 40), ("launches", C.c_uint64), ("gated", C.c_uint64),
                ("total_ms", C.c_double), ("bytes", C.c_double)]


_lib = None


def load():
    """Load the in-tree shared object (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() or "
                          "`make -C paper_2601_01596_b200/csrc`")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    lib.ffcz_cuda_create.argtypes = [C.POINTER(P), C.c_int, P]
    lib.ffcz_cuda_destroy.argtypes = [P]
    lib.ffcz_cuda_destroy.restype = None
    lib.ffcz_cuda_last_error.restype = C.c_char_p
    lib.ffcz_cuda_default_options.argtypes = [C.POINTER(Options)]
    lib.ffcz_cuda_default_options.restype = None
    lib.ffcz_cuda_correct.argtypes = [P, C.POINTER(FieldDesc), P, P, C.POINTER(BoundsDesc),
                                      C.c_int, C.c_uint64, C.POINTER(Options), C.POINTER(Result)]
    lib.ffcz_cuda_correct_batch.argtypes = [P, C.POINTER(FieldDesc), C.c_uint64, P, P,
                                            C.POINTER(BoundsDesc), C.c_int, C.c_uint64,
                                            C.POINTER(Options), C.c_int, C.POINTER(Result)]
    lib.ffcz_cuda_slab.argtypes = [P, P, C.POINTER(C.c_double)]
    lib.ffcz_cuda_apply_archive.argtypes = [P, P, C.c_uint64, C.POINTER(FieldDesc), P, C.c_uint32,
                                            P]
    lib.ffcz_cuda_huffman_encode.argtypes = [P, P, C.c_uint64, P, C.c_uint64,
                                             C.POINTER(C.c_uint64)]
    lib.ffcz_cuda_outer_compress.argtypes = [P, P, C.c_uint64, P, C.c_uint64,
                                             C.POINTER(C.c_uint64)]
    lib.ffcz_cuda_crc32c_device.argtypes = [P, P, C.c_uint64, C.c_int, C.POINTER(C.c_uint32)]
    lib.ffcz_cuda_slab_pitch.argtypes = [C.c_uint64]
    lib.ffcz_cuda_ipc_handle.argtypes = [P, P, P, C.POINTER(C.c_uint64)]
    lib.ffcz_cuda_ipc_open.argtypes = [P, P, C.POINTER(C.c_void_p)]
    lib.ffcz_cuda_ipc_close.argtypes = [P, P]
    lib.ffcz_cuda_launch_count.argtypes = [P]
    lib.ffcz_cuda_launch_count.restype = C.c_uint64
    lib.ffcz_cuda_slab_pitch.restype = C.c_uint64
    lib.ffcz_cuda_result_free.argtypes = [C.POINTER(Result)]
    lib.ffcz_cuda_result_free.restype = None
    lib.ffcz_cuda_alternating_projection.argtypes = [
        P, C.POINTER(FieldDesc), P, C.POINTER(BoundsDesc), C.c_uint64, C.c_double,
        C.POINTER(Options), P, P, P, C.POINTER(Report)]
    lib.ffcz_cuda_forward_dft.argtypes = [P, C.POINTER(FieldDesc), P, P]
    lib.ffcz_cuda_spectrum_bound.argtypes = [P, C.POINTER(FieldDesc), P, C.c_int, C.c_double, P]
    lib.ffcz_cuda_metrics.argtypes = [P, C.POINTER(FieldDesc), P, P, C.c_int,
                                      C.POINTER(MetricsOut)]
    lib.ffcz_cuda_power_spectrum.argtypes = [P, C.POINTER(FieldDesc), P, C.c_int, C.c_uint64, P, P,
                                             C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                             C.POINTER(C.c_int)]
    lib.ffcz_cuda_inverse_dft.argtypes = [P, C.POINTER(FieldDesc), P, C.c_int, P]
    lib.ffcz_cuda_r2c_device.argtypes = [P, C.POINTER(FieldDesc), P, P]
    lib.ffcz_cuda_c2r_device.argtypes = [P, C.POINTER(FieldDesc), P, P]
    lib.ffcz_cuda_crc32c.argtypes = [P, C.c_size_t]
    lib.ffcz_cuda_crc32c.restype = C.c_uint32
    lib.ffcz_cuda_profile_enable.argtypes = [P, C.c_int]
    lib.ffcz_cuda_profile_read.argtypes = [P, C.POINTER(KernelStat), C.c_int, C.POINTER(C.c_int)]
    lib.ffcz_cuda_bench_passes.argtypes = [P, C.POINTER(FieldDesc), C.c_int,
                                           C.POINTER(KernelStat), C.c_int, C.POINTER(C.c_int)]
    _lib = lib
    return lib
