"""The C-ABI shared library loads and exports exactly what include/ffcz_cuda.h declares.  CPU."""
import ctypes
import os
import re

import pytest

from paper_2601_01596_b200 import _capi as capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "ffcz_cuda.h")).read()
    return sorted(set(re.findall(r"\b(ffcz_cuda_\w+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    lib = capi.load()
    syms = declared_symbols()
    assert set(syms) == set(capi.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s


def test_library_is_sm100a():
    data = open(capi.LIB_PATH, "rb").read()
    assert b"sm_100a" in data


def test_abi_version_and_crc_without_gpu():
    lib = capi.load()
    assert lib.ffcz_cuda_abi_version() == 1
    s = b"123456789"
    assert lib.ffcz_cuda_crc32c(s, len(s)) == 0xE3069283


def test_struct_layouts_match_header():
    # sizes of the C structs as laid out by the C compiler (x86-64 SysV)
    assert ctypes.sizeof(capi.FieldDesc) == 40
    assert ctypes.sizeof(capi.BoundsDesc) == 56
    assert ctypes.sizeof(capi.Options) == 24
    assert ctypes.sizeof(capi.Escape) == 32


def test_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = capi.load()
    h = ctypes.c_void_p()
    assert lib.ffcz_cuda_create(ctypes.byref(h), 0, None) != 0


def test_metrics_struct_layout():
    assert ctypes.sizeof(capi.MetricsOut) == 32


def test_missing_library_fails_loudly(tmp_path):
    # no CPU fallback: without the shared object the package refuses to run
    import subprocess
    import sys
    env = dict(os.environ, FFCZ_CUDA_LIB=str(tmp_path / "absent.so"))
    code = "from paper_2601_01596_b200 import _capi; _capi.load()"
    p = subprocess.run([sys.executable, "-c", code], env=env, cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert p.returncode != 0
    assert "absent.so" in p.stderr
