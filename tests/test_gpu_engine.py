"""FFT engine at production sizes (FP32 and FP64 R2C/C2R on device) against torch.fft in FP64
(test checker only).  Tolerances: FP64 1e-12 relative to the spectrum peak, FP32 2e-6."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [(512, 512, 512), (256, 256, 256), (2048, 2048), (64, 64, 64), (1024, 4096), (8192,) * 1,
          (4, 2048, 8), (128, 1024, 32)]


@pytest.fixture(scope="module")
def torch():
    import torch as t
    if not t.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return t


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("shape", SHAPES, ids=[str(s) for s in SHAPES])
def test_r2c_c2r_device(torch, shape, dtype):
    import paper_2601_01596_b200.ffcz as F
    dt = getattr(torch, dtype)
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand(shape, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
    xs = x.to(dt).contiguous()
    half_shape = shape[:-1] + (shape[-1] // 2 + 1,)
    cdt = torch.complex64 if dt == torch.float32 else torch.complex128
    out = torch.empty(half_shape, device="cuda", dtype=cdt)
    F.r2c_device(xs, out)
    ref = torch.fft.rfftn(xs.to(torch.float64))
    err = (out.to(torch.complex128) - ref).abs().max().item() / ref.abs().max().item()
    tol = 2e-6 if dt == torch.float32 else 1e-12
    assert err < tol, err
    back = torch.empty_like(xs)
    F.c2r_device(out, back)
    err2 = (back.to(torch.float64) - xs.to(torch.float64)).abs().max().item()
    assert err2 < (5e-6 if dt == torch.float32 else 1e-12), err2
