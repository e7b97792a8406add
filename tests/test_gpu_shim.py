"""Drop-in parity through the C++ shim: oracle/_ref/shim_parity links the unmodified reference
core and include/ffcz_cuda.hpp (over libffcz_cuda.so) and checks, with the reference's OWN types,
reader and verifier, that ffcz::cuda::correct reproduces ffcz::correct."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_parity")


def test_cpp_shim_drop_in():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/shim_parity not built (built where /root/reference exists)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    bad = [x for x in lines if x.get("ok") is False]
    assert out.returncode == 0 and not bad, (out.returncode, bad, out.stderr[-2000:])
    cases = [x for x in lines if x.get("case", "").startswith("accept_like")]
    assert len(cases) == 24
    # decoded by the REFERENCE reader, the GPU archives satisfy both bounds exactly
    assert all(x["ref_decoder_verify_ok"] for x in cases)
