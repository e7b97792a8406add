"""Mixed FP32 -> FP64 policy (BASELINE north star: FP32 with
iteration counts within +-1 and both bounds exact).  Against the reference's golden outputs:
converged flag equal, iterations within +-1, both bounds hold exactly on the FP64 corrected field
(the gate is FP64: spatial excess 0.0, every frequency component within 1e-15 of its Delta
under numpy's FFT), flag counts within 1 % of the reference's digest on every case, and flags
and codes agreeing on >= 99 % of entries where the reference's archive is stored."""
import json
import os

import numpy as np
import pytest

import cases
from oracle import ffcz_oracle as O

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(cases.GOLDEN, "golden.json")))
ARCH = dict(np.load(os.path.join(cases.GOLDEN, "archives.npz")))
NAMES = ["config1_c2.0", "config1_c1.0", "config1_c0.6", "config1_c0.4", "config4_comb32",
         "config3_frame256", "config2_rho32", "m8_32cube"]
CASES = [c for c in cases.all_cases() if c.name in NAMES]


@pytest.fixture(scope="module")
def ffcz():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2601_01596_b200 as P
    return P


@pytest.mark.parametrize("case", CASES, ids=[c.name for c in CASES])
def test_mixed_policy(ffcz, case):
    g = GOLD[case.name]
    b = ffcz.DualBounds(case.E, case.Dre, case.Dim)
    r = ffcz.correct(case.original, case.decompressed, b, case.m, case.max_iters, case.precision,
                     policy="mixed")
    assert r.report.converged == g["converged"]
    assert abs(r.report.iterations - g["iterations"]) <= 1, (r.report.iterations, g["iterations"])
    assert r.verify_ok
    ok, ms, mf = O.verify_bounds(case.original, r.corrected, O.DualBounds(case.E, case.Dre, case.Dim))
    assert ms == 0.0
    assert cases.freq_excess_per_component(case.original, r.corrected, case.Dre, case.Dim) <= 1e-15
    # flags: every case against the reference's digest (flag counts within 1 %, and the full
    # flag / code comparison where the reference's archive is stored)
    dg = cases.digest_of_result(r)
    for k in ("popcount_s", "popcount_f"):
        assert abs(dg[k] - g["digest"][k]) <= max(1, g["digest"][k] // 100), (k, dg[k], g["digest"][k])
    mine = O.read_archive(r.archive_bytes)
    if case.name in ARCH:
        ref = O.read_archive(ARCH[case.name].tobytes())
        assert np.mean(mine.spatial_flags == ref.spatial_flags) >= 0.99
        assert np.mean(mine.frequency_flags == ref.frequency_flags) >= 0.99
        if np.array_equal(mine.frequency_flags, ref.frequency_flags) and ref.frequency_codes.size:
            assert np.mean(mine.frequency_codes == ref.frequency_codes) >= 0.99


def test_mixed_uses_fp32_phase(ffcz):
    case = {c.name: c for c in CASES}["config1_c1.0"]   # 11 iterations in the reference
    b = ffcz.DualBounds(case.E, case.Dre, case.Dim)
    r = ffcz.correct(case.original, case.decompressed, b, case.m, case.max_iters, case.precision,
                     policy="mixed", want_archive=False)
    f64 = ffcz.correct(case.original, case.decompressed, b, case.m, case.max_iters,
                       case.precision, want_archive=False)
    assert f64.iterations_fp32 == 0
    assert r.iterations_fp32 >= 1                           # the FP32 phase ran
    assert r.report.iterations - r.iterations_fp32 >= 1     # and handed over to FP64
    assert abs(r.report.iterations - f64.report.iterations) <= 1
    # corrected fields agree to the FP32 phase's perturbation (<< E)
    assert np.max(np.abs(r.corrected - f64.corrected)) <= 1e-3 * case.E


def test_policy_validation(ffcz):
    case = CASES[0]
    b = ffcz.DualBounds(case.E, case.Dre, case.Dim)
    with pytest.raises(ffcz.ValidationError):
        ffcz.correct(case.original, case.decompressed, b, policy="fp16")
    with pytest.raises(ffcz.ValidationError):
        ffcz.correct(case.original, case.decompressed, b, policy="mixed", tau=2.0)
