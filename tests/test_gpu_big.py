"""GPU parity at the BASELINE sizes: config 2 at 256^3 and 512^3 (the driver's
headline workload recipe, rho-mode per-component Delta), one 2048^2 config-3 frame, config 4 at
256^3.  The reference outputs come from the UNMODIFIED reference run here
(tests/golden/make_golden.py --big, MKL-backed FFT provider) and are pinned in
tests/golden/golden_big.json as report scalars plus digests: input hashes (so input drift is
told apart from a parity failure), flag hashes and per-65,536-code block hashes of the int32
codes decoded by the reference's own read_archive.

Bar, FP64 policy: iterations, converged, active counts and verify exact (where the reference's
own verify flags round-off, this side must verify); flags identical; every code block identical
(at most 0.1 % of the blocks above 1000 blocks: FFT round-off at quantisation ties); escape keys identical or counts within 10 %; the FP64
corrected field satisfies the spatial bound exactly and every frequency component
|Re d_k| - D_k <= 1e-15 D_k (and Im) under numpy's FFT."""
import json
import os

import numpy as np
import pytest

import cases

pytestmark = pytest.mark.gpu

PATH = os.path.join(cases.GOLDEN, "golden_big.json")
GOLD = json.load(open(PATH)) if os.path.exists(PATH) else {}
NAMES = [n for n in cases.BIG_CASES if n in GOLD]


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2601_01596_b200 as P
    return P


@pytest.mark.parametrize("name", NAMES)
def test_big_case_matches_reference(P, name):
    g = GOLD[name]
    c = cases.big_case(name)
    assert cases.input_digest(c) == g["inputs"], "input recipe drifted from the golden run"
    o32 = c.original.astype(np.float32)
    d32 = c.decompressed.astype(np.float32)
    r = P.correct(o32, d32, P.DualBounds(c.E, c.Dre, c.Dim), c.m, c.max_iters, c.precision,
                  want_archive=False, want_edits=True, want_corrected=True)
    rep = r.report
    assert (rep.iterations, rep.converged, rep.active_spatial, rep.active_frequency) == \
        (g["iterations"], g["converged"], g["active_spatial"], g["active_frequency"]), rep
    if g["verify_ok"]:
        assert r.verify_ok
    else:
        # the reference's own FP64 verify flags round-off on its output (config 2 at 512^3:
        # 3.6e-14 on one component); the decoder-view repair
        # repairs exactly those, so this side must verify
        assert g["verify_max_spatial_excess"] == 0.0
        assert g["verify_max_freq_excess"] <= 1e-12 * float(np.max(c.Dre))
        assert r.verify_ok
    cmp = cases.compare_digest(cases.digest_of_result(r), g["digest"])
    print(name, "escapes (mine, ref):", cmp["n_escapes"], "rounds:", r.escape_rounds)
    assert cmp["flags"], cmp
    # int32 codes are bit-exact wherever the FP64 projected values agree; an
    # FFT round-off difference (this FFT vs MKL's) can move a value across a quantisation tie:
    # at 512^3 (134M frequency codes, 2050 blocks) one 65,536-code block differs.  Allowed: 0.1 %
    # of the blocks when there are more than 1000, none below
    nblk = len(g["digest"]["blocks_f"])
    assert cmp["code_blocks_s"] == 0 and cmp["code_blocks_f"] <= nblk // 1000, cmp
    ne, ne_ref = cmp["n_escapes"]
    assert cmp["escapes"] or abs(ne - ne_ref) <= max(2, ne_ref // 10), cmp
    # the guarantee on the FP64 corrected field, checked independently of the engine
    corr = r.corrected
    del r
    assert float(np.max(np.abs(corr - c.original) - c.E)) <= 0.0
    rel = cases.freq_excess_per_component(c.original, corr, c.Dre, c.Dim)
    assert rel <= 1e-15, rel


@pytest.mark.parametrize("name", [n for n in ("config4_comb256", "config3_xrd2048") if n in GOLD])
def test_big_case_mixed_policy(P, name):
    """The mixed FP32 -> FP64 policy (SURVEY.md §8c parity contract for the FP32 target):
    iterations within +-1 of the reference, converged and verified, both bounds exact on the
    FP64 corrected field.  Flags follow the FP32 phase's round-off on borderline components
    (config 4 at 256^3: a few in 10^5 differ; SURVEY.md §8c(5)-(6) pins them only in FP64
    mode): active counts within 1e-4 of the reference's."""
    g = GOLD[name]
    c = cases.big_case(name)
    r = P.correct(c.original.astype(np.float32), c.decompressed.astype(np.float32),
                  P.DualBounds(c.E, c.Dre, c.Dim), c.m, c.max_iters, c.precision,
                  want_archive=False, want_edits=True, want_corrected=True, policy="mixed")
    rep = r.report
    print(name, "mixed: iterations", rep.iterations, "(fp32", r.iterations_fp32, ") ref",
          g["iterations"])
    assert abs(rep.iterations - g["iterations"]) <= 1
    assert rep.converged == g["converged"] and r.verify_ok
    for k in ("active_spatial", "active_frequency"):
        mine, ref = getattr(rep, k), g[k]
        print(name, k, mine, ref)
        assert abs(mine - ref) <= max(2, 1e-4 * ref), (k, mine, ref)
    corr = r.corrected
    del r
    assert float(np.max(np.abs(corr - c.original) - c.E)) <= 0.0
    assert cases.freq_excess_per_component(c.original, corr, c.Dre, c.Dim) <= 1e-15
