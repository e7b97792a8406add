"""The loop's check + clip as one round-trip column pass (HookRT / k_col_tma1_rt, the default)
against the two-pass K3a / K3b loop (FFCZ_LOOP_RT=0, read once per process: a subprocess).

The round trip clips speculatively before the decision; when the decision ends the loop the
reference never clips (projection.cpp:104-116), so the engine re-forms the spectrum and clears
the marks only that clip set.  Both endings are covered: converged, and max_iters reached
(the speculative clip of the last check moves components).  The golden suite
(test_gpu_parity.py) pins the default path against the unmodified reference; this file pins
the loop forms against each other on the golden cases, run to convergence and cut short.
The fused K1 row pass (FFCZ_LOOP_K1) is switched off with it in the two-pass run."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SNIPPET = r"""
import sys, json, hashlib
sys.path.insert(0, %r); sys.path.insert(0, %r)
import numpy as np
import cases
import paper_2601_01596_b200 as P
by_name = {c.name: c for c in cases.all_cases()}
out = {}
for name, iters in %r:
    c = by_name[name]
    r = P.correct(c.original, c.decompressed, P.DualBounds(c.E, c.Dre, c.Dim), c.m,
                  iters or c.max_iters, c.precision)
    out["%%s/%%s" %% (name, iters)] = {
        "iterations": r.report.iterations, "converged": bool(r.report.converged),
        "residual_f": r.report.residual_f, "active_s": r.report.active_spatial,
        "active_f": r.report.active_frequency, "verify_ok": bool(r.verify_ok),
        "escapes": int(r.escape_count),
        "flags": hashlib.sha256(r.frequency_flags.tobytes() + r.spatial_flags.tobytes()).hexdigest(),
        "codes": hashlib.sha256(r.frequency_codes.tobytes() + r.spatial_codes.tobytes()).hexdigest(),
        "corrected": np.asarray(r.corrected, dtype=np.float64).ravel().tolist()}
print(json.dumps(out))
"""

# (golden case, max_iters override or None): multi-iteration cases, and the same cases cut
# short so the loop ends at max_iters with a speculative clip that moves components
CASES = [
    ("config1_c0.6", None), ("config1_c0.6", 5), ("config1_c0.6", 1),
    ("config1_c1.0", None), ("config4_comb32", None), ("config4_comb32", 4),
    ("config3_frame256", None), ("config3_frame256", 3), ("accept_09", None),
    ("m8_32cube", None), ("per_point_2d", None), ("per_point_2d", 2), ("accept_06", None),
]


def _run(rt):
    env = dict(os.environ)
    if rt:
        env.pop("FFCZ_LOOP_RT", None)
        env.pop("FFCZ_LOOP_K1", None)
    else:
        env["FFCZ_LOOP_RT"] = "0"
        env["FFCZ_LOOP_K1"] = "0"
    env["PYTHONHASHSEED"] = "0"
    code = _SNIPPET % (ROOT, os.path.join(ROOT, "tests"), CASES)
    p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_round_trip_loop_matches_two_pass_loop():
    two = _run(False)
    rt = _run(True)
    assert set(two) == set(rt) and len(rt) == len(CASES)
    ended_by_max = 0
    for name in two:
        a, b = two[name], rt[name]
        ca, cb = np.array(a.pop("corrected")), np.array(b.pop("corrected"))
        # the spectrum of the completing axis comes from another FFT kernel (round-off level)
        assert np.abs(ca - cb).max() <= 1e-12 * max(1.0, np.abs(ca).max()), name
        ra, rb = a.pop("residual_f"), b.pop("residual_f")
        assert abs(ra - rb) <= 1e-9 * max(abs(ra), 1e-300), (name, ra, rb)
        assert a == b, (name, a, b)
        ended_by_max += not b["converged"]
    # the max_iters ending (speculative last clip) is exercised
    assert ended_by_max >= 3, {k: (v["iterations"], v["converged"]) for k, v in rt.items()}
