"""Generate the golden vectors from the UNMODIFIED CPU reference (oracle/_ref, built from
/root/reference by oracle/Makefile).  Run here (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Writes tests/golden/inputs.npz (inputs whose recipe needs the reference's synth_field),
tests/golden/golden.json (report / escape / verify scalars per case, plus the edit digest: flag
and code hashes decoded by the reference's own read_archive, cases.edit_digest) and
tests/golden/archives.npz (the reference's archive bytes per case, small ones only).

    python tests/golden/make_golden.py --big [names...]

runs the BASELINE-size cases (cases.BIG_CASES: config 2 at 256^3 / 512^3, one 2048^2 config-3
frame, config 4 at 256^3) through the reference with the MKL-backed FFT provider and writes
tests/golden/golden_big.json: report scalars, input digests (so the GPU box can tell input drift
from a parity failure) and edit digests.  The small set runs on the radix-2 stand-in provider
(FFCZ_REF_FFT=radix2) so its numbers stay those pinned since round 1.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

if len(sys.argv) > 1 and sys.argv[1] == "--big":
    os.environ.setdefault("FFCZ_REF_FFT", "mkl")
else:
    os.environ.setdefault("FFCZ_REF_FFT", "radix2")
from oracle import ref_binding as ref  # noqa: E402
import cases  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def make_inputs():
    # config 1: synth_field(power_law, alpha=3, seed=20260117), 64^3, f32
    o = ref.synth_field(1, (64, 64, 64), 20260117, 3.0).astype(np.float32).astype(np.float64)
    E = 0.1 / 100.0 * cases.value_range(o)
    d = cases.uniform_perturb(o, E, 7)
    # config 2 recipe at 32^3: log-normal of a power-law GRF (alpha = 2.5), rho = 1e-3
    g = ref.synth_field(1, (32, 32, 32), 424242, 2.5)
    rho_b = np.exp(1.5 * g / g.std() - 1.125).astype(np.float32).astype(np.float64)
    E2 = 0.1 / 100.0 * cases.value_range(rho_b)
    d2 = cases.uniform_perturb(rho_b, E2, 8)
    delta = ref.rho_bounds(rho_b, 1e-3)
    # decompressed fields are regenerated from numpy's PCG64 (cases.uniform_perturb)
    np.savez_compressed(os.path.join(OUT, "inputs.npz"), c1_orig=o.astype(np.float32),
                        c2_orig=rho_b.astype(np.float32), c2_delta=delta)


def record(r) -> dict:
    e = ref.archive_edits(r.archive)
    g = {
        "iterations": r.report.iterations, "active_spatial": r.report.active_spatial,
        "active_frequency": r.report.active_frequency, "converged": r.report.converged,
        "residual_f": r.report.residual_f, "residual_s": r.report.residual_s,
        "escape_count": r.escape_count, "verify_ok": r.verify_ok,
        "verify_max_spatial_excess": r.verify_max_spatial_excess,
        "verify_max_freq_excess": r.verify_max_freq_excess, "archive_len": len(r.archive),
        "correct_wall_s": r.correct_wall_s,
        "archive_sha256": hashlib.sha256(r.archive).hexdigest(),
        "digest": cases.edit_digest(e.spatial_flags, e.frequency_flags, e.spatial_codes,
                                    e.frequency_codes, e.escape_index, e.escape_frequency),
    }
    return g


def main_big(names):
    path = os.path.join(OUT, "golden_big.json")
    golden = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        c = cases.big_case(name)
        r = ref.correct(c.original, c.decompressed, c.E, c.Dre, c.Dim, c.m, c.max_iters,
                        c.precision)
        g = record(r)
        g["inputs"] = cases.input_digest(c)
        g["shape"] = list(c.original.shape)
        g["fft_provider"] = ref.fft_backend()
        golden[name] = g
        print(f"{name:22s} it={r.report.iterations:3d} s={r.report.active_spatial:9d} "
              f"f={r.report.active_frequency:10d} esc={r.escape_count:6d} ok={r.verify_ok} "
              f"arch={len(r.archive)} t={r.correct_wall_s:.1f}s", flush=True)
        del c, r
        with open(path, "w") as f:
            json.dump(golden, f, indent=1, sort_keys=True)


def main():
    make_inputs()
    golden, archives = {}, {}
    for c in cases.all_cases():
        try:
            r = ref.correct(c.original, c.decompressed, c.E, c.Dre, c.Dim, c.m, c.max_iters,
                            c.precision)
        except ref.RefError as e:
            golden[c.name] = {"error": e.kind, "message": str(e)}
            continue
        golden[c.name] = record(r)
        if len(r.archive) <= 256 * 1024:  # keep the fixture small; larger ones by hash only
            archives[c.name] = np.frombuffer(r.archive, dtype=np.uint8)
        print(f"{c.name:22s} it={r.report.iterations:3d} s={r.report.active_spatial:6d} "
              f"f={r.report.active_frequency:7d} esc={r.escape_count:4d} ok={r.verify_ok} "
              f"arch={len(r.archive)} t={r.correct_wall_s:.2f}s")
    # hand trace (alternating_projection seam)
    eps0, E, D = cases.hand_trace()
    S, F, eps, rep = ref.alternating_projection(eps0, E, D, None, 100)
    golden["hand_trace"] = {"iterations": rep.iterations, "active_spatial": rep.active_spatial,
                            "active_frequency": rep.active_frequency, "converged": rep.converged,
                            "final_epsilon": eps.tolist(), "F_re": F.real.tolist(),
                            "F_im": F.imag.tolist()}
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(golden, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(OUT, "archives.npz"), **archives)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--big":
        main_big(sys.argv[2:] or list(cases.BIG_CASES))
    else:
        main()
