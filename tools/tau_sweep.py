"""Mixed-policy switch point sweep on the bench workload (1024^3 config-4 recipe by default):
iterations, FP32 iterations, device time, and agreement of the edit set with the FP64 policy.
Usage: python tools/tau_sweep.py [n] [tau,...]"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2601_01596_b200 as P  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    taus = [float(t) for t in (sys.argv[2] if len(sys.argv) > 2 else "1e-4,1e-5,1e-6,1e-7").split(",")]
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    ctx = P.Context(0, stream.cuda_stream)
    orig, dec, E, delta = bench.make_workload_combustion(n, 4321, dev)
    torch.cuda.empty_cache()
    b = P.DualBounds(E, delta)

    def run(policy, tau):
        P.correct(orig, dec, b, 16, 1000, "f32", want_archive=False, want_edits=False,
                  want_corrected=False, policy=policy, tau=tau, ctx=ctx)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = P.correct(orig, dec, b, 16, 1000, "f32", want_archive=False, want_edits=True,
                      want_corrected=False, policy=policy, tau=tau, ctx=ctx)
        e1.record(stream)
        torch.cuda.synchronize()
        h = hashlib.sha256(r.frequency_flags.tobytes() + r.spatial_flags.tobytes()).hexdigest()[:16]
        return {"policy": policy, "tau": tau, "ms": round(e0.elapsed_time(e1), 1),
                "iterations": r.report.iterations, "iterations_fp32": r.iterations_fp32,
                "active_s": r.report.active_spatial, "active_f": r.report.active_frequency,
                "escapes": int(r.escape_count), "verify_ok": bool(r.verify_ok), "flags": h}

    print(json.dumps(run("fp64", 1e-4)), flush=True)
    for t in taus:
        print(json.dumps(run("mixed", t)), flush=True)


if __name__ == "__main__":
    main()
