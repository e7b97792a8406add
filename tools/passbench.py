"""Per-pass micro-benchmark of the FFT engine (ffcz_cuda_bench_passes): achieved GB/s of every
pass kind against the measured HBM copy peak.  Usage: python tools/passbench.py [n] [reps]"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2601_01596_b200 import _capi  # noqa: E402
import paper_2601_01596_b200 as P  # noqa: E402


def run(shape, dtype, reps, ctx, peak):
    lib = _capi.load()
    fd = _capi.FieldDesc()
    fd.ndim = len(shape)
    for i, s in enumerate(shape):
        fd.dims[i] = s
    fd.dtype = dtype
    fd.precision = 1
    stats = (_capi.KernelStat * 32)()
    n = C.c_int()
    rc = lib.ffcz_cuda_bench_passes(ctx.handle, C.byref(fd), reps, stats, 32, C.byref(n))
    if rc:
        raise RuntimeError(lib.ffcz_cuda_last_error().decode())
    for i in range(n.value):
        s = stats[i]
        ms = s.total_ms / s.launches
        gbs = s.bytes / (s.total_ms * 1e-3) / 1e9
        print(json.dumps({"shape": list(shape), "dtype": "f64" if dtype else "f32",
                          "pass": s.name.decode(), "ms": round(ms, 4), "GBps": round(gbs, 1),
                          "frac_of_peak": round(gbs / peak, 3)}))


def main():
    # argv[1]: n (n^3 and 2048^2) or a comma list of shapes "AxBxC,..."; argv[3]: f64|f32|both
    spec = sys.argv[1] if len(sys.argv) > 1 else "512"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    which = sys.argv[3] if len(sys.argv) > 3 else "both"
    dts = {"f64": (1,), "f32": (0,), "both": (1, 0)}[which]
    peak = 6548.2
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peak = json.load(open(pk))["hbm_gbs"]
    ctx = P.Context(0)
    if "x" in spec:
        shapes = [tuple(int(v) for v in sh.split("x")) for sh in spec.split(",")]
    else:
        n = int(spec)
        shapes = [(n, n, n), (2048, 2048)]
    for shape in shapes:
        for dt in dts:
            run(shape, dt, reps, ctx, peak)


if __name__ == "__main__":
    main()
