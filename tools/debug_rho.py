"""Config-2 workload with the cuFFT Delta vs the library's device bound: correct() outcome."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2601_01596_b200 as P

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
ctx = P.Context(0, stream.cuda_stream)
for n in [int(v) for v in sys.argv[1:]] or [64, 128, 256, 512]:
    orig, dec, E, dt = bench.make_workload(n, 1234, dev)
    dl = P.spectrum_bound_to_freq_bounds(orig, bench.RHO, ctx=ctx)
    diff = (dl - dt).abs()
    print(n, "max|dl-dt|", diff.max().item(), "rel", (diff / dt).max().item(),
          "asym_lib", (dl.flatten() != dl.flip(0).flip(1).flip(2).roll((1, 1, 1), (0, 1, 2)).flatten()).sum().item(),
          flush=True)
    for name, D in (("torch", dt), ("lib", dl)):
        r = P.correct(orig, dec, P.DualBounds(E, D), 16, 1000, "f32", want_archive=False,
                      want_corrected=False, ctx=ctx)
        print(" ", name, r.report.iterations, r.verify_ok, r.verify_max_spatial_excess, r.verify_max_freq_excess, getattr(r, "escape_rounds", None),
              len(r.escapes), r.report.active_frequency, flush=True)
