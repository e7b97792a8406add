"""Escape composition of one correct() at the bench workload (spatial vs frequency)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import bench  # noqa: E402
import paper_2601_01596_b200 as P  # noqa: E402


def main():
    import torch
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    dev = torch.device("cuda", 0)
    o, d, E, D = bench.make_workload(n, 1234, dev)
    torch.cuda.empty_cache()
    r = P.correct(o, d, P.DualBounds(E, D), 16, 1000, "f32", want_archive=False,
                  want_corrected=False)
    f = r.escapes["frequency"] != 0
    print({"n": n, "iterations": r.report.iterations, "rounds": r.escape_rounds,
           "escapes": int(r.escape_count), "spatial": int((~f).sum()), "frequency": int(f.sum()),
           "active_s": r.report.active_spatial, "active_f": r.report.active_frequency})


if __name__ == "__main__":
    main()
