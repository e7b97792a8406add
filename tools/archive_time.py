"""Archive serialisation time at 512^3 (config-2 workload): host Huffman + zlib-9 (byte-identical
to the reference) vs device Huffman + host outer stage at zlib level 1 / 0 (stored)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2601_01596_b200 as P  # noqa: E402


def main():
    import torch
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    dev = torch.device("cuda", 0)
    o, d, E, D = bench.make_workload(n, 1234, dev)
    torch.cuda.empty_cache()
    ctx = P.Context(0, torch.cuda.current_stream(dev).cuda_stream)
    b = P.DualBounds(E, D)
    out = {}
    for name, kw in [("host_zlib9", dict()), ("device_huffman_zlib9", dict(device_encode=True)),
                     ("device_huffman_zlib1", dict(device_encode=True, zlib_level=1)),
                     ("device_huffman_stored", dict(device_encode=True, zlib_level=0))]:
        r = P.correct(o, d, b, 16, 1000, "f32", want_corrected=False, ctx=ctx, **kw)
        out[name] = {"t_archive_ms": r.timings_ms["t_archive_ms"], "bytes": len(r.archive_bytes),
                     "t_feasible_ms": r.timings_ms["t_feasible_ms"]}
        print(json.dumps({name: out[name]}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
