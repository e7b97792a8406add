"""Kernel cost of the fused slab transpose, emulated in one process (both ranks' receive buffers
local): FWD_LOCAL + pack copy vs FWD_LOCAL_PEER; COL0_CLIP_INV + pack vs COL0_CLIP_INV_PEER.
Also checks the scattered buffers equal the packed ones."""
import json, sys, torch
sys.path.insert(0, ".")
from paper_2601_01596_b200.slab_gpu import GpuSlabBackend
from paper_2601_01596_b200 import slab

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
W = 2
dev = torch.device("cuda", 0)
be = GpuSlabBackend(n, dev)
c0 = c1 = n // W
P = be.P
out = {"n": n, "W": W}
with torch.cuda.stream(be.stream):
    g = torch.Generator(device=dev).manual_seed(1)
    eps = torch.randn((c0, n, n), dtype=torch.float64, device=dev, generator=g)
    A = be.zeros_half((c0, n))
    Bs = [be.zeros_half((n, c1)) for _ in range(W)]
    peer = {"A": A, "B": Bs[0], "W": W, "r": 0,
            "to_B": torch.tensor([b.data_ptr() for b in Bs], dtype=torch.int64, device=dev)}

    class C1:  # local "all-to-all": the permute copy of slab._transpose_ab, W = 1 comm
        size = 1
    def ev():
        return torch.cuda.Event(enable_timing=True)

    def timeit(f, reps=10):
        for _ in range(2):
            f()
        a, b = ev(), ev()
        a.record(be.stream)
        for _ in range(reps):
            f()
        b.record(be.stream)
        b.synchronize()
        return a.elapsed_time(b) / reps

    def plain_fwd():
        be.fwd_local(eps, A, n ** 3)
        send = A.view(c0, W, c1, P).permute(1, 0, 2, 3).contiguous()
        return send
    out["fwd_plain_ms"] = timeit(lambda: be.fwd_local(eps, A, n ** 3))
    out["fwd_plain_pack_ms"] = timeit(plain_fwd)
    out["fwd_peer_ms"] = timeit(lambda: be.fwd_local_peer(eps, peer))
    # check: rank 0's contribution lands in Bs[s] rows (i0 in [0, c0)) = send[s]
    send = plain_fwd()
    be.fwd_local_peer(eps, peer)
    torch.cuda.synchronize()
    H = n // 2 + 1
    out["fwd_match"] = all(bool(torch.equal(Bs[s][:c0, :, :H], send[s][:, :, :H])) for s in range(W))
    # backward: clip + inverse axis 0 of B, scattered into A buffers of both ranks
    B = Bs[0]
    F = be.zeros_half((n, c1))
    moved = be.zeros_moved((n, c1))
    As = [be.zeros_half((c0, n)) for _ in range(W)]
    peerb = {"A": As[0], "B": B, "W": W, "r": 0,
             "to_A": torch.tensor([a.data_ptr() for a in As], dtype=torch.int64, device=dev)}
    Bsave = B.clone()
    D = 1e-3 * float(B.abs().max())
    def plain_clip():
        B.copy_(Bsave)
        be.col0_clip_inv(B, D, 1.0, F, moved, False)
        return B.reshape(W, c0, c1, P)
    def peer_clip():
        be.col0_clip_inv_peer(D, 1.0, F, moved, False, peerb)
    out["copy_ms"] = timeit(lambda: B.copy_(Bsave))
    out["clip_plain_ms(incl copy)"] = timeit(lambda: plain_clip())
    out["clip_peer_ms"] = timeit(peer_clip)
    recv = plain_clip().clone()
    B.copy_(Bsave)
    peer_clip()
    torch.cuda.synchronize()
    # rank 0 holds i1 in [0, c1): As[s][:, 0:c1] = recv[s]
    out["clip_match"] = all(bool(torch.equal(As[s][:, :c1, :H], recv[s][:, :, :H])) for s in range(W))
print(json.dumps(out))
