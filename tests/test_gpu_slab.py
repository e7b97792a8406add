"""Slab-decomposed correction on the B200 engine (GpuSlabBackend, ffcz_cuda_slab): at world 1 it
must reproduce the single-volume engine path and the oracle; at world 2 (two ranks sharing the
GPU, collectives staged through gloo) it must agree with world 1 exactly as the CPU stand-in
does (tests/test_slab_dist.py)."""
import os
import pickle
import socket
import sys
import tempfile

import numpy as np
import pytest

import cases
from oracle import ffcz_oracle as O

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def field(n, seed, c):
    o = cases.combustion(n, seed)
    E = 0.1 / 100.0 * cases.value_range(o)
    d = cases.uniform_perturb(o, E, seed + 1)
    return o, d, E, c * cases.mean_abs_delta0(o, d)


def bound_arrays(n, E, D, seed):
    """Per-point E (>= the global E of the perturbation) and Hermitian-consistent per-component
    (Re, Im) Delta lanes."""
    rng = np.random.default_rng(seed + 50)
    shape = (n, n, n)
    def sym(g):  # exactly Hermitian-consistent: g[k] == g[-k] bit for bit (bounds.cpp:50-54)
        return 0.5 * (g + np.roll(np.flip(g), 1, axis=tuple(range(g.ndim))))
    g1 = sym(np.abs(np.fft.fftn(rng.standard_normal(shape))))
    g2 = sym(np.abs(np.fft.fftn(rng.standard_normal(shape))))
    return (E * (1.0 + rng.uniform(0.0, 1.0, shape)), D * (0.6 + g1 / g1.max()),
            D * (0.7 + 0.5 * g2 / g2.max()))


def _worker(rank, world, port, n, seed, c, out_dir, arrays=False, peer=True):
    os.environ["FFCZ_SLAB_PEER"] = "1" if peer else "0"
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    from paper_2601_01596_b200 import slab
    from paper_2601_01596_b200.slab_gpu import GpuSlabBackend
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o, d, E, D = field(n, seed, c)
        c0 = n // world
        sl = slice(rank * c0, (rank + 1) * c0)
        to = torch.from_numpy(o[sl].astype(np.float32)).cuda()
        td = torch.from_numpy(d[sl].astype(np.float32)).cuda()
        be = GpuSlabBackend(n, to.device)
        if arrays:
            Ea, Dre, Dim = bound_arrays(n, E, D, seed)
            E = torch.from_numpy(Ea[sl].copy()).cuda()
            D = (torch.from_numpy(Dre[sl].copy()).cuda(), torch.from_numpy(Dim[sl].copy()).cuda())
        res = slab.correct_slab(be, slab.Comm(stage_cpu=True), (n, n, n), to, td, E, D)
        torch.cuda.synchronize()
        res.corrected = res.corrected.cpu().numpy()
        _to_host(res, n)
        with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as f:
            pickle.dump(res, f)
        be.ctx.close()
    finally:
        dist.destroy_process_group()


def _to_host(res, n):
    from paper_2601_01596_b200.slab_gpu import GpuSlabBackend
    ns = res.corrected.size if hasattr(res.corrected, "size") else res.corrected.numel()
    H = n // 2 + 1
    res.spatial_flags = GpuSlabBackend.flags_to_bool(res.spatial_flags, ns)
    res.frequency_flags = GpuSlabBackend.flags_to_bool(res.frequency_flags, ns // n * H)
    res.spatial_codes = res.spatial_codes.cpu().numpy()
    res.frequency_codes = res.frequency_codes.cpu().numpy()


def run_world(world, n, seed, c, arrays=False, peer=True):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, _free_port(), n, seed, c, tmp, arrays, peer),
                 nprocs=world, join=True)
        return [pickle.load(open(os.path.join(tmp, f"r{r}.pkl"), "rb")) for r in range(world)]


def cat(parts, k):
    return np.concatenate([getattr(p, k) for p in parts])


@pytest.mark.parametrize("n,c", [(32, 0.6), (32, 1.0), (64, 0.6)])
def test_slab_gpu_world1_matches_engine_and_oracle(n, c):
    import torch
    import paper_2601_01596_b200 as P
    from paper_2601_01596_b200.slab_gpu import correct_slab_gpu
    o, d, E, D = field(n, 5, c)
    to = torch.from_numpy(o.astype(np.float32)).cuda()
    td = torch.from_numpy(d.astype(np.float32)).cuda()
    res = correct_slab_gpu(to, td, (n, n, n), E, D)
    res.corrected = res.corrected.cpu().numpy()
    _to_host(res, n)
    ref = O.correct(o, d, O.DualBounds(E, D), 16, 1000, "f32")
    eng = P.correct(o.astype(np.float32), d.astype(np.float32), P.DualBounds(E, D), 16, 1000,
                    "f32")
    for r in (ref.report, eng.report):
        assert res.iterations == r.iterations
        assert res.converged == r.converged
        assert res.active_spatial == r.active_spatial
        assert res.active_frequency == r.active_frequency
    assert res.verify_ok and eng.verify_ok
    arch = O.read_archive(eng.archive_bytes)
    assert np.array_equal(res.spatial_flags, arch.spatial_flags.ravel())
    assert np.array_equal(res.frequency_flags, arch.frequency_flags.ravel())
    assert np.mean(res.frequency_codes == arch.frequency_codes) >= 0.999
    ok, ms, mf = O.verify_bounds(o, res.corrected, O.DualBounds(E, D))
    assert ms == 0.0 and mf <= 1e-12 * D
    assert abs(len(res.escapes) - eng.escape_count) <= max(2, eng.escape_count // 10)


@pytest.mark.parametrize("world", [2, 4])
def test_slab_gpu_worlds_agree(world):
    n, seed, c = 32, 7, 0.7
    a, b = run_world(1, n, seed, c), run_world(world, n, seed, c)
    for k in ("iterations", "converged", "active_spatial", "active_frequency", "verify_ok",
              "escape_rounds"):
        assert getattr(a[0], k) == getattr(b[0], k), k
    for k in ("spatial_flags", "frequency_flags", "spatial_codes", "frequency_codes"):
        assert np.array_equal(cat(a, k), cat(b, k)), k
    assert [e[:2] for e in a[0].escapes] == [e[:2] for e in b[0].escapes]
    ca, cb = cat(a, "corrected"), cat(b, "corrected")
    np.testing.assert_allclose(ca, cb, rtol=0, atol=1e-12 * np.abs(ca).max())


@pytest.mark.parametrize("world,n,c,arrays", [(2, 32, 0.7, False), (4, 32, 0.7, False),
                                              (2, 64, 0.6, False), (2, 32, 0.7, True)])
def test_slab_gpu_peer_transpose_matches_all_to_all(world, n, c, arrays):
    """The fused all-to-all (the forward axis-1 pass and the clip + inverse axis-0 pass storing
    straight into the other ranks' receive buffers over CUDA IPC; here two / four processes on
    one GPU) moves the same values as the NCCL / gloo all-to-all path: every product identical,
    bit for bit."""
    a = run_world(world, n, 7, c, arrays=arrays, peer=False)
    b = run_world(world, n, 7, c, arrays=arrays, peer=True)
    for k in ("iterations", "converged", "active_spatial", "active_frequency", "verify_ok",
              "escape_rounds", "residual_f", "residual_s"):
        assert getattr(a[0], k) == getattr(b[0], k), k
    for k in ("spatial_flags", "frequency_flags", "spatial_codes", "frequency_codes",
              "corrected"):
        assert np.array_equal(cat(a, k), cat(b, k)), k
    assert list(a[0].escapes) == list(b[0].escapes)


@pytest.mark.parametrize("world", [1, 2])
def test_slab_gpu_bound_arrays(world):
    """Per-point E and per-component (Re, Im) Delta split across ranks like the field
    (bounds.hpp:11-47): the ranks' products equal the single-volume engine's with the same
    DualBounds arrays, and the guarantee holds against those bounds."""
    import paper_2601_01596_b200 as P
    n, seed, c = 32, 7, 0.7
    o, d, E, D = field(n, seed, c)
    Ea, Dre, Dim = bound_arrays(n, E, D, seed)
    parts = run_world(world, n, seed, c, arrays=True)
    eng = P.correct(o.astype(np.float32), d.astype(np.float32), P.DualBounds(Ea, Dre, Dim), 16,
                    1000, "f32")
    ref = O.correct(o, d, O.DualBounds(Ea, Dre, Dim), 16, 1000, "f32")
    r0 = parts[0]
    for r in (eng.report, ref.report):
        assert (r0.iterations, r0.converged, r0.active_spatial, r0.active_frequency) == \
            (r.iterations, r.converged, r.active_spatial, r.active_frequency)
    assert r0.verify_ok and eng.verify_ok
    arch = O.read_archive(eng.archive_bytes)
    assert np.array_equal(cat(parts, "spatial_flags"), arch.spatial_flags.ravel())
    assert np.array_equal(cat(parts, "frequency_flags"), arch.frequency_flags.ravel())
    assert np.mean(cat(parts, "frequency_codes") == arch.frequency_codes) >= 0.999
    ok, ms, mf = O.verify_bounds(o, cat(parts, "corrected"), O.DualBounds(Ea, Dre, Dim))
    assert ok and ms == 0.0
