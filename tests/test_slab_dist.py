"""Slab-decomposed correction — the orchestration of
paper_2601_01596_b200/slab.py (transposes, all-reduced decisions, cross-rank escape repair) under
gloo at world sizes 1, 2 and 4 on CPU, with the torch stand-in backend for the device passes.
Every world size must reproduce the reference control flow of a single-volume correct()
(pipeline.cpp:26-178) on the same inputs, checked against the numpy oracle."""
import os
import pickle
import socket
import sys
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import cases
from oracle import ffcz_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def field(shape, seed, c):
    o = cases.combustion(shape[0], seed)[: shape[0], : shape[1], : shape[2]] \
        if shape[0] == shape[1] == shape[2] else cases.noise(shape, seed, "f32")
    E = 0.1 / 100.0 * cases.value_range(o) if shape[0] == shape[1] == shape[2] else 0.05
    d = cases.uniform_perturb(o, E, seed + 1)
    D = c * cases.mean_abs_delta0(o, d)
    return o, d, E, D


def bound_arrays(shape, o, E, D, seed):
    """Per-point E (>= the global E the perturbation respects) and per-component (Re, Im)
    Delta lanes, Hermitian-consistent (|FFT(real)| is symmetric under k -> -k)."""
    rng = np.random.default_rng(seed + 50)
    Ea = E * (1.0 + rng.uniform(0.0, 1.0, shape))
    def sym(g):  # exactly Hermitian-consistent: g[k] == g[-k] bit for bit (bounds.cpp:50-54)
        return 0.5 * (g + np.roll(np.flip(g), 1, axis=tuple(range(g.ndim))))
    g1 = sym(np.abs(np.fft.fftn(rng.standard_normal(shape))))
    g2 = sym(np.abs(np.fft.fftn(rng.standard_normal(shape))))
    return Ea, D * (0.6 + g1 / g1.max()), D * (0.7 + 0.5 * g2 / g2.max())


def _worker(rank, world, port, shape, seed, c, m, max_iters, out_dir, arrays=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (root, os.path.join(root, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    from paper_2601_01596_b200 import slab
    from slab_cpu_backend import CpuSlabBackend
    torch.set_num_threads(1)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o, d, E, D = field(shape, seed, c)
        c0 = shape[0] // world
        sl = slice(rank * c0, (rank + 1) * c0)
        be = CpuSlabBackend(shape[2])
        if arrays:
            Ea, Dre, Dim = bound_arrays(shape, o, E, D, seed)
            E = torch.from_numpy(Ea[sl].copy())
            D = (torch.from_numpy(Dre[sl].copy()), torch.from_numpy(Dim[sl].copy()))
        res = slab.correct_slab(be, slab.Comm(), shape, torch.from_numpy(o[sl].copy()),
                                torch.from_numpy(d[sl].copy()), E, D, m, max_iters)
        res.corrected = res.corrected.numpy()
        with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as f:
            pickle.dump(res, f)
    finally:
        dist.destroy_process_group()


def run_world(world, shape, seed=3, c=0.6, m=16, max_iters=1000, arrays=False):
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, _free_port(), shape, seed, c, m, max_iters, tmp, arrays),
                 nprocs=world, join=True)
        parts = [pickle.load(open(os.path.join(tmp, f"r{r}.pkl"), "rb")) for r in range(world)]
    return parts


def merged(parts):
    p0 = parts[0]
    return dict(
        iterations=p0.iterations, converged=p0.converged, active_s=p0.active_spatial,
        active_f=p0.active_frequency, verify_ok=p0.verify_ok, escapes=p0.escapes,
        sflags=np.concatenate([p.spatial_flags for p in parts]),
        fflags=np.concatenate([p.frequency_flags for p in parts]),
        scodes=np.concatenate([p.spatial_codes for p in parts]),
        fcodes=np.concatenate([p.frequency_codes for p in parts]),
        corrected=np.concatenate([p.corrected for p in parts]),
        rounds=p0.escape_rounds)


@pytest.mark.parametrize("shape,c", [((16, 16, 16), 0.6), ((16, 8, 8), 1.0), ((16, 16, 16), 2.0)])
def test_slab_world1_matches_oracle(shape, c):
    o, d, E, D = field(shape, 3, c)
    ref = O.correct(o, d, O.DualBounds(E, D), 16, 1000, "f32")
    g = merged(run_world(1, shape, c=c))
    assert g["iterations"] == ref.report.iterations
    assert g["converged"] == ref.report.converged
    assert g["active_s"] == ref.report.active_spatial
    assert g["active_f"] == ref.report.active_frequency
    arch = ref.archive
    assert np.array_equal(g["sflags"], arch.spatial_flags.ravel())
    assert np.array_equal(g["fflags"], arch.frequency_flags.ravel())
    assert np.mean(g["fcodes"] == arch.frequency_codes) >= 0.999
    assert g["verify_ok"] and ref.verify_ok
    ok, ms, mf = O.verify_bounds(o, g["corrected"], O.DualBounds(E, D))
    assert ms == 0.0 and mf <= 1e-12 * D
    assert abs(len(g["escapes"]) - len(arch.escapes)) <= max(2, len(arch.escapes) // 10)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("shape,c", [((16, 16, 16), 0.6), ((16, 8, 8), 1.0)])
def test_slab_worlds_agree(world, shape, c):
    a = merged(run_world(1, shape, c=c))
    b = merged(run_world(world, shape, c=c))
    for k in ("iterations", "converged", "active_s", "active_f", "verify_ok", "rounds"):
        assert a[k] == b[k], k
    for k in ("sflags", "fflags", "scodes", "fcodes"):
        assert np.array_equal(a[k], b[k]), k
    assert len(a["escapes"]) == len(b["escapes"])
    assert [e[:2] for e in a["escapes"]] == [e[:2] for e in b["escapes"]]
    np.testing.assert_allclose(a["corrected"], b["corrected"], rtol=0, atol=1e-12 * np.abs(a["corrected"]).max())


def test_slab_bound_arrays_match_oracle():
    """Per-point E and per-component (Re, Im) Delta split across ranks like the field
    (bounds.hpp:11-47): world 1 against the oracle, worlds 2 and 4 against world 1."""
    shape, c = (16, 16, 16), 0.6
    o, d, E, D = field(shape, 3, c)
    Ea, Dre, Dim = bound_arrays(shape, o, E, D, 3)
    ref = O.correct(o, d, O.DualBounds(Ea, Dre, Dim), 16, 1000, "f32")
    g = merged(run_world(1, shape, c=c, arrays=True))
    assert (g["iterations"], g["converged"], g["active_s"], g["active_f"]) == \
        (ref.report.iterations, ref.report.converged, ref.report.active_spatial,
         ref.report.active_frequency)
    arch = ref.archive
    assert np.array_equal(g["sflags"], arch.spatial_flags.ravel())
    assert np.array_equal(g["fflags"], arch.frequency_flags.ravel())
    assert np.mean(g["fcodes"] == arch.frequency_codes) >= 0.999
    assert g["verify_ok"] and ref.verify_ok
    ok, ms, mf = O.verify_bounds(o, g["corrected"], O.DualBounds(Ea, Dre, Dim))
    assert ok and ms == 0.0
    for world in (2, 4):
        b = merged(run_world(world, shape, c=c, arrays=True))
        for k in ("iterations", "converged", "active_s", "active_f", "verify_ok", "rounds"):
            assert g[k] == b[k], (world, k)
        for k in ("sflags", "fflags", "scodes", "fcodes"):
            assert np.array_equal(g[k], b[k]), (world, k)


# ---- cross-rank escape repair of conjugate plane partners (pipeline.cpp:140-153) ---------------

def _repair_reference(cur, ds, dt, viol, dims):
    """pipeline.cpp:140-153 verbatim over the half grid in ascending order (natural layout)."""
    n0, n1, n2 = dims
    H = n2 // 2 + 1
    out = cur.copy()
    esc = {}
    for h in np.flatnonzero(viol.ravel()):
        rv = cur.ravel()[h] + (ds.ravel()[h] - dt.ravel()[h])
        esc[h] = rv
        i0, i1, k2 = np.unravel_index(h, (n0, n1, H))
        if k2 == 0 or 2 * k2 == n2:
            hm = np.ravel_multi_index(((-i0) % n0, (-i1) % n1, k2), (n0, n1, H))
            if hm != h:
                esc[hm] = np.conj(rv)
    for h, v in esc.items():
        out.ravel()[h] = v
    return out, sorted(esc)


def _repair_worker(rank, world, port, dims, seed, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (root, os.path.join(root, "tests")):
        if p not in sys.path:
            sys.path.insert(0, p)
    from paper_2601_01596_b200 import slab
    from slab_cpu_backend import CpuSlabBackend
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cur, ds, dt, viol = _repair_inputs(dims, seed)
        n0, n1, n2 = dims
        c1 = n1 // world
        sl = slice(rank * c1, (rank + 1) * c1)
        be = CpuSlabBackend(n2)
        fc = torch.from_numpy(cur[:, sl].copy())
        pos = be.positions(torch.from_numpy(viol[:, sl].copy()))
        fixed = slab._repair_frequency(be, slab.Comm(), pos, fc, torch.from_numpy(ds[:, sl].copy()),
                                       torch.from_numpy(dt[:, sl].copy()), n0, n1, n2, c1, rank)
        with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as f:
            pickle.dump((fc.numpy(), fixed.numpy()), f)
    finally:
        dist.destroy_process_group()


def _repair_inputs(dims, seed):
    n0, n1, n2 = dims
    H = n2 // 2 + 1
    rng = np.random.default_rng(seed)
    shp = (n0, n1, H)
    cplx = lambda: rng.standard_normal(shp) + 1j * rng.standard_normal(shp)  # noqa: E731
    cur, ds, dt = cplx(), cplx(), cplx()
    viol = rng.random(shp) < 0.05
    k2 = np.arange(H)
    plane = (k2 == 0) | (2 * k2 == n2)
    viol[:, :, plane] |= rng.random((n0, n1, int(plane.sum()))) < 0.4   # many plane pairs
    return cur, ds, dt, viol


@pytest.mark.parametrize("world", [1, 2, 4])
def test_cross_rank_plane_repair(world):
    dims = (8, 8, 8)
    cur, ds, dt, viol = _repair_inputs(dims, 11)
    want, want_h = _repair_reference(cur, ds, dt, viol, dims)
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_repair_worker, args=(world, _free_port(), dims, 11, tmp), nprocs=world,
                 join=True)
        parts = [pickle.load(open(os.path.join(tmp, f"r{r}.pkl"), "rb")) for r in range(world)]
    got = np.concatenate([p[0] for p in parts], axis=1)
    assert np.array_equal(got, want)
    assert sorted(np.concatenate([p[1] for p in parts]).tolist()) == want_h
