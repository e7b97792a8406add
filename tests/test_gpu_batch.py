"""Batched frames (BASELINE config 3): ffcz_cuda_correct_batch must give, for every frame, exactly
what an independent ffcz::correct() of that frame gives (pipeline.cpp:26-178) — the reference has
no batch API; a batch is a loop of correct() calls.  Checked against per-frame correct() on the
engine (bit-identical products) and against the numpy oracle / the reference's golden outputs."""
import json
import os

import numpy as np
import pytest

import cases
from oracle import ffcz_oracle as O

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(cases.GOLDEN, "golden.json")))


@pytest.fixture(scope="module")
def ffcz():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2601_01596_b200 as P
    return P


def frames(n, count, seed0=100, spots=20):
    """config-3 recipe per frame: own E (0.1% of the frame range) and Delta = 0.8 mean|delta0|."""
    os_, ds, bs = [], [], []
    for f in range(count):
        o = cases.xrd_frame(n, seed0 + f, spots=spots)
        E = 0.1 / 100.0 * cases.value_range(o)
        d = cases.uniform_perturb(o, E, 7 + f)
        os_.append(o)
        ds.append(d)
        bs.append((E, 0.8 * cases.mean_abs_delta0(o, d)))
    return np.stack(os_), np.stack(ds), bs


def same_result(a, b):
    assert a.report == b.report or (
        a.report.iterations == b.report.iterations and a.report.converged == b.report.converged
        and a.report.active_spatial == b.report.active_spatial
        and a.report.active_frequency == b.report.active_frequency)
    assert a.verify_ok == b.verify_ok and a.escape_count == b.escape_count
    assert np.array_equal(a.spatial_flags, b.spatial_flags)
    assert np.array_equal(a.frequency_flags, b.frequency_flags)
    assert np.array_equal(a.spatial_codes, b.spatial_codes)
    assert np.array_equal(a.frequency_codes, b.frequency_codes)
    assert np.array_equal(a.escapes, b.escapes)
    assert np.array_equal(a.corrected, b.corrected)
    assert a.archive_bytes == b.archive_bytes


@pytest.mark.parametrize("lanes", [1, 3, 8])
def test_batch_equals_per_frame_correct(ffcz, lanes):
    o, d, bs = frames(128, 7)
    o32, d32 = o.astype(np.float32), d.astype(np.float32)
    bounds = [ffcz.DualBounds(E, D) for E, D in bs]
    rb = ffcz.correct_batch(o32, d32, bounds, 16, 1000, "f32", lanes=lanes)
    assert len(rb) == 7
    for i in range(7):
        ri = ffcz.correct(o32[i], d32[i], bounds[i], 16, 1000, "f32")
        same_result(rb[i], ri)
        assert rb[i].report.converged and rb[i].verify_ok


def test_batch_against_oracle(ffcz):
    o, d, bs = frames(64, 3, seed0=300, spots=8)
    rb = ffcz.correct_batch(o.astype(np.float32), d.astype(np.float32),
                            [ffcz.DualBounds(E, D) for E, D in bs], 16, 1000, "f32", lanes=2)
    for i in range(3):
        ref = O.correct(o[i], d[i], O.DualBounds(*bs[i]), 16, 1000, "f32")
        r = rb[i]
        assert r.report.iterations == ref.report.iterations
        assert r.report.converged == ref.report.converged
        assert r.report.active_spatial == ref.report.active_spatial
        assert r.report.active_frequency == ref.report.active_frequency
        mine, theirs = O.read_archive(r.archive_bytes), O.read_archive(ref.archive_bytes)
        assert np.array_equal(mine.spatial_flags, theirs.spatial_flags)
        assert np.array_equal(mine.frequency_flags, theirs.frequency_flags)
        assert np.mean(mine.frequency_codes == theirs.frequency_codes) >= 0.999


def test_batch_golden_frame(ffcz):
    case = {c.name: c for c in cases.all_cases()}["config3_frame256"]
    g = GOLD[case.name]
    o = np.stack([case.original, case.original]).astype(np.float32)
    d = np.stack([case.decompressed, case.decompressed]).astype(np.float32)
    rb = ffcz.correct_batch(o, d, ffcz.DualBounds(case.E, case.Dre), case.m, case.max_iters,
                            case.precision, lanes=2)
    for r in rb:
        assert r.report.iterations == g["iterations"]
        assert r.report.active_spatial == g["active_spatial"]
        assert r.report.active_frequency == g["active_frequency"]
        assert r.verify_ok == g["verify_ok"]
    same_result(rb[0], rb[1])


def test_batch_device_inputs(ffcz):
    import torch
    o, d, bs = frames(128, 4, seed0=500)
    to = torch.from_numpy(o.astype(np.float32)).cuda()
    td = torch.from_numpy(d.astype(np.float32)).cuda()
    bounds = [ffcz.DualBounds(E, D) for E, D in bs]
    rd = ffcz.correct_batch(to, td, bounds, 16, 1000, "f32", lanes=4)
    rh = ffcz.correct_batch(o.astype(np.float32), d.astype(np.float32), bounds, 16, 1000, "f32",
                            lanes=4)
    for a, b in zip(rd, rh):
        same_result(a, b)


def test_batch_error_is_reported(ffcz):
    o, d, bs = frames(64, 3, seed0=700, spots=4)
    bounds = [ffcz.DualBounds(E, D) for E, D in bs]
    bounds[1] = ffcz.DualBounds(1e-12, bs[1][1])  # precondition violated on frame 1
    with pytest.raises(ffcz.ValidationError):
        ffcz.correct_batch(o, d, bounds, 16, 1000, "f32", lanes=2)


def test_batch_lanes_path_per_point_bounds(ffcz):
    """Per-point E sends the batch down the per-frame lanes path; still equal to correct()."""
    o, d, bs = frames(64, 3, seed0=900, spots=6)
    bounds = []
    for i, (E, D) in enumerate(bs):
        e = np.full(o[i].shape, E)
        e[::7, ::5] *= 1.5
        bounds.append(ffcz.DualBounds(e, D))
    rb = ffcz.correct_batch(o.astype(np.float32), d.astype(np.float32), bounds, 16, 1000, "f32",
                            lanes=2)
    for i in range(3):
        ri = ffcz.correct(o[i].astype(np.float32), d[i].astype(np.float32), bounds[i], 16, 1000,
                          "f32")
        same_result(rb[i], ri)


def test_batch_mixed_policy_runs_per_frame(ffcz):
    o, d, bs = frames(64, 2, seed0=950, spots=6)
    bounds = [ffcz.DualBounds(E, D) for E, D in bs]
    rb = ffcz.correct_batch(o.astype(np.float32), d.astype(np.float32), bounds, 16, 1000, "f32",
                            lanes=2, policy="mixed")
    for i in range(2):
        ri = ffcz.correct(o[i].astype(np.float32), d[i].astype(np.float32), bounds[i], 16, 1000,
                          "f32", policy="mixed")
        same_result(rb[i], ri)
        assert rb[i].verify_ok
