"""Argument validation of the Python mirror (ffcz.correct), before any device work — so these run
on CPU.  The reference raises validation_error for each (bounds.cpp:65-71 validate_for,
projection.cpp:20-22 compute_error); a short bound array would otherwise make the engine read
past the caller's buffer."""
import numpy as np
import pytest

import paper_2601_01596_b200 as P


def _fields(shape=(8, 8), dtype=np.float64):
    o = np.zeros(shape, dtype=dtype)
    return o, o.copy()


def test_per_point_bound_length():
    o, d = _fields()
    with pytest.raises(P.ValidationError, match="per-point spatial bound length"):
        P.correct(o, d, P.DualBounds(np.ones(63), 1.0))


def test_per_component_bound_length():
    o, d = _fields()
    with pytest.raises(P.ValidationError, match="per-component frequency bound length"):
        P.correct(o, d, P.DualBounds(1.0, np.ones(10)))
    with pytest.raises(P.ValidationError, match="per-component frequency bound length"):
        P.correct(o, d, P.DualBounds(1.0, np.ones(64), np.ones(65)))


def test_per_component_needs_both_lanes_as_arrays():
    o, d = _fields()
    with pytest.raises(P.ValidationError, match="both Re and Im"):
        P.correct(o, d, P.DualBounds(1.0, np.ones(64), 2.0))


def test_dims_and_dtype_mismatch():
    o, _ = _fields()
    with pytest.raises(P.ValidationError, match="dims/precision mismatch"):
        P.correct(o, np.zeros((8, 9)), P.DualBounds(1.0, 1.0))
    with pytest.raises(P.ValidationError, match="dims/precision mismatch"):
        P.correct(o, np.zeros((8, 8), np.float32), P.DualBounds(1.0, 1.0))


def test_empty_and_4d_fields():
    with pytest.raises(P.ValidationError):
        P.correct(np.zeros((0, 4)), np.zeros((0, 4)), P.DualBounds(1.0, 1.0))
    with pytest.raises(P.ValidationError):
        P.correct(np.zeros((2, 2, 2, 2)), np.zeros((2, 2, 2, 2)), P.DualBounds(1.0, 1.0))


def test_torch_bound_dtype_and_location():
    torch = pytest.importorskip("torch")
    o, d = _fields()
    # a float32 bound tensor is never reinterpreted as float64
    with pytest.raises(P.ValidationError, match="float64"):
        P.correct(o, d, P.DualBounds(torch.ones(64, dtype=torch.float32), 1.0))
    # host fields with host torch bounds of the right dtype pass the checks (they are numpy-viewed)
    m = P.ffcz._Marshal()
    bd = P.ffcz._bounds_desc(P.DualBounds(torch.ones(64, dtype=torch.float64), 1.0), m, (8, 8), False)
    assert bd.spatial_per_point == 1


def test_unknown_options():
    o, d = _fields()
    with pytest.raises(P.ValidationError, match="repair order"):
        P.correct(o, d, P.DualBounds(1.0, 1.0), repair_order="fast")
    with pytest.raises(P.ValidationError, match="F update"):
        P.correct(o, d, P.DualBounds(1.0, 1.0), f_update="none")
