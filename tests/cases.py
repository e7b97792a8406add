"""Seeded parity cases shared by the golden-vector generator and the GPU parity tests.

Inputs are either regenerated from numpy's PCG64 (identical on every box) or, where the recipe
needs the reference's own synth_field (mt19937_64 + random-phase spectra,
/root/reference/proj/core/src/synth.cpp:29-50), stored in tests/golden/inputs.npz by
tests/golden/make_golden.py.  Recipes follow SURVEY.md §8d / BASELINE.json configs, shrunk to
sizes the CPU reference finishes in seconds.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@dataclass
class Case:
    name: str
    original: np.ndarray          # float64 values (f32-representable when precision == "f32")
    decompressed: np.ndarray
    E: float | np.ndarray
    Dre: float | np.ndarray
    Dim: float | np.ndarray | None = None
    m: int = 16
    max_iters: int = 1000
    precision: str = "f64"
    tags: list = field(default_factory=list)


def noise(shape, seed, precision="f64"):
    """acceptance.cpp:33-42 recipe (uniform [-1, 1), f32 rounded) on numpy's PCG64."""
    v = np.random.default_rng(seed).uniform(-1.0, 1.0, size=shape)
    if precision == "f32":
        v = v.astype(np.float32).astype(np.float64)
    return v


def quantize_base(x, E):
    """uniform_quantize_compress (baseline.cpp:14-32): round(x / 2E) * 2E, half away from zero."""
    step = 2.0 * E
    q = x / step
    t = np.trunc(q)
    c = np.where(np.abs(q - t) >= 0.5, t + np.sign(q), t)
    return c * step


def value_range(x):
    return float(x.max() - x.min())


def peak_abs_spectrum(x):
    return float(np.max(np.abs(np.fft.fftn(x))))


def acceptance_cases():
    """acceptance.cpp:61-102 (criterion 1) on a subset of its shape pool."""
    pool = [(17,), (64,), (1000,), (32, 32), (64, 48), (128, 128), (8, 8, 8), (16, 16, 16),
            (32, 32, 32), (64, 64, 64)]
    pct = [1e-1, 1e-2, 1e-3]
    out = []
    for c in range(0, 30, 1):
        shape = pool[c % len(pool)]
        prec = "f64" if (c // 10) % 2 else "f32"
        o = noise(shape, 5000 + c, prec)
        E = 0.1 / 100.0 * value_range(o)
        D = pct[c % 3] / 100.0 * peak_abs_spectrum(o)
        d = quantize_base(o, E)
        out.append(Case(f"accept_{c:02d}", o, d, E, D, precision=prec, tags=["acceptance"]))
    return out


def uniform_perturb(o, E, seed, frac=0.99, precision="f32"):
    u = np.random.default_rng(seed).uniform(-frac * E, frac * E, size=o.shape)
    d = o + u
    if precision == "f32":
        d = d.astype(np.float32).astype(np.float64)
    return d


def mean_abs_delta0(o, d):
    return float(np.mean(np.abs(np.fft.fftn(d - o))))


def load_inputs():
    path = os.path.join(GOLDEN, "inputs.npz")
    return dict(np.load(path)) if os.path.exists(path) else {}


def config1_cases(inputs=None):
    """Config 1: 64^3 FP32 power-law (alpha=3), uniform +-0.99E perturbation, global Delta =
    c * mean|delta0|, c in {2.0, 1.0, 0.6, 0.4}."""
    inputs = inputs if inputs is not None else load_inputs()
    if "c1_orig" not in inputs:
        return []
    o = inputs["c1_orig"].astype(np.float64)
    E = 0.1 / 100.0 * value_range(o)
    d = uniform_perturb(o, E, 7)
    typ = mean_abs_delta0(o, d)
    return [Case(f"config1_c{c}", o, d, E, c * typ, precision="f32", tags=["config1"])
            for c in (2.0, 1.0, 0.6, 0.4)]


def config2_cases(inputs=None):
    """Config 2 recipe at 32^3: log-normal Nyx-like field, rho = 1e-3 per-component Delta."""
    inputs = inputs if inputs is not None else load_inputs()
    if "c2_orig" not in inputs:
        return []
    o = inputs["c2_orig"].astype(np.float64)
    E = 0.1 / 100.0 * value_range(o)
    d = uniform_perturb(o, E, 8)
    return [Case("config2_rho32", o, d, E, inputs["c2_delta"], precision="f32",
                 tags=["config2", "per_component"])]


def xrd_frame(n, seed, spots=60):
    """Config 3 recipe: background 2*U[0,1) plus Gaussian spots."""
    rng = np.random.default_rng(seed)
    img = 2.0 * rng.random((n, n))
    yy, xx = np.mgrid[0:n, 0:n]
    for _ in range(spots):
        a = 50.0 + 1000.0 * rng.random()
        cy, cx = rng.random() * n, rng.random() * n
        img += a * np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * 2.0))
    return img.astype(np.float32).astype(np.float64)


def combustion(n, seed):
    """Config 4 recipe, small: tanh flame front with a wrinkled interface plus turbulence."""
    rng = np.random.default_rng(seed)
    z = np.arange(n)[:, None, None]

    def grf(shape, alpha):
        k = np.sqrt(sum(np.meshgrid(*[np.fft.fftfreq(s) * s for s in shape], indexing="ij")[i] ** 2
                        for i in range(len(shape))))
        k[(0,) * len(shape)] = 1.0
        amp = k ** (-alpha / 2.0)
        ph = np.exp(2j * np.pi * rng.random(shape))
        f = np.fft.ifftn(amp * ph).real
        return f / f.std()

    h = grf((n, n), 3.0)[None, :, :]
    g = grf((n, n, n), 11.0 / 3.0)
    c = 0.05 * (1.0 + np.tanh((z - n / 2 - 0.08 * n * h) / (n / 128.0 * 8))) + 0.002 * g
    return c.astype(np.float32).astype(np.float64)


def misc_cases():
    out = []
    # config 3 shape, small frame
    o = xrd_frame(256, 5)
    E = 0.1 / 100.0 * value_range(o)
    d = uniform_perturb(o, E, 105)
    out.append(Case("config3_frame256", o, d, E, 0.8 * mean_abs_delta0(o, d), precision="f32",
                    tags=["config3"]))
    # config 4 recipe at 32^3
    o = combustion(32, 9)
    E = 0.1 / 100.0 * value_range(o)
    d = uniform_perturb(o, E, 109)
    out.append(Case("config4_comb32", o, d, E, 0.6 * mean_abs_delta0(o, d), precision="f32",
                    tags=["config4"]))
    # iteration cap (acceptance.cpp:306-347): error pinned to the cube faces, cap 1 and 3
    o = noise((64,), 8080, "f64")
    E = 0.1 / 100.0 * value_range(o)
    rng = np.random.default_rng(8081)
    d = o + np.where(rng.random(64) < 0.5, E, -E)
    typ = mean_abs_delta0(o, d)
    for cap in (1, 3):
        out.append(Case(f"capped_{cap}", o, d, E, 0.6 * typ, max_iters=cap, tags=["capped"]))
    out.append(Case("capped_full", o, d, E, 0.6 * typ, tags=["capped"]))
    # per-point spatial bound
    o = noise((32, 48), 77, "f64")
    Epp = 0.001 * (1.0 + np.random.default_rng(78).random((32, 48)))
    d = o + np.random.default_rng(79).uniform(-0.99, 0.99, (32, 48)) * Epp
    out.append(Case("per_point_2d", o, d, Epp, 0.7 * mean_abs_delta0(o, d), tags=["per_point"]))
    # coarse quantizer m = 8 (acceptance.cpp:276-302)
    o = noise((32, 32, 32), 7003, "f64")
    E = 0.1 / 100.0 * value_range(o)
    out.append(Case("m8_32cube", o, quantize_base(o, E), E, 0.1 / 100.0 * peak_abs_spectrum(o),
                    m=8, tags=["m8"]))
    # already feasible: no edits
    o = noise((16, 16), 5, "f64")
    d = o + 0.001 * noise((16, 16), 6, "f64")
    out.append(Case("feasible_2d", o, d, 0.01, 1.0, tags=["feasible"]))
    # odd last axis + non power of two axes through the direct passes
    o = noise((12, 10, 9), 31, "f64")
    E = 0.05
    d = uniform_perturb(o, E, 32, precision="f64")
    out.append(Case("odd_12x10x9", o, d, E, 0.7 * mean_abs_delta0(o, d), tags=["odd"]))
    rng = np.random.default_rng(33)
    d = o + np.where(rng.random(o.shape) < 0.5, E, -E)
    out.append(Case("odd_faces_12x10x9", o, d, E, 0.6 * mean_abs_delta0(o, d), tags=["odd"]))
    o = noise((24, 40), 34, "f64")
    d = o + np.where(np.random.default_rng(35).random(o.shape) < 0.5, E, -E)
    out.append(Case("odd_faces_24x40", o, d, E, 0.6 * mean_abs_delta0(o, d), tags=["odd"]))
    return out


def all_cases():
    inputs = load_inputs()
    return acceptance_cases() + config1_cases(inputs) + config2_cases(inputs) + misc_cases()


def hand_trace():
    """test_projection.cpp:48-59 / acceptance.cpp:130-146: eps0 = [1, 1], E = Delta = 1."""
    return np.array([1.0, 1.0]), 1.0, 1.0
