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
    out.append(overflow_case())
    return out


def mirror_flat(shape):
    """Flat index of the conjugate partner (-k mod n per axis) of every flat index
    (field.cpp:41-50 mirror_index), row-major."""
    idx = np.indices(shape).reshape(len(shape), -1)
    m = np.zeros(idx.shape[1], dtype=np.int64)
    for a, n in enumerate(shape):
        m = m * n + (-idx[a]) % n
    return m


def overflow_case():
    """Quantiser overflow escapes (pipeline.cpp:54-88): m = 24 and a per-component Delta that is
    tiny (1e-3 of the typical |delta0|) on the 8 largest-|delta0| components and their mirrors, so
    their frequency edits exceed 2147483520 quantisation steps and go to the escape list."""
    shape = (16, 16, 16)
    o = noise(shape, 9090, "f64")
    E = 0.1 / 100.0 * value_range(o)
    d = uniform_perturb(o, E, 9091, precision="f64")
    d0 = np.abs(np.fft.fftn(d - o)).ravel()
    typ = float(np.mean(d0))
    D = np.full(d0.size, 0.7 * typ)
    mir = mirror_flat(shape)
    top = np.argsort(d0)[::-1][1:9]       # skip the DC term
    D[top] = 1e-3 * typ
    D[mir[top]] = 1e-3 * typ
    return Case("overflow_m24", o, d, E, D.reshape(shape), m=24, tags=["overflow", "per_component"])


def all_cases():
    inputs = load_inputs()
    return acceptance_cases() + config1_cases(inputs) + config2_cases(inputs) + misc_cases()


def hand_trace():
    """test_projection.cpp:48-59 / acceptance.cpp:130-146: eps0 = [1, 1], E = Delta = 1."""
    return np.array([1.0, 1.0]), 1.0, 1.0


# ---- digests of an edit set (flags / int32 codes / escapes) -------------------------------------

BLOCK = 1 << 16   # codes per block hash (65,536 = the reference's Huffman block, huffman.hpp:13)


def _sha(b) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(b).tobytes() if isinstance(b, np.ndarray)
                          else bytes(b)).hexdigest()


def _blocks(codes: np.ndarray) -> list:
    import hashlib
    c = np.ascontiguousarray(codes, dtype="<i4")
    return [hashlib.sha256(c[i:i + BLOCK].tobytes()).hexdigest()[:12]
            for i in range(0, c.size, BLOCK)]


def edit_digest(sflags, fflags, scodes, fcodes, esc_index, esc_freq) -> dict:
    """Size-independent fingerprint of an edit set as the archive carries it (flag bytes
    LSB-first, int32 codes in flag order, frequency codes interleaved Re/Im, escape keys in the
    reference's std::map order).  Codes also get one hash per 65,536-code block so a mismatch is
    localised and counted."""
    sflags = np.frombuffer(bytes(sflags), np.uint8) if not isinstance(sflags, np.ndarray) else sflags
    fflags = np.frombuffer(bytes(fflags), np.uint8) if not isinstance(fflags, np.ndarray) else fflags
    esc = np.stack([np.asarray(esc_freq, np.uint64), np.asarray(esc_index, np.uint64)], axis=1) \
        if len(esc_index) else np.zeros((0, 2), np.uint64)
    return {"flags_s": _sha(sflags.astype(np.uint8)), "flags_f": _sha(fflags.astype(np.uint8)),
            "popcount_s": int(np.unpackbits(sflags.astype(np.uint8)).sum()),
            "popcount_f": int(np.unpackbits(fflags.astype(np.uint8)).sum()),
            "codes_s": _sha(np.asarray(scodes, "<i4")), "codes_f": _sha(np.asarray(fcodes, "<i4")),
            "blocks_s": _blocks(scodes), "blocks_f": _blocks(fcodes),
            "n_escapes": int(esc.shape[0]),
            "escapes": esc.tolist() if esc.shape[0] <= 4096 else _sha(esc)}


def digest_of_result(r) -> dict:
    """edit_digest of a CorrectionResult of the GPU engine (want_edits=True)."""
    e = r.escapes
    return edit_digest(r.spatial_flags, r.frequency_flags, r.spatial_codes, r.frequency_codes,
                       e["index"] if len(e) else [], e["frequency"] if len(e) else [])


def compare_digest(mine: dict, ref: dict) -> dict:
    """{flags equal, code blocks that differ (s, f), escape keys equal} of two digests."""
    bs = sum(a != b for a, b in zip(mine["blocks_s"], ref["blocks_s"])) + \
        abs(len(mine["blocks_s"]) - len(ref["blocks_s"]))
    bf = sum(a != b for a, b in zip(mine["blocks_f"], ref["blocks_f"])) + \
        abs(len(mine["blocks_f"]) - len(ref["blocks_f"]))
    return {"flags": mine["flags_s"] == ref["flags_s"] and mine["flags_f"] == ref["flags_f"],
            "code_blocks_s": int(bs), "code_blocks_f": int(bf),
            "escapes": mine["escapes"] == ref["escapes"],
            "n_escapes": (mine["n_escapes"], ref["n_escapes"])}


def freq_excess_per_component(original, corrected, Dre, Dim=None):
    """max over components of (|Re d_k| - Dre_k, |Im d_k| - Dim_k) / D_k with d = FFT(corrected -
    original) in numpy FP64; <= 0 means every component holds exactly."""
    d = np.fft.fftn(np.asarray(corrected, np.float64) - np.asarray(original, np.float64))
    Dr = np.broadcast_to(np.asarray(Dre, np.float64), d.shape)
    Di = Dr if Dim is None else np.broadcast_to(np.asarray(Dim, np.float64), d.shape)
    return float(max(np.max((np.abs(d.real) - Dr) / Dr), np.max((np.abs(d.imag) - Di) / Di)))


# ---- BASELINE-size parity cases (reference outputs in golden/golden_big.json) ----


def xrd_frame_windowed(n, seed, spots=400):
    """Config 3 frame recipe at full size: background 2*U[0,1) plus `spots` Gaussian spots
    (sigma^2 = 2 px^2, amplitude 50 + 1000 U, uniform positions), each evaluated on its 15x15
    window (the spot is < 1e-10 of its amplitude outside it)."""
    rng = np.random.default_rng(seed)
    img = 2.0 * rng.random((n, n))
    w = np.arange(-7, 8)
    for _ in range(spots):
        a = 50.0 + 1000.0 * rng.random()
        cy, cx = rng.random() * n, rng.random() * n
        iy = int(np.floor(cy)) + w
        ix = int(np.floor(cx)) + w
        iy, ix = iy[(iy >= 0) & (iy < n)], ix[(ix >= 0) & (ix < n)]
        img[np.ix_(iy, ix)] += a * np.exp(-((iy[:, None] - cy) ** 2 + (ix[None, :] - cx) ** 2) / 4.0)
    return img.astype(np.float32).astype(np.float64)


def nyx_workload(n, seed):
    """Config 2 recipe (bench.make_workload_numpy): log-normal of a power-law GRF (alpha = 2.5),
    E = 0.1% of the range, +-0.99E uniform base error, rho = 1e-3 per-component Delta derived in
    numpy from FFT(original) (Hermitian-consistent by construction: min(|X_k|, |X_-k|))."""
    import bench
    return bench.make_workload_numpy(n, seed)


BIG_CASES = ("config2_nyx256", "config2_nyx512", "config3_xrd2048", "config4_comb256")


def big_case(name: str) -> Case:
    if name.startswith("config2_nyx"):
        n = int(name[len("config2_nyx"):])
        o, d, E, D = nyx_workload(n, 2601 + n)
        return Case(name, o, d, E, D, precision="f32", tags=["config2", "per_component", "big"])
    if name == "config3_xrd2048":
        o = xrd_frame_windowed(2048, 5)
        E = 0.1 / 100.0 * value_range(o)
        d = uniform_perturb(o, E, 205)
        return Case(name, o, d, E, 0.8 * mean_abs_delta0(o, d), precision="f32",
                    tags=["config3", "big"])
    if name == "config4_comb256":
        o = combustion(256, 19)
        E = 0.1 / 100.0 * value_range(o)
        d = uniform_perturb(o, E, 219)
        return Case(name, o, d, E, 0.6 * mean_abs_delta0(o, d), precision="f32",
                    tags=["config4", "big"])
    raise KeyError(name)


def input_digest(c: Case) -> dict:
    out = {"orig": _sha(np.asarray(c.original, np.float32)),
           "dec": _sha(np.asarray(c.decompressed, np.float32)), "E": float(c.E)}
    out["delta"] = _sha(np.asarray(c.Dre, np.float64)) if isinstance(c.Dre, np.ndarray) \
        else float(c.Dre)
    return out
