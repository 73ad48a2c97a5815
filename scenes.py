"""Seeded synthetic inputs for the BASELINE.json configs.

The reference measures on no public dataset; these generators stand in for the
paper's images.  Every array is produced from ``numpy.random.default_rng(seed)``
so the oracle, the reference and the CUDA path consume identical inputs.
Images are float32 (the reference promotes them to float64 on entry,
optimizer.py:102); label images are int32.

Decisions recorded in DESIGN.md: "kernel width w" maps to length scale E = 2w
(strict cutoff d < w); Gaussian-noised configs use the gauss noise model,
Poisson-noised configs the poisson model; bubble initialisations use
vanish_grace = 5 (the reference CLI's rule for seeded inits, cli.py:93-96).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np
from scipy import ndimage


@dataclass
class Scene:
    name: str
    image: np.ndarray           # float32
    labels: np.ndarray          # int32 initial labels
    region: str                 # "pc" | "ps"
    noise: str                  # "gauss" | "poisson"
    length_scale: float         # E = 2w
    smooth_radius: int = 8
    lam: float = 0.0
    iterations: int = 50
    vanish_grace: int = 0
    extra: dict = field(default_factory=dict)


def _ellipse(shape, centre, semi):
    """Boolean mask of the axis-aligned ellipsoid sum(((x_k - c_k)/a_k)^2) <= 1."""
    m = np.zeros(shape, bool)
    _paint(m, centre, semi, True)
    return m


def _paint(arr, centre, semi, value):
    """Set arr to value inside the ellipsoid, touching only its bounding box."""
    lo = [max(0, int(np.floor(c - a))) for c, a in zip(centre, semi)]
    hi = [min(n, int(np.ceil(c + a)) + 1) for c, a, n in zip(centre, semi, arr.shape)]
    if any(h <= l for l, h in zip(lo, hi)):
        return
    g = np.ogrid[tuple(slice(l, h) for l, h in zip(lo, hi))]
    acc = 0.0
    for gi, c, a in zip(g, centre, semi):
        acc = acc + ((gi - c) / a) ** 2
    sub = arr[tuple(slice(l, h) for l, h in zip(lo, hi))]
    sub[acc <= 1.0] = value


def bubbles(shape, per_axis: int, radius: float) -> np.ndarray:
    """n-per-axis lattice of balls labelled 1.. in row-major lattice order
    (the reference's ``bubbles:<n>:<r>`` initialisation, optimizer.py:325-335)."""
    labels = np.zeros(shape, np.int32)
    centres = [[(i + 0.5) * d / per_axis for i in range(per_axis)] for d in shape]
    for lab, c in enumerate(itertools.product(*centres), start=1):
        _paint(labels, c, [radius] * len(shape), lab)
    return labels


# -- blur / Poisson noise: the reference pipeline (rcseg/synth.py:87-182) ------
#
# Every generator below blurs and noises exactly as the reference's
# ``blur`` / ``poissonize`` do.  By default the device
# pipeline of this package computes them (bit-identical to the reference,
# tests/golden/synth.npz); the fixture script (tests/golden/make_golden.py)
# swaps in the reference's own functions with ``use_backend``, and a GPU
# test checks the device-made images equal the fixture images bit for bit.

_BACKEND: dict = {"blur": None, "poissonize": None}


def use_backend(blur=None, poissonize=None) -> None:
    """Route blur(image, sigma) / poissonize(image, psnr, seed) through the
    given callables (None restores the device pipeline)."""
    _BACKEND["blur"] = blur
    _BACKEND["poissonize"] = poissonize


def _ref_kernel(sigma: float) -> np.ndarray:
    """synth.py:96-99: exp(-t^2 / (2 sigma^2)) over |t| <= ceil(4 sigma), / sum."""
    radius = int(np.ceil(4.0 * sigma))
    t = np.arange(-radius, radius + 1, dtype=np.float64)
    k = np.exp(-(t * t) / (2.0 * sigma * sigma))
    k /= k.sum()
    return k


def _device_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


def _blur(img, sigma):
    """Reference blur; ``sigma`` may be a per-axis tuple (cfg3's anisotropic
    PSF: the reference's correlate1d pass per axis with that axis' kernel)."""
    img = np.asarray(img, np.float64)
    sig = tuple(sigma) if np.ndim(sigma) else (float(sigma),) * img.ndim
    if _BACKEND["blur"] is not None and len(set(sig)) == 1:
        return _BACKEND["blur"](img, sig[0])
    if len(set(sig)) == 1 and _device_ok():
        from paper_1403_0240_b200 import synth as dsynth
        return dsynth.blur(img, sig[0])
    out = img.copy()
    for axis, s in enumerate(sig):
        if s > 0:
            out = ndimage.correlate1d(out, _ref_kernel(s), axis=axis, mode="mirror")
    return out


def _poisson(img, peak, seed):
    """Reference poissonize(img, NoiseSpec(psnr=sqrt(peak), seed)): the blurred
    image rescaled to peak mean psnr**2, per-pixel counter-based draws."""
    psnr = float(np.sqrt(peak))
    if _BACKEND["poissonize"] is not None:
        out = _BACKEND["poissonize"](img, psnr, seed)
    else:
        from paper_1403_0240_b200 import synth as dsynth
        out = dsynth.poissonize(img, dsynth.NoiseSpec(psnr, seed))
    return np.asarray(out).astype(np.float32)


def cfg1(seed: int = 0) -> Scene:
    shape = (256, 256)
    img = np.zeros(shape)
    img[_ellipse(shape, (80, 80), (40, 25))] = 1.0
    img[_ellipse(shape, (170, 170), (30, 30))] = 1.0
    img += np.random.default_rng(seed).normal(0.0, 0.3, size=shape)
    lab = np.zeros(shape, np.int32)
    lab[28:228, 28:228] = 1
    return Scene("cfg1", img.astype(np.float32), lab, "pc", "gauss", 4.0, iterations=50)


def _cfg2_image(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    shape = (n, n)
    img = np.tile(np.linspace(0.2, 0.5, n), (n, 1))
    for _ in range(16):
        c = rng.uniform(0, n, size=2)
        a = rng.uniform(15, 60, size=2)
        val = rng.uniform(0.6, 1.0)
        _paint(img, c, a, val)
    img = _blur(img, 1.5)
    return _poisson(img, 50.0, seed)


def cfg2(seed: int = 2) -> Scene:
    img = _cfg2_image(1024, seed)
    lab = bubbles(img.shape, 16, 10.0)
    return Scene("cfg2", img, lab, "ps", "poisson", 6.0, smooth_radius=4,
                 iterations=100, vanish_grace=5)


def cfg2_small(seed: int = 2, n: int = 256) -> Scene:
    """Oracle-sized cfg2: a crop of the 1024^2 image with bubbles:4:10."""
    img = _cfg2_image(1024, seed)[:n, :n].copy()
    lab = bubbles(img.shape, n // 64, 10.0)
    return Scene("cfg2_small", img, lab, "ps", "poisson", 6.0, smooth_radius=4,
                 iterations=100, vanish_grace=5)


def cfg3(seed: int = 3, n: int = 128) -> Scene:
    rng = np.random.default_rng(seed)
    shape = (n, n, n)
    img = np.full(shape, 0.1)
    for _ in range(8):
        r = rng.uniform(10, 25) * n / 128
        c = rng.uniform(r, n - r, size=3)
        _paint(img, c, (r, r, r), 1.0)
    img = _blur(img, (2.0, 1.0, 1.0))
    img += rng.normal(0.0, 0.25, size=shape)
    lab = np.zeros(shape, np.int32)
    m = int(round(14 * n / 128))
    lab[m:n - m, m:n - m, m:n - m] = 1
    return Scene("cfg3", img.astype(np.float32), lab, "pc", "gauss", 4.0, iterations=100)


def cfg4(seed: int = 4, n: int = 512, n_obj: int = 64, per_axis: int = 8,
         radius: float | None = None) -> Scene:
    rng = np.random.default_rng(seed)
    shape = (n, n, n)
    z = np.arange(n, dtype=np.float64)[:, None, None]
    img = np.broadcast_to(0.2 + 0.1 * z / (n - 1), shape).copy()
    for _ in range(n_obj):
        c = rng.uniform(0, n, size=3)
        a = rng.uniform(10, 50, size=3) * n / 512
        val = rng.uniform(0.5, 1.0)
        _paint(img, c, a, val)
    img = _blur(img, 1.5)
    img = _poisson(img, 30.0, seed)
    if radius is None:
        radius = 15.0 * n / 512 if n < 512 else 15.0
    lab = bubbles(shape, per_axis, radius)
    return Scene("cfg4", img, lab, "ps", "poisson", 6.0, smooth_radius=4,
                 iterations=200, vanish_grace=5)


def cfg4_small(seed: int = 4) -> Scene:
    """cfg4': 128^3, 8 ellipsoids, bubbles:2:15, PS/Poisson R=4, E=6."""
    s = cfg4(seed, n=128, n_obj=8, per_axis=2, radius=15.0)
    s.name = "cfg4_small"
    return s


def cfg4_sample(seed: int = 4, n: int = 64) -> Scene:
    """The bounded CPU sample of cfg4 that the reference arm and the CPU
    baseline time (bench.py): the cfg4 generator at 64^3 -- smooth
    background, 4 ellipsoids (semi-axes scaled by n/512), blur 1.5, Poisson
    peak 30 -- with one seed sphere of cfg4's radius 15 (bubbles:1:15);
    PS/Poisson R = 4, E = 6 like cfg4."""
    s = cfg4(seed, n=n, n_obj=4, per_axis=1, radius=15.0)
    s.name = "cfg4_sample"
    return s


def cfg5_image(i: int, n: int = 512) -> Scene:
    rng = np.random.default_rng(1000 + i)
    shape = (n, n)
    img = np.zeros(shape)
    for _ in range(int(rng.integers(4, 13))):
        c = rng.uniform(0, n, size=2)
        a = rng.uniform(15, 60, size=2)
        _paint(img, c, a, 1.0)
    img += rng.normal(0.0, 0.3, size=shape)
    lab = np.zeros(shape, np.int32)
    m = int(round(56 * n / 512))
    lab[m:n - m, m:n - m] = 1
    return Scene(f"cfg5[{i}]", img.astype(np.float32), lab, "pc", "gauss", 4.0, iterations=50)


def two_region_small(shape=(48, 48), seed: int = 0) -> Scene:
    """A small cfg1 analogue used by the parity tests."""
    rng = np.random.default_rng(seed)
    img = np.zeros(shape)
    h, w = shape
    img[_ellipse(shape, (h * 0.3, w * 0.3), (h * 0.16, w * 0.1))] = 1.0
    img[_ellipse(shape, (h * 0.66, w * 0.66), (h * 0.12, w * 0.12))] = 1.0
    img += rng.normal(0.0, 0.3, size=shape)
    lab = np.zeros(shape, np.int32)
    m = max(1, h // 9)
    lab[m:h - m, m:w - m] = 1
    return Scene("two_region_small", img.astype(np.float32), lab, "pc", "gauss", 4.0,
                 iterations=30)


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg2_small": cfg2_small, "cfg3": cfg3,
           "cfg4": cfg4, "cfg4_small": cfg4_small, "cfg4_sample": cfg4_sample,
           "cfg5_0": lambda: cfg5_image(0), "cfg5_1": lambda: cfg5_image(1)}
