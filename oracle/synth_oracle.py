"""CPU restatement of the reference's synthetic-data pipeline (SURVEY §8f row
1; rcseg/synth.py) — TEST INFRASTRUCTURE ONLY: imported by tests/ as the
checker of the device pipeline (paper_1403_0240_b200/synth.py), never by the
product.  Pinned bit for bit against tests/golden/synth.npz, which the
reference itself produced (tests/golden/make_golden_synth.py).

* render_scene (synth.py:73-84): shapes in order, later ones overwrite; masks
  from float64 squared distances summed in axis order.
* blur (synth.py:87-103): separable Gaussian, radius ceil(4 sigma), kernel
  renormalised, mirror borders, axes in order.  scipy's correlate1d takes its
  symmetric-kernel path: out[i] = x[i] k[r] + sum over j = r..1 of
  (x[i-j] + x[i+j]) k[r+j], accumulated in that order (verified bit for bit
  against scipy 1.18.1 on 2-D/3-D inputs, every axis, lattices narrower than
  the kernel).
* poissonize (synth.py:106-182): peak mean psnr^2, per-pixel counter-based
  splitmix64 stream, CDF inversion below mean 30, Hormann's PTRS above.
"""
from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1
INVERSION_LIMIT = 30.0


def shape_mask(kind, dims, center=(), radius=0.0, inner=0.0, outer=0.0, origin=(), size=()):
    """synth.py:38-51"""
    grids = np.indices(dims, dtype=np.float64)
    if kind == "disk":
        d2 = sum((g - c) ** 2 for g, c in zip(grids, center))
        return d2 <= radius ** 2
    if kind == "annulus":
        d2 = sum((g - c) ** 2 for g, c in zip(grids, center))
        return (d2 >= inner ** 2) & (d2 <= outer ** 2)
    if kind == "rect":
        m = np.ones(dims, dtype=bool)
        for g, o, s in zip(grids, origin, size):
            m &= (g >= o) & (g < o + s)
        return m
    raise ValueError(f"unknown shape kind {kind!r}")


def render_scene(spec: dict):
    """synth.py:73-84 on a scene dict (synth.py:195-236 layout)."""
    dims = tuple(int(d) for d in spec["dims"])
    labels = np.zeros(dims, dtype=np.int32)
    image = np.full(dims, float(spec.get("background", 0.0)), dtype=np.float64)
    for i, s in enumerate(spec.get("shapes", []), start=1):
        m = shape_mask(s["kind"], dims, tuple(s.get("center", ())), float(s.get("radius", 0.0)),
                       float(s.get("inner", 0.0)), float(s.get("outer", 0.0)),
                       tuple(s.get("origin", ())), tuple(s.get("size", ())))
        labels[m] = i
        image[m] = float(s["intensity"])
    return labels, image


def gauss_kernel(sigma: float) -> np.ndarray:
    """synth.py:96-99"""
    radius = int(math.ceil(4.0 * sigma))
    t = np.arange(-radius, radius + 1, dtype=np.float64)
    k = np.exp(-(t * t) / (2.0 * sigma * sigma))
    k /= k.sum()
    return k


def mirror_index(i: np.ndarray, n: int) -> np.ndarray:
    """scipy 'mirror' boundary: (d c b | a b c d | c b a)."""
    if n == 1:
        return np.zeros_like(i)
    p = 2 * (n - 1)
    i = np.mod(i, p)
    return np.where(i < n, i, p - i)


def correlate1d_mirror(x: np.ndarray, k: np.ndarray, axis: int) -> np.ndarray:
    r = (len(k) - 1) // 2
    x = np.moveaxis(x, axis, -1)
    n = x.shape[-1]
    i = np.arange(n)
    out = x * k[r]
    for j in range(r, 0, -1):
        out = out + (x[..., mirror_index(i - j, n)] + x[..., mirror_index(i + j, n)]) * k[r + j]
    return np.ascontiguousarray(np.moveaxis(out, -1, axis))


def blur(image: np.ndarray, sigma: float) -> np.ndarray:
    """synth.py:87-103"""
    if sigma < 0:
        raise ValueError("sigma must be >= 0")
    if sigma == 0:
        return image.copy()
    k = gauss_kernel(sigma)
    out = image.astype(np.float64, copy=True)
    for axis in range(image.ndim):
        out = correlate1d_mirror(out, k, axis)
    return out


def mix64(x: int) -> int:
    """synth.py:106-110 (splitmix64 finaliser)"""
    x &= MASK64
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9 & MASK64
    x = (x ^ (x >> 27)) * 0x94D049BB133111EB & MASK64
    return x ^ (x >> 31)


class Stream:
    """synth.py:113-130: per-pixel counter-based splitmix64 stream."""

    def __init__(self, seed: int, index: int):
        self.state = mix64((seed & MASK64) * 0x9E3779B97F4A7C15 ^ mix64(index + 1))

    def next_u01(self) -> float:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        return ((mix64(self.state) >> 11) + 1) * (2.0 ** -53)


def poisson_draw(lam: float, st: Stream) -> int:
    """synth.py:133-166"""
    if lam <= 0.0:
        return 0
    if lam < INVERSION_LIMIT:
        u = st.next_u01()
        p = math.exp(-lam)
        cum = p
        k = 0
        cap = int(lam + 40.0 * math.sqrt(lam) + 100.0)
        while u > cum and k < cap:
            k += 1
            p *= lam / k
            cum += p
        return k
    smu = math.sqrt(lam)
    b = 0.931 + 2.53 * smu
    a = -0.059 + 0.02483 * b
    inv_alpha = 1.1239 + 1.1328 / (b - 3.4)
    v_r = 0.9277 - 3.6224 / (b - 2.0)
    log_lam = math.log(lam)
    while True:
        u = st.next_u01() - 0.5
        v = st.next_u01()
        us = 0.5 - abs(u)
        k = int(math.floor((2.0 * a / us + b) * u + lam + 0.43))
        if us >= 0.07 and v <= v_r:
            return k
        if k < 0 or (us < 0.013 and v > us):
            continue
        if (math.log(v) + math.log(inv_alpha) - math.log(a / (us * us) + b)
                <= k * log_lam - lam - math.lgamma(k + 1.0)):
            return k


def poissonize(image: np.ndarray, psnr: float, seed: int) -> np.ndarray:
    """synth.py:169-182"""
    if image.size and image.min() < 0:
        raise ValueError("poissonize requires nonnegative intensities")
    peak = float(image.max()) if image.size else 0.0
    out = np.zeros(image.shape, dtype=np.float64)
    if peak <= 0.0:
        return out
    scale = (psnr ** 2) / peak
    lam = image.ravel() * scale
    flat = out.ravel()
    for i in range(lam.size):
        flat[i] = poisson_draw(float(lam[i]), Stream(seed, i))
    return out
