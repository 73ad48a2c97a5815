"""Initial labelings from a scheme string (mirror of rcseg.optimizer.initialize,
optimizer.py:284-405).

Host-side set-up that runs once per image, before the device engine: ``rect``,
``bubbles:<n>[:<r>]``, ``otsu``, ``maxima:<sigma>:<r>`` (the blur is the
device ``synth.blur``, bit-identical to the reference's) and ``file:<path>``.
Every scheme ends in ``split_disjoint_labels`` so each positive label is one
connected component, numbered 1..K in (old label, scipy component) order.
Parity: ``tests/golden/init.npz`` (``make_golden_init.py``, written by the
reference's ``initialize``).
"""
from __future__ import annotations

import itertools
import warnings

import numpy as np
from scipy import ndimage

from .grid import LABEL_DTYPE, Connectivity, validate_image


def otsu_threshold(hist: np.ndarray) -> int | None:
    """optimizer.py:284-308: t maximising the between-class variance of the
    split [0, t] | [t+1, 255]; None when no split has two non-empty classes."""
    h = np.asarray(hist, dtype=np.float64)
    if h.shape != (256,):
        raise ValueError("otsu_threshold expects a 256-bin histogram")
    w0 = np.cumsum(h)
    s0 = np.cumsum(h * np.arange(256, dtype=np.float64))
    w1, s1 = w0[-1] - w0[:-1], s0[-1] - s0[:-1]
    w0, s0 = w0[:-1], s0[:-1]
    ok = (w0 > 0) & (w1 > 0)
    if not ok.any():
        return None
    m0 = np.where(w0 > 0, s0 / np.maximum(w0, 1), 0.0)
    m1 = np.where(w1 > 0, s1 / np.maximum(w1, 1), 0.0)
    return int(np.argmax(np.where(ok, w0 * w1 * (m0 - m1) ** 2, -np.inf)))


def split_disjoint_labels(labels: np.ndarray, conn: Connectivity) -> np.ndarray:
    """optimizer.py:311-322 (components by the device union-find,
    grid.flood_fill_components' numbering = ndimage.label's)"""
    from .grid import _components
    out = np.zeros(labels.shape, dtype=LABEL_DTYPE)
    nxt = 1
    for lab in np.unique(labels):
        if lab <= 0:
            continue
        comp, n = _components(labels, int(lab), conn)
        for k in range(1, n + 1):
            out[comp == k] = nxt
            nxt += 1
    return out


def _paint_disks(dims, centers, radius: float) -> np.ndarray:
    """Label i+1 on the closed ball around centers[i]; later balls overwrite."""
    out = np.zeros(dims, dtype=LABEL_DTYPE)
    grids = np.indices(dims, dtype=np.float64)
    for i, c in enumerate(centers, start=1):
        d2 = sum((g - x) ** 2 for g, x in zip(grids, c))
        out[d2 <= radius * radius] = i
    return out


def _fields(scheme: str, prefix: str, counts) -> list[str]:
    parts = scheme.split(":")
    if len(parts) not in counts:
        raise ValueError(f"bad {prefix} scheme {scheme!r}")
    return parts[1:]


def initialize(image: np.ndarray, scheme: str, conn: Connectivity | None = None) -> np.ndarray:
    """optimizer.py:338-405"""
    validate_image(image)
    conn = conn or Connectivity.default(image.ndim)
    dims = image.shape
    if scheme == "rect":
        lab = np.zeros(dims, dtype=LABEL_DTYPE)
        lab[tuple(slice(max(1, s // 4), s - max(1, s // 4)) for s in dims)] = 1
    elif scheme.startswith("bubbles:"):
        f = _fields(scheme, "bubbles", (2, 3))
        per_axis, radius = int(f[0]), (float(f[1]) if len(f) == 2 else 4.0)
        if per_axis < 1 or radius <= 0:
            raise ValueError(f"bad bubbles scheme {scheme!r}")
        axes = [[(i + 0.5) * d / per_axis for i in range(per_axis)] for d in dims]
        lab = _paint_disks(dims, itertools.product(*axes), radius)
    elif scheme == "otsu":
        lo, hi = float(image.min()), float(image.max())
        if hi == lo:
            warnings.warn("otsu seeding on a constant image: empty foreground")
            return np.zeros(dims, dtype=LABEL_DTYPE)
        bins = np.rint((image - lo) / (hi - lo) * 255.0).astype(np.int64)
        t = otsu_threshold(np.bincount(bins.ravel(), minlength=256)[:256])
        if t is None:
            warnings.warn("otsu seeding found no valid split: empty foreground")
            return np.zeros(dims, dtype=LABEL_DTYPE)
        lab = (bins > t).astype(LABEL_DTYPE)
    elif scheme.startswith("maxima:"):
        from .synth import blur
        f = _fields(scheme, "maxima", (3,))
        sigma, radius = float(f[0]), float(f[1])
        smooth = blur(image, sigma)
        foot = np.ones((3,) * image.ndim, dtype=bool)
        foot[(1,) * image.ndim] = False
        nmax = ndimage.maximum_filter(smooth, footprint=foot, mode="constant", cval=-np.inf)
        lab = _paint_disks(dims, np.argwhere(smooth > nmax), radius)
    elif scheme.startswith("file:"):
        from .imageio import read_labels
        lab = read_labels(scheme[5:])
        if lab.shape != dims:
            raise ValueError(f"label file shape {lab.shape} does not match image {dims}")
    else:
        raise ValueError(f"unknown initialization scheme {scheme!r}")
    return split_disjoint_labels(lab, conn)
