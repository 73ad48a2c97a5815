"""Contour particles (mirror of rcseg.contour, contour.py:1-241).

``scan_contour`` is the K1 stream compaction on the GPU.  The returned
``ContourState`` is a host view of the particle set with the reference's
query methods; the engine itself never materialises it (the particle set is
re-extracted on the device every iteration).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .grid import Connectivity, validate_labels


class StaleParticleError(RuntimeError):
    """The particle's stored labels no longer match the raster (contour.py:20-21)."""


class ContourState:
    """Particle set keyed by (pixel, competing label) (contour.py:24-63)."""

    def __init__(self, xs=None, comps=None):
        self._comp: dict[int, set[int]] = {}
        if xs is not None:
            for x, c in zip(np.asarray(xs).tolist(), np.asarray(comps).tolist()):
                self._comp.setdefault(x, set()).add(c)

    def __len__(self) -> int:
        return sum(len(c) for c in self._comp.values())

    def competitors_at(self, pixel: int) -> frozenset:
        return frozenset(self._comp.get(pixel, ()))

    def set_pixel(self, pixel: int, competitors) -> None:
        if competitors:
            self._comp[pixel] = set(competitors)
        else:
            self._comp.pop(pixel, None)

    def as_key_set(self) -> set:
        return {(x, c) for x, cs in self._comp.items() for c in cs}

    def as_arrays(self, labels: np.ndarray):
        keys = sorted(self.as_key_set())
        xs = np.array([k[0] for k in keys], dtype=np.int64)
        cs = np.array([k[1] for k in keys], dtype=np.int64)
        return xs, labels.ravel()[xs].astype(np.int64), cs

    def pixels_of_region(self, label: int, labels: np.ndarray) -> np.ndarray:
        flat = labels.ravel()
        return np.array(sorted(x for x in self._comp if flat[x] == label), dtype=np.int64)


def scan_particles(labels: np.ndarray, conn: Connectivity):
    """GPU particle extraction: (xs, owners, competitors) int64, sorted by
    (x, competitor)."""
    validate_labels(labels)
    lab = np.ascontiguousarray(labels, np.int32)
    dims = _lib.dims_arr(lab.shape)
    n = C.c_int64(0)
    cap = 0
    e = np.empty(0, np.int64)
    bufs = (e, e, e)
    for _ in range(2):
        st = _lib.lib.rcb_scan_contour(_lib.ptr(lab), lab.ndim, _lib.ptr(dims),
                                       int(conn.full_fg), _lib.ptr(bufs[0]), _lib.ptr(bufs[1]),
                                       _lib.ptr(bufs[2]), cap, C.byref(n))
        if st == _lib.RCB_ERR_CAPACITY:
            cap = n.value
            bufs = tuple(np.empty(cap, np.int64) for _ in range(3))
            continue
        _lib.check(st)
        break
    k = n.value
    return bufs[0][:k], bufs[1][:k], bufs[2][:k]


def scan_contour(labels: np.ndarray, conn: Connectivity) -> ContourState:
    """contour.py:84-116"""
    xs, _, cs = scan_particles(labels, conn)
    return ContourState(xs, cs)
