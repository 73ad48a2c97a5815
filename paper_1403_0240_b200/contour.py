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
        self._competitors: dict[int, set[int]] = {}
        if xs is not None:
            for x, c in zip(np.asarray(xs).tolist(), np.asarray(comps).tolist()):
                self._competitors.setdefault(x, set()).add(c)

    def __len__(self) -> int:
        return sum(len(c) for c in self._competitors.values())

    def competitors_at(self, pixel: int) -> frozenset:
        return frozenset(self._competitors.get(pixel, ()))

    def set_pixel(self, pixel: int, competitors) -> None:
        if competitors:
            self._competitors[pixel] = set(competitors)
        else:
            self._competitors.pop(pixel, None)

    def as_key_set(self) -> set:
        return {(x, c) for x, cs in self._competitors.items() for c in cs}

    def as_arrays(self, labels: np.ndarray):
        keys = sorted(self.as_key_set())
        xs = np.array([k[0] for k in keys], dtype=np.int64)
        cs = np.array([k[1] for k in keys], dtype=np.int64)
        return xs, labels.ravel()[xs].astype(np.int64), cs

    def pixels_of_region(self, label: int, labels: np.ndarray) -> np.ndarray:
        flat = labels.ravel()
        return np.array(sorted(x for x in self._competitors if flat[x] == label), dtype=np.int64)


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


def _neighbor_labels(labels: np.ndarray, coord: tuple, offsets: np.ndarray) -> list:
    """contour.py:66-81: labels of the in-bounds neighbours of one pixel."""
    out = []
    shape = labels.shape
    for off in offsets:
        idx = tuple(coord[k] + int(off[k]) for k in range(len(shape)))
        if all(0 <= idx[k] < shape[k] for k in range(len(shape))):
            out.append(int(labels[idx]))
    return out


def repair_pixel(labels: np.ndarray, contour: ContourState, pixel: int,
                 conn: Connectivity) -> None:
    """contour.py:119-125: recompute one pixel's particles from the raster."""
    coord = np.unravel_index(pixel, labels.shape)
    own = int(labels.ravel()[pixel])
    contour.set_pixel(pixel, {l for l in _neighbor_labels(labels, coord, conn.bg_offsets)
                              if l != own})


def moves_admissible(labels: np.ndarray, pixels, competitors, conn: Connectivity,
                     allow_fusion: bool = False, allow_vanish: bool = True,
                     region_counts=None) -> np.ndarray:
    """Batched contour.py:171-207 on the device (rcb_moves_admissible): the
    local 3^d test per query and, where it is inconclusive, a device flood
    fill of the donor region minus the pixel."""
    validate_labels(labels)
    lab = np.ascontiguousarray(labels, np.int32)
    xs = _lib.c64(np.atleast_1d(pixels))
    cs = _lib.c64(np.atleast_1d(competitors))
    if len(xs) != len(cs):
        raise ValueError("pixels and competitors differ in length")
    rc = None if region_counts is None else _lib.c64(np.atleast_1d(region_counts))
    out = np.zeros(len(xs), np.int32)
    if len(xs):
        _lib.require_device()
        _lib.check(_lib.lib.rcb_moves_admissible(
            _lib.ptr(lab), lab.ndim, _lib.ptr(_lib.dims_arr(lab.shape)), int(conn.full_fg),
            _lib.ptr(xs), _lib.ptr(cs), _lib.ptr(rc) if rc is not None else None, len(xs),
            int(bool(allow_fusion)), int(bool(allow_vanish)), _lib.ptr(out)))
    return out.astype(bool)


def is_move_admissible(labels: np.ndarray, pixel: int, competitor: int, conn: Connectivity,
                       allow_fusion: bool = False, allow_vanish: bool = True,
                       region_count: int | None = None) -> bool:
    """contour.py:171-207: every foreground region stays one component, no
    contact of distinct foreground labels unless fusion is allowed, and a
    region's last pixel goes only when vanishing is allowed."""
    rc = None if region_count is None else [int(region_count)]
    return bool(moves_admissible(labels, [int(pixel)], [int(competitor)], conn, allow_fusion,
                                 allow_vanish, rc)[0])


def apply_move(labels: np.ndarray, contour: ContourState, stats, image: np.ndarray,
               pixel: int, owner: int, competitor: int, conn: Connectivity) -> None:
    """contour.py:210-241: execute one move on host arrays (label, region
    statistics, local particle repair); StaleParticleError when the stored
    owner no longer matches or the competitor is no longer adjacent."""
    flat = labels.ravel()
    if int(flat[pixel]) != owner:
        raise StaleParticleError(f"pixel {pixel}: owner changed")
    coord = np.unravel_index(pixel, labels.shape)
    if competitor not in _neighbor_labels(labels, coord, conn.bg_offsets):
        raise StaleParticleError(f"pixel {pixel}: competitor {competitor} not adjacent")
    value = float(image.ravel()[pixel])
    flat[pixel] = competitor
    stats.remove(owner, value)
    stats.add(competitor, value)
    repair_pixel(labels, contour, pixel, conn)
    shape = labels.shape
    for off in conn.bg_offsets:
        idx = tuple(coord[k] + int(off[k]) for k in range(len(shape)))
        if all(0 <= idx[k] < shape[k] for k in range(len(shape))):
            repair_pixel(labels, contour, int(np.ravel_multi_index(idx, shape)), conn)
