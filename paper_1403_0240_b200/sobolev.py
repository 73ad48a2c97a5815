"""Sobolev-gradient filter (mirror of rcseg.sobolev, sobolev.py:1-192).

``sobolev_filter`` runs the K6 lattice-stencil kernel on the GPU.  The
kernel *table* w[d2] = kernel_eval(sqrt(d2)) is evaluated here on the host by
the reference's own formula, which is what makes the device sums
bit-identical.
"""
from __future__ import annotations

import ctypes as C
import functools
import math
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass(frozen=True)
class SobolevParams:
    """sobolev.py:18-31: kernel support (-E/2, E/2), metric weight eps."""
    length_scale: float = 12.0
    epsilon: float = 1.0 / 24.0

    def __post_init__(self):
        if self.length_scale <= 0:
            raise ValueError("length_scale must be positive")
        if self.epsilon <= 0:
            raise ValueError("epsilon must be positive")

    @property
    def cutoff(self) -> float:
        return self.length_scale / 2.0


def kernel_eval(r, params: SobolevParams):
    """Eq. 5 kernel K(r) = (1 + (u^2 - u + 1/6)/(2 eps)) / E, u = |r|/E
    (sobolev.py:34-49); raises outside the support."""
    r = np.asarray(r, dtype=np.float64)
    E = params.length_scale
    if np.any(np.abs(r) > E / 2.0):
        raise ValueError("kernel evaluated outside its support")
    u = np.abs(r) / E
    val = (1.0 + (u * u - u + 1.0 / 6.0) / (2.0 * params.epsilon)) / E
    return float(val) if val.ndim == 0 else val


@functools.lru_cache(maxsize=64)
def weight_table(length_scale: float, epsilon: float) -> np.ndarray:
    """w[d2] for every integer d2 < cutoff^2 (strict cutoff, sobolev.py:121)."""
    p = SobolevParams(length_scale, epsilon)
    c2 = p.cutoff * p.cutoff
    d2 = np.arange(int(math.ceil(c2)), dtype=np.int64)
    d2 = d2[d2 < c2]
    w = np.ascontiguousarray(np.atleast_1d(kernel_eval(np.sqrt(d2.astype(np.float64)), p)),
                             np.float64)
    w.setflags(write=False)
    return w


def sobolev_cfg(params: SobolevParams):
    """Fill the C struct; the returned tuple keeps the table alive."""
    w = weight_table(float(params.length_scale), float(params.epsilon))
    cfg = _lib.SobolevCfg(float(params.length_scale), float(params.epsilon),
                          w.ctypes.data_as(C.POINTER(C.c_double)), len(w))
    return cfg, w


class CellList:
    """sobolev.py:50-122: the bucket grid's query interface.  Buckets are
    floor_divide(coords, edge); a pair or point hit needs its buckets to be box
    neighbours and the squared distance below cutoff^2 (strict) — the
    reference's semantics, cutoffs beyond the edge included.  Both queries run
    on the device (rcb_cell_pairs / rcb_cell_query); the engine's Sobolev
    filter does not use them (it walks the lattice CSR index instead)."""

    def __init__(self, coords: np.ndarray, edge: float):
        coords = np.asarray(coords)
        if coords.ndim != 2 or coords.shape[1] not in (2, 3):
            raise ValueError("coords must be (n, 2) or (n, 3)")
        if edge <= 0:
            raise ValueError("bucket edge must be positive")
        self.coords = np.ascontiguousarray(coords, dtype=np.int64)
        self.edge = float(edge)

    def __len__(self) -> int:
        return len(self.coords)

    def query(self, point, cutoff: float, exclude: int | None = None) -> np.ndarray:
        """Indices of particles strictly within ``cutoff`` of ``point``, ascending."""
        n = len(self.coords)
        if n == 0:
            return np.empty(0, dtype=np.int64)
        pt = np.ascontiguousarray(np.asarray(point, dtype=np.float64).ravel())
        if pt.size != self.coords.shape[1]:
            raise ValueError("point dimension differs from the coordinates")
        out = np.empty(n, np.int64)
        k = C.c_int64(0)
        _lib.require_device()
        _lib.check(_lib.lib.rcb_cell_query(
            _lib.ptr(self.coords), n, self.coords.shape[1], self.edge, _lib.ptr(pt), float(cutoff),
            -1 if exclude is None else int(exclude), _lib.ptr(out), C.byref(k)))
        return out[:k.value]

    def pairs(self, cutoff: float):
        """All ordered pairs (p, q) with d(p, q) < cutoff, p == q included:
        (p_idx, q_idx, distance), sorted by (p, q)."""
        n = len(self.coords)
        e = np.empty(0, dtype=np.int64)
        if n == 0:
            return e, e, np.empty(0, dtype=np.float64)
        _lib.require_device()
        cap = 0
        bufs = (e, e, np.empty(0, np.float64))
        tot = C.c_int64(0)
        for _ in range(2):
            st = _lib.lib.rcb_cell_pairs(_lib.ptr(self.coords), n, self.coords.shape[1], self.edge,
                                         float(cutoff), _lib.ptr(bufs[0]), _lib.ptr(bufs[1]),
                                         _lib.ptr(bufs[2]), cap, C.byref(tot))
            if st == _lib.RCB_ERR_CAPACITY:
                cap = tot.value
                bufs = (np.empty(cap, np.int64), np.empty(cap, np.int64), np.empty(cap, np.float64))
                continue
            _lib.check(st)
            break
        k = tot.value
        return bufs[0][:k], bufs[1][:k], bufs[2][:k]


def build_cell_list(coords: np.ndarray, params: SobolevParams) -> CellList:
    """sobolev.py:133-134"""
    return CellList(coords, params.cutoff)


def sobolev_filter(coords, owners, competitors, raw, params: SobolevParams,
                   cells: CellList | None = None, return_pairs: bool = False):
    """Two-sided kernel smoothing of per-particle increments (Eq. 6),
    bit-identical to sobolev.py:137-174 and independent of storage order."""
    if cells is not None:
        coords = cells.coords
    coords = np.ascontiguousarray(coords, np.int64)
    if coords.ndim != 2 or coords.shape[1] not in (2, 3):
        raise ValueError("coords must be (n, 2) or (n, 3)")
    owners = _lib.c64(owners)
    competitors = _lib.c64(competitors)
    raw = np.ascontiguousarray(raw, np.float64)
    n = len(raw)
    out = np.zeros(n, np.float64)
    pairs = C.c_int64(0)
    if n:
        cfg, _keep = sobolev_cfg(params)
        _lib.check(_lib.lib.rcb_sobolev_filter(
            _lib.ptr(coords), n, coords.shape[1], _lib.ptr(owners), _lib.ptr(competitors),
            _lib.ptr(raw), C.byref(cfg), _lib.ptr(out), C.byref(pairs)))
    return (out, pairs.value) if return_pairs else out


def detect_oscillation(energies, moves, window: int = 10, tol_rel: float = 1e-6) -> bool:
    """Host-side scalar rule of sobolev.py:177-192: the last ``window``
    iterations all moved, yet energy fell by at most tol_rel*|E_last|."""
    if len(energies) < window or window < 2:
        return False
    e = list(energies[-window:])
    if min(list(moves[-window:])) <= 0:
        return False
    return (e[0] - e[-1]) <= tol_rel * abs(e[-1])
