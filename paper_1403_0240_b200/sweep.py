"""Sobolev-kernel sweep workload (BASELINE.json configs[4], second part):
contour particles of seeded sphere unions (radius U(6, 20)) in lattices up to
2048x2048x512, raw increments ~ N(0, 1); K6 alone, on the device."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .sobolev import SobolevParams, sobolev_cfg


def sphere_list(shape, n_spheres: int, seed: int, rmin: float = 6.0, rmax: float = 20.0):
    rng = np.random.default_rng(seed)
    nd = len(shape)
    out = np.zeros((n_spheres, 4), np.float32)
    for k in range(nd):
        out[:, 3 - nd + k] = rng.uniform(0, shape[k], size=n_spheres)
    out[:, 3] = rng.uniform(rmin, rmax, size=n_spheres)
    if nd == 2:  # (z, y, x, r) with z unused
        out[:, 0] = 0.0
    return np.ascontiguousarray(out)


class SobolevSweep:
    def __init__(self, shape, n_spheres: int, width: int, seed: int = 0, device: int = 0):
        _lib.require_device()
        self.shape = tuple(int(s) for s in shape)
        self.params = SobolevParams(2.0 * width)   # E = 2w
        sph = sphere_list(self.shape, n_spheres, seed)
        cfg, self._wt = sobolev_cfg(self.params)
        dims = _lib.dims_arr(self.shape)
        h = C.c_void_p()
        _lib.check(_lib.lib.rcb_sweep_create(len(self.shape), _lib.ptr(dims), _lib.ptr(sph),
                                             len(sph), seed, C.byref(cfg), device, C.byref(h)))
        self._h = h
        n = C.c_int64()
        v = C.c_int64()
        st = C.c_void_p()
        _lib.check(_lib.lib.rcb_sweep_info(h, C.byref(n), C.byref(v), C.byref(st)))
        self.n_particles, self.n_sites, self.stream = n.value, v.value, st.value or 0

    def run(self):
        pairs = C.c_int64()
        ms = C.c_float()
        _lib.check(_lib.lib.rcb_sweep_run(self._h, C.byref(pairs), C.byref(ms)))
        return pairs.value, ms.value

    def get(self):
        n = self.n_particles
        xs, ow, cm = (np.empty(n, np.int64) for _ in range(3))
        raw, out = np.empty(n), np.empty(n)
        _lib.check(_lib.lib.rcb_sweep_get(self._h, _lib.ptr(xs), _lib.ptr(ow), _lib.ptr(cm),
                                          _lib.ptr(raw), _lib.ptr(out), n))
        return xs, ow, cm, raw, out

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.lib.rcb_sweep_destroy(h)
            self._h = None
