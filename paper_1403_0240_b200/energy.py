"""Region energies and single-flip increments (mirror of rcseg.energy,
energy.py:1-408).  Increments and totals are computed by the CUDA library:
K3 (PC increment, perimeter change), K4/K5 (PS own-label ball fields and
increment) and K9 (correctly rounded totals, math.fsum semantics)."""
from __future__ import annotations

import ctypes as C
import functools
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import DegenerateStatsError  # noqa: F401  (re-export, energy.py:33)
from .grid import StatsTable, validate_image, validate_labels

POISSON_MEAN_FLOOR = 1e-8


@dataclass
class EnergyConfig:
    """energy.py:37-50"""
    region_model: str = "pc"
    noise_model: str = "gauss"
    lam: float = 0.0
    smooth_radius: int = 8

    def __post_init__(self):
        if self.region_model not in ("pc", "ps"):
            raise ValueError(f"unknown region model {self.region_model!r}")
        if self.noise_model not in ("gauss", "poisson"):
            raise ValueError(f"unknown noise model {self.noise_model!r}")
        if self.smooth_radius < 1:
            raise ValueError("smooth_radius must be >= 1")

    def c_struct(self) -> _lib.EnergyCfg:
        return _lib.EnergyCfg(int(self.region_model == "ps"), int(self.noise_model == "poisson"),
                              float(self.lam), int(self.smooth_radius))


@dataclass(frozen=True)
class EnergyValue:
    total: float
    external: float
    internal: int


@functools.lru_cache(maxsize=None)
def ball_offsets(ndim: int, radius: int) -> np.ndarray:
    """Ball offsets, centre first, |o|^2 ascending (energy.py:60-70) — the
    walk order of the PS kernels."""
    g = np.stack(np.meshgrid(*([np.arange(-radius, radius + 1)] * ndim), indexing="ij"),
                 -1).reshape(-1, ndim)
    d2 = (g * g).sum(axis=1)
    keep = d2 <= radius * radius
    out = np.ascontiguousarray(g[keep][np.argsort(d2[keep], kind="stable")])
    out.setflags(write=False)
    return out


@functools.lru_cache(maxsize=None)
def _ball_mask(ndim: int, radius: int) -> np.ndarray:
    """energy.py:73-79: boolean (2r+1)^d mask of |o|^2 <= r^2."""
    g = np.meshgrid(*([np.arange(-radius, radius + 1)] * ndim), indexing="ij")
    mask = sum(x * x for x in g) <= radius * radius
    mask.setflags(write=False)
    return mask


def _ball_sum(field: np.ndarray, radius: int) -> np.ndarray:
    """energy.py:161-193: sum of ``field`` over the radius ball around every
    cell, zero outside — on the device (rcb_ball_sum) with the reference's
    cumulative-sum spans, so float fields round identically."""
    f = np.ascontiguousarray(field, np.float64)
    if f.ndim not in (2, 3):
        raise ValueError("field must be 2-D or 3-D")
    out = np.empty_like(f)
    _lib.require_device()
    _lib.check(_lib.lib.rcb_ball_sum(_lib.ptr(f), f.ndim, _lib.ptr(_lib.dims_arr(f.shape)),
                                     int(radius), _lib.ptr(out)))
    return out


def smooth_fields(labels: np.ndarray, image: np.ndarray, radius: int, n_labels: int):
    """energy.py:196-223: dense per-label ball counts C and sums S, shape
    (n_labels, *dims), each label windowed to its bounding box grown by the
    radius as the reference does (rcb_smooth_fields).  The engine never
    builds these (it keeps own-label fields only); this is the function-level
    drop-in."""
    validate_labels(labels)
    lab = np.ascontiguousarray(labels, np.int32)
    img = np.ascontiguousarray(image, np.float64)
    if lab.shape != img.shape:
        raise ValueError("label and intensity rasters differ in shape")
    Cf = np.empty((int(n_labels),) + lab.shape, np.float64)
    Sf = np.empty_like(Cf)
    _lib.require_device()
    _lib.check(_lib.lib.rcb_smooth_fields(_lib.ptr(lab), _lib.ptr(img), lab.ndim,
                                          _lib.ptr(_lib.dims_arr(lab.shape)), int(radius),
                                          int(n_labels), _lib.ptr(Cf), _lib.ptr(Sf)))
    return Cf, Sf


def perimeter(labels: np.ndarray) -> int:
    """energy.py:82-88: face-adjacent pairs with different labels (the
    device total's internal term)."""
    validate_labels(labels)
    lab = np.ascontiguousarray(labels, np.int32)
    return evaluate_total(lab, np.zeros(lab.shape), EnergyConfig("pc", "gauss")).internal


def _particles(labels, pixels, owners, competitors):
    return (_lib.c64(pixels), _lib.c64(owners), _lib.c64(competitors))


def delta_internal_batch(labels, pixels, owners, competitors) -> np.ndarray:
    """energy.py:111-126 on the GPU."""
    lab = np.ascontiguousarray(labels, np.int32)
    xs, ow, cm = _particles(labels, pixels, owners, competitors)
    out = np.zeros(len(xs), np.int64)
    if len(xs):
        dims = _lib.dims_arr(lab.shape)
        _lib.check(_lib.lib.rcb_delta_internal_batch(
            _lib.ptr(lab), lab.ndim, _lib.ptr(dims), _lib.ptr(xs), _lib.ptr(ow), _lib.ptr(cm),
            len(xs), _lib.ptr(out)))
    return out


def delta_internal(labels, pixel: int, competitor: int) -> int:
    """energy.py:91-108"""
    own = int(np.asarray(labels).ravel()[pixel])
    return int(delta_internal_batch(labels, [pixel], [own], [competitor])[0])


def evaluate_total(labels, image, config: EnergyConfig) -> EnergyValue:
    """energy.py:233-257: from-scratch energy; external is correctly rounded."""
    validate_labels(labels)
    validate_image(image)
    if config.noise_model == "poisson" and image.size and image.min() < 0:
        raise ValueError("Poisson noise model requires nonnegative intensities")
    lab = np.ascontiguousarray(labels, np.int32)
    img = np.ascontiguousarray(image, np.float64)
    dims = _lib.dims_arr(lab.shape)
    ext = C.c_double(0.0)
    inter = C.c_int64(0)
    cfg = config.c_struct()
    _lib.check(_lib.lib.rcb_evaluate_total(_lib.ptr(img), _lib.ptr(lab), lab.ndim,
                                           _lib.ptr(dims), C.byref(cfg), C.byref(ext),
                                           C.byref(inter)))
    internal = int(inter.value)
    external = float(ext.value)
    return EnergyValue(external + config.lam * internal, external, internal)


class EnergyModel:
    """Incremental energy bookkeeping bound to (labels, image)
    (energy.py:260-408).  PC increments read ``self.stats``; PS increments
    rebuild the own-label ball fields from the current raster on the GPU, so
    ``apply_flip`` has nothing to shift, and the dense ``_C`` / ``_S`` views
    are derived from the current raster when read (equal to the reference's
    incrementally shifted fields for integer data, where every ball sum is
    exact; within rounding otherwise)."""

    def __init__(self, image, labels, config: EnergyConfig):
        validate_image(image)
        validate_labels(labels)
        if image.shape != labels.shape:
            raise ValueError("label and intensity rasters differ in shape")
        if config.noise_model == "poisson" and image.size and image.min() < 0:
            raise ValueError("Poisson noise model requires nonnegative intensities")
        self.image = image
        self.labels = labels
        self.config = config
        self.n_labels = int(labels.max()) + 1
        self.stats = None
        self.refresh()

    def refresh(self) -> None:
        self.stats = StatsTable.from_labels(self.labels, self.image, self.n_labels)

    def delta_external(self, pixel: int, owner: int, competitor: int) -> float:
        if self.stats.count[owner] == 0:
            raise DegenerateStatsError(f"region {owner} is empty")
        return float(self.delta_external_batch(np.array([pixel]), np.array([owner]),
                                               np.array([competitor]))[0])

    def delta_external_batch(self, pixels, owners, competitors) -> np.ndarray:
        xs, ow, cm = _particles(self.labels, pixels, owners, competitors)
        out = np.zeros(len(xs), np.float64)
        if not len(xs):
            return out
        lab = np.ascontiguousarray(self.labels, np.int32)
        img = np.ascontiguousarray(self.image, np.float64)
        dims = _lib.dims_arr(lab.shape)
        cfg = self.config.c_struct()
        st = self.stats
        cnt = np.ascontiguousarray(st.count, np.int64)
        tot = np.ascontiguousarray(st.total, np.float64)
        tsq = np.ascontiguousarray(st.total_sq, np.float64)
        _lib.check(_lib.lib.rcb_delta_external_batch(
            _lib.ptr(img), _lib.ptr(lab), lab.ndim, _lib.ptr(dims), C.byref(cfg), st.n_labels,
            _lib.ptr(cnt), _lib.ptr(tot), _lib.ptr(tsq), _lib.ptr(xs), _lib.ptr(ow),
            _lib.ptr(cm), len(xs), _lib.ptr(out)))
        return out

    def delta_total(self, pixel: int, owner: int, competitor: int) -> float:
        return (self.delta_external(pixel, owner, competitor)
                + self.config.lam * delta_internal(self.labels, pixel, competitor))

    def apply_flip(self, pixel: int, owner: int, competitor: int) -> None:
        """energy.py:381-408 — a no-op here: PS fields are derived from the
        raster on the device at every evaluation."""
        return None

    @property
    def _C(self):
        return self._fields()[0]

    @property
    def _S(self):
        return self._fields()[1]

    def _fields(self):
        if self.config.region_model != "ps":
            return None, None
        return smooth_fields(self.labels, self.image, self.config.smooth_radius, self.n_labels)
