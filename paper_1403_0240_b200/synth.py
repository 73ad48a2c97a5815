"""Synthetic benchmark scenes on the device: the reference's rcseg.synth
interface (rcseg/synth.py) — render, blur, poissonize, generate and the JSON
scene specs — with render/blur/poissonize computed by librcseg_b200
(csrc/synth.cu), bit-identical to the reference (tests/golden/synth.npz).
The reference's per-pixel Python loop in poissonize (synth.py:179-181) makes
512^3 inputs impractical; here the whole pipeline is one device pass.
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib

_MASK64 = (1 << 64) - 1
_KINDS = {"disk": 0, "rect": 1, "annulus": 2}
_WORDS = 15


@dataclass
class Shape:
    """synth.py:27-51"""
    kind: str
    intensity: float
    center: tuple = ()
    radius: float = 0.0
    inner: float = 0.0
    outer: float = 0.0
    origin: tuple = ()
    size: tuple = ()


@dataclass
class NoiseSpec:
    """synth.py:54-61"""
    psnr: float
    seed: int

    def __post_init__(self):
        if self.psnr <= 0:
            raise ValueError("psnr must be positive")


@dataclass
class SceneSpec:
    """synth.py:64-70"""
    dims: tuple
    background: float = 0.0
    shapes: list = field(default_factory=list)
    blur_sigma: float = 0.0
    noise: NoiseSpec | None = None


def _flatten(shapes) -> np.ndarray:
    """Shapes as the 15-double records of rcb_synth_generate (include/rcb.h);
    the squared radii and rectangle ends are formed here in Python exactly as
    the reference forms them (synth.py:42-50)."""
    out = np.zeros((max(len(shapes), 1), _WORDS), np.float64)
    for i, s in enumerate(shapes):
        if s.kind not in _KINDS:
            raise ValueError(f"unknown shape kind {s.kind!r}")
        r = out[i]
        r[0] = _KINDS[s.kind]
        r[1] = float(s.intensity)
        c = tuple(s.center)[:3]
        r[2] = len(c)
        r[3:3 + len(c)] = [float(v) for v in c]
        if s.kind == "disk":
            r[6], r[7] = -math.inf, s.radius ** 2
        elif s.kind == "annulus":
            r[6], r[7] = s.inner ** 2, s.outer ** 2
        else:
            pairs = list(zip(s.origin, s.size))[:3]
            r[8] = len(pairs)
            for a, (o, z) in enumerate(pairs):
                r[9 + a] = float(o)
                r[12 + a] = float(o + z)
    return np.ascontiguousarray(out)


def _kernel(sigma: float) -> np.ndarray:
    """synth.py:96-99 (host: a few taps)"""
    radius = int(math.ceil(4.0 * sigma))
    t = np.arange(-radius, radius + 1, dtype=np.float64)
    k = np.exp(-(t * t) / (2.0 * sigma * sigma))
    k /= k.sum()
    return np.ascontiguousarray(k)


def _dims(dims) -> tuple:
    dims = tuple(int(d) for d in dims)
    if len(dims) not in (2, 3):
        raise ValueError("scene must be 2-D or 3-D")
    return dims


def _run(spec: SceneSpec, blur_sigma: float, noise, want_clean: bool):
    _lib.require_device()
    dims = _dims(spec.dims)
    if blur_sigma < 0:
        raise ValueError("sigma must be >= 0")
    shp = _flatten(spec.shapes)
    k = _kernel(blur_sigma) if blur_sigma > 0 else np.zeros(1)
    labels = np.empty(dims, np.int32)
    clean = np.empty(dims, np.float64) if want_clean else None
    image = np.empty(dims, np.float64)
    _lib.check(_lib.lib.rcb_synth_generate(
        len(dims), _lib.ptr(_lib.dims_arr(dims)), float(spec.background), _lib.ptr(shp),
        len(spec.shapes), _lib.ptr(k), len(k) if blur_sigma > 0 else 0, int(noise is not None),
        float(noise.psnr ** 2) if noise is not None else 0.0,
        (int(noise.seed) & _MASK64) if noise is not None else 0, _lib.ptr(labels),
        _lib.ptr(clean) if clean is not None else None, _lib.ptr(image)))
    return labels, clean, image


def render_scene(spec: SceneSpec) -> tuple[np.ndarray, np.ndarray]:
    """synth.py:73-84: (truth labels, clean intensity image)."""
    labels, _, image = _run(spec, 0.0, None, False)
    return labels, image


def blur(image: np.ndarray, sigma: float) -> np.ndarray:
    """synth.py:87-103: separable Gaussian, 4-sigma truncation, mirror borders."""
    if sigma < 0:
        raise ValueError("sigma must be >= 0")
    img = np.ascontiguousarray(image, np.float64)
    if sigma == 0:
        return img.copy()
    _lib.require_device()
    dims = _dims(img.shape)
    k = _kernel(sigma)
    out = np.empty_like(img)
    _lib.check(_lib.lib.rcb_synth_blur(_lib.ptr(img), len(dims), _lib.ptr(_lib.dims_arr(dims)),
                                       _lib.ptr(k), len(k), _lib.ptr(out)))
    return out


def poissonize(image: np.ndarray, noise: NoiseSpec) -> np.ndarray:
    """synth.py:169-182: peak mean psnr**2, per-pixel counter-based draws."""
    img = np.ascontiguousarray(image, np.float64)
    out = np.zeros(img.shape, np.float64)
    if img.size == 0:
        return out
    _lib.require_device()
    _lib.check(_lib.lib.rcb_synth_poissonize(_lib.ptr(img), img.size, float(noise.psnr ** 2),
                                             int(noise.seed) & _MASK64, _lib.ptr(out)))
    return out


def generate(spec: SceneSpec) -> tuple[np.ndarray, np.ndarray]:
    """synth.py:185-192: render -> blur -> (poissonize), one device pass."""
    labels, _, image = _run(spec, spec.blur_sigma, spec.noise, False)
    return labels, image


# -- JSON spec files (synth.py:195-250) -----------------------------------

def scene_to_dict(spec: SceneSpec) -> dict:
    shapes = []
    for s in spec.shapes:
        d = {"kind": s.kind, "intensity": s.intensity}
        if s.kind in ("disk", "annulus"):
            d["center"] = list(s.center)
        if s.kind == "disk":
            d["radius"] = s.radius
        if s.kind == "annulus":
            d["inner"] = s.inner
            d["outer"] = s.outer
        if s.kind == "rect":
            d["origin"] = list(s.origin)
            d["size"] = list(s.size)
        shapes.append(d)
    out = {"dims": list(spec.dims), "background": spec.background, "shapes": shapes,
           "blur_sigma": spec.blur_sigma}
    if spec.noise is not None:
        out["noise"] = {"psnr": spec.noise.psnr, "seed": spec.noise.seed}
    return out


def scene_from_dict(d: dict) -> SceneSpec:
    shapes = [Shape(kind=s["kind"], intensity=float(s["intensity"]),
                    center=tuple(s.get("center", ())), radius=float(s.get("radius", 0.0)),
                    inner=float(s.get("inner", 0.0)), outer=float(s.get("outer", 0.0)),
                    origin=tuple(s.get("origin", ())), size=tuple(s.get("size", ())))
              for s in d.get("shapes", [])]
    noise = None
    if d.get("noise") is not None:
        noise = NoiseSpec(psnr=float(d["noise"]["psnr"]), seed=int(d["noise"]["seed"]))
    return SceneSpec(dims=tuple(int(v) for v in d["dims"]),
                     background=float(d.get("background", 0.0)), shapes=shapes,
                     blur_sigma=float(d.get("blur_sigma", 0.0)), noise=noise)


def save_scene(spec: SceneSpec, path) -> None:
    with open(path, "w") as fh:
        json.dump(scene_to_dict(spec), fh, indent=2)
        fh.write("\n")


def load_scene(path) -> SceneSpec:
    with open(path) as fh:
        return scene_from_dict(json.load(fh))


# -- stock benchmark scenes (synth.py:252-296) --------------------------------

def desk_scene(noise_seed: int = 7) -> SceneSpec:
    """64x64: two blurred disks and a rectangle in Poisson noise."""
    return SceneSpec(dims=(64, 64), background=0.5,
                     shapes=[Shape("disk", 10.0, center=(18, 18), radius=8.0),
                             Shape("disk", 8.0, center=(44, 16), radius=6.0),
                             Shape("rect", 10.0, origin=(36, 36), size=(16, 13))],
                     blur_sigma=2.0, noise=NoiseSpec(psnr=6.0, seed=noise_seed))


def two_blob_scene(noise_seed: int = 7) -> SceneSpec:
    """64x64: two blurred disks of different brightness on a dark field."""
    return SceneSpec(dims=(64, 64), background=0.0,
                     shapes=[Shape("disk", 10.0, center=(19, 19), radius=7.0),
                             Shape("disk", 6.0, center=(45, 45), radius=5.0)],
                     blur_sigma=2.0, noise=NoiseSpec(psnr=6.0, seed=noise_seed))


def two_sphere_scene(noise_seed: int = 7) -> SceneSpec:
    """32^3: two bright spheres, for 3-D sanity runs."""
    return SceneSpec(dims=(32, 32, 32), background=0.0,
                     shapes=[Shape("disk", 10.0, center=(10, 10, 10), radius=6.0),
                             Shape("disk", 8.0, center=(22, 22, 22), radius=5.0)],
                     blur_sigma=1.5, noise=NoiseSpec(psnr=6.0, seed=noise_seed))
