"""CPU oracle for the Region Competition iteration — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_1403_0240_b200``) must never import it and fails loudly when its CUDA
library is missing.

It restates, in numpy, the algorithm of the CPU reference package ``rcseg``
(``/root/reference/pkg/src/rcseg``).  Every function cites the reference
file:line it follows.  The reference is pure Python on numpy/scipy; the
restatement keeps the same fp64 expression trees and summation orders so that
it is bit-identical to the reference on Gaussian models and on integer-valued
Poisson data (``log`` comes from the same numpy on the same machine).

Parity pin: ``tests/golden/*.npz`` were produced by running the reference
itself in the build container (``tests/golden/make_golden.py``); the CPU test
suite checks this oracle against every one of them (``tests/test_oracle_golden.py``).
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np
from scipy import ndimage

POISSON_MEAN_FLOOR = 1e-8            # energy.py:30
_MASK64 = 0xFFFFFFFFFFFFFFFF


class StaleParticleError(RuntimeError):
    """contour.py:20-21"""


class DegenerateStatsError(RuntimeError):
    """energy.py:33-34"""


# ---------------------------------------------------------------------------
# lattice neighbourhoods (grid.py:42-96)
# ---------------------------------------------------------------------------

def box_offsets(ndim: int, radius: int = 1) -> np.ndarray:
    """All offsets of the (2r+1)^d box in lexicographic (C) order."""
    rng = np.arange(-radius, radius + 1)
    mesh = np.stack(np.meshgrid(*([rng] * ndim), indexing="ij"), axis=-1)
    return mesh.reshape(-1, ndim).astype(np.int64)


def face_offsets(ndim: int) -> np.ndarray:
    b = box_offsets(ndim)
    return b[np.abs(b).sum(axis=1) == 1]


def full_offsets(ndim: int) -> np.ndarray:
    b = box_offsets(ndim)
    return b[np.any(b != 0, axis=1)]


@dataclass(frozen=True)
class Conn:
    """Foreground/background adjacency pair (grid.py:57-96).

    ``full_fg`` True is the default (8/4 in 2-D, 26/6 in 3-D)."""
    ndim: int
    full_fg: bool = True

    @property
    def fg(self) -> np.ndarray:
        return full_offsets(self.ndim) if self.full_fg else face_offsets(self.ndim)

    @property
    def bg(self) -> np.ndarray:
        return face_offsets(self.ndim) if self.full_fg else full_offsets(self.ndim)

    @property
    def fg_structure(self) -> np.ndarray:
        return ndimage.generate_binary_structure(self.ndim, self.ndim if self.full_fg else 1)


def _inb(coord, shape) -> bool:
    return all(0 <= c < s for c, s in zip(coord, shape))


# ---------------------------------------------------------------------------
# region statistics (grid.py:142-181)
# ---------------------------------------------------------------------------

class Stats:
    """count/total/total_sq per label; rebuild is a raster-order sequential
    sum per label (np.bincount, grid.py:155-169)."""

    def __init__(self, labels: np.ndarray, image: np.ndarray, n_labels: int):
        flat = labels.ravel()
        vals = image.ravel().astype(np.float64)
        self.count = np.bincount(flat, minlength=n_labels).astype(np.int64)
        self.total = np.bincount(flat, weights=vals, minlength=n_labels)
        self.total_sq = np.bincount(flat, weights=vals * vals, minlength=n_labels)

    def move(self, a: int, b: int, v: float) -> None:
        # contour.py:226-227 -> grid.py:171-181: remove(a) then add(b)
        if self.count[a] == 0:
            raise ValueError(f"removing a pixel from empty region {a}")
        self.count[a] -= 1
        self.total[a] -= v
        self.total_sq[a] -= v * v
        self.count[b] += 1
        self.total[b] += v
        self.total_sq[b] += v * v


# ---------------------------------------------------------------------------
# contour particles (contour.py:84-116)
# ---------------------------------------------------------------------------

def scan_particles(labels: np.ndarray, conn: Conn):
    """Particle set sorted by (x, competitor): one particle per distinct label
    c != L[x] among the in-bounds background-adjacency neighbours of x.
    Returns int64 (xs, owners, comps)."""
    shape = labels.shape
    flat = labels.ravel()
    xs_parts, cs_parts = [], []
    idx = np.arange(flat.size, dtype=np.int64).reshape(shape)
    for off in conn.bg:
        src = tuple(slice(max(0, -o), s - max(0, o)) for o, s in zip(off, shape))
        dst = tuple(slice(max(0, o), s + min(0, o)) for o, s in zip(off, shape))
        diff = labels[src] != labels[dst]
        xs_parts.append(idx[src][diff])
        cs_parts.append(labels[dst][diff].astype(np.int64))
    if not xs_parts:
        e = np.empty(0, np.int64)
        return e, e.copy(), e.copy()
    xs = np.concatenate(xs_parts)
    cs = np.concatenate(cs_parts)
    key = np.unique(np.stack([xs, cs], axis=1), axis=0)
    if key.size == 0:
        e = np.empty(0, np.int64)
        return e, e.copy(), e.copy()
    xs, cs = key[:, 0].copy(), key[:, 1].copy()
    return xs, flat[xs].astype(np.int64), cs


def site_competitors(labels: np.ndarray, x: int, conn: Conn) -> set:
    """Competitor set of one site from the raster (contour.py:119-125)."""
    coord = np.unravel_index(x, labels.shape)
    own = int(labels.ravel()[x])
    out = set()
    for off in conn.bg:
        nb = tuple(int(c + o) for c, o in zip(coord, off))
        if _inb(nb, labels.shape):
            l = int(labels[nb])
            if l != own:
                out.add(l)
    return out


# ---------------------------------------------------------------------------
# length prior (energy.py:82-126)
# ---------------------------------------------------------------------------

def perimeter(labels: np.ndarray) -> int:
    n = 0
    for ax in range(labels.ndim):
        a = np.swapaxes(labels, 0, ax)
        n += int(np.count_nonzero(a[1:] != a[:-1]))
    return n


def delta_internal_batch(labels, xs, owners, comps) -> np.ndarray:
    """Sum over the 2d in-bounds faces of [L[n] != c] - [L[n] != a]."""
    shape = labels.shape
    flat = labels.ravel()
    coords = np.unravel_index(xs, shape)
    out = np.zeros(len(xs), dtype=np.int64)
    stride = 1
    strides = []
    for s in reversed(shape):
        strides.append(stride)
        stride *= s
    strides = strides[::-1]
    for ax in range(labels.ndim):
        for step in (-1, 1):
            c = coords[ax] + step
            ok = (c >= 0) & (c < shape[ax])
            nb = np.where(ok, xs + step * strides[ax], 0)
            l = flat[nb]
            t = (l != comps).astype(np.int64) - (l != owners).astype(np.int64)
            out += np.where(ok, t, 0)
    return out


def delta_internal(labels, x: int, b: int) -> int:
    return int(delta_internal_batch(labels, np.array([x]), np.array([int(labels.ravel()[x])]),
                                    np.array([b]))[0])


# ---------------------------------------------------------------------------
# piecewise-constant increments (energy.py:129-143, 308-324; Appendix B3)
# ---------------------------------------------------------------------------

def _g_gauss(n, s, q):
    n = np.asarray(n, np.float64)
    s = np.asarray(s, np.float64)
    q = np.asarray(q, np.float64)
    d = np.where(n > 0, n, 1.0)
    return np.where(n > 0, q - s * s / d, 0.0)


def _g_poisson(n, s):
    n = np.asarray(n, np.float64)
    s = np.asarray(s, np.float64)
    d = np.where(n > 0, n, 1.0)
    m = np.maximum(s / d, POISSON_MEAN_FLOOR)
    return np.where(n > 0, s - s * np.log(m), 0.0)


def delta_pc(image_flat, stats: Stats, xs, owners, comps, noise: str) -> np.ndarray:
    v = image_flat[xs]
    na = stats.count[owners].astype(np.float64)
    nb = stats.count[comps].astype(np.float64)
    sa, sb = stats.total[owners], stats.total[comps]
    if noise == "gauss":
        qa, qb = stats.total_sq[owners], stats.total_sq[comps]
        old = _g_gauss(na, sa, qa) + _g_gauss(nb, sb, qb)
        new = _g_gauss(na - 1, sa - v, qa - v * v) + _g_gauss(nb + 1, sb + v, qb + v * v)
    else:
        old = _g_poisson(na, sa) + _g_poisson(nb, sb)
        new = _g_poisson(na - 1, sa - v) + _g_poisson(nb + 1, sb + v)
    return new - old


# ---------------------------------------------------------------------------
# piecewise-smooth fields and increments (energy.py:60-79, 146-230, 326-408)
# ---------------------------------------------------------------------------

def ball_offsets(ndim: int, r: int) -> np.ndarray:
    """Ball offsets, |off|^2 ascending, stable over lexicographic order,
    centre first (energy.py:60-70)."""
    b = box_offsets(ndim, r)
    d2 = (b * b).sum(axis=1)
    b = b[d2 <= r * r]
    d2 = d2[d2 <= r * r]
    return b[np.argsort(d2, kind="stable")]


def ball_mask(ndim: int, r: int) -> np.ndarray:
    g = np.meshgrid(*([np.arange(-r, r + 1)] * ndim), indexing="ij")
    return sum(x * x for x in g) <= r * r


def _ball_runs(ndim: int, r: int):
    """Ball as runs along the last axis: (transverse offset, half length),
    transverse offsets in lexicographic order (energy.py:146-164)."""
    if ndim == 1:
        return [((), r)]
    t = box_offsets(ndim - 1, r)
    tt = (t * t).sum(axis=1)
    keep = tt <= r * r
    return [(tuple(int(o) for o in off), int(math.isqrt(int(r * r - q))))
            for off, q in zip(t[keep], tt[keep])]


def _ball_window_sum(field: np.ndarray, r: int) -> np.ndarray:
    """Sum of ``field`` over the ball of every cell, clipped at the window
    border, by prefix sums along the last axis, runs accumulated in run order
    (energy.py:167-193)."""
    last = field.shape[-1]
    pref = np.zeros(field.shape[:-1] + (last + 1,), np.float64)
    np.cumsum(field, axis=-1, out=pref[..., 1:])
    z = np.arange(last)
    out = np.zeros(field.shape, np.float64)
    for off, h in _ball_runs(field.ndim, r):
        if any(abs(d) >= n for d, n in zip(off, field.shape)):
            continue
        dst = tuple(slice(max(0, -d), n - max(0, d)) for d, n in zip(off, field.shape))
        src = tuple(slice(max(0, d), n + min(0, d)) for d, n in zip(off, field.shape))
        rows = pref[src]
        hi = np.minimum(z + h, last - 1) + 1
        lo = np.maximum(z - h, 0)
        out[dst] += np.take(rows, hi, axis=-1) - np.take(rows, lo, axis=-1)
    return out


def smooth_fields(labels, image, r: int, n_labels: int):
    """Dense per-label ball counts C and sums S, shape (L, *dims)
    (energy.py:196-223): each label over its bounding box grown by r."""
    C = np.zeros((n_labels,) + labels.shape)
    S = np.zeros((n_labels,) + labels.shape)
    boxes = ndimage.find_objects(labels, max_label=n_labels - 1)
    for l in range(n_labels):
        if l == 0:
            if not np.any(labels == 0):
                continue
            win = tuple(slice(0, s) for s in labels.shape)
        else:
            bx = boxes[l - 1]
            if bx is None:
                continue
            win = tuple(slice(max(0, sl.start - r), min(s, sl.stop + r))
                        for sl, s in zip(bx, labels.shape))
        m = (labels[win] == l).astype(np.float64)
        C[(l,) + win] = _ball_window_sum(m, r)
        S[(l,) + win] = _ball_window_sum(m * image[win], r)
    return C, S


def rho(i, theta, noise: str):
    """energy.py:226-230"""
    if noise == "gauss":
        d = i - theta
        return d * d
    return theta - i * np.log(np.maximum(theta, POISSON_MEAN_FLOOR))


def delta_ps(labels, image_flat, C, S, xs, owners, comps, r: int, noise: str) -> np.ndarray:
    """PS increment, owner side then competitor side, each in ball-offset
    order, then the centre terms (energy.py:326-372; Appendix B4)."""
    shape = labels.shape
    nl = C.shape[0]
    C2 = C.reshape(nl, -1)
    S2 = S.reshape(nl, -1)
    flat = labels.ravel()
    offs = ball_offsets(labels.ndim, r)[1:]
    strides = np.array([int(np.prod(shape[k + 1:])) for k in range(len(shape))], np.int64)
    out = np.empty(len(xs))
    step = max(64, 1_000_000 // max(1, len(offs)))
    for s0 in range(0, len(xs), step):
        px = xs[s0:s0 + step]
        pa = owners[s0:s0 + step]
        pb = comps[s0:s0 + step]
        cc = np.stack(np.unravel_index(px, shape), axis=1)
        ok = np.ones((len(px), len(offs)), bool)
        for k in range(len(shape)):
            ck = cc[:, k, None] + offs[None, :, k]
            ok &= (ck >= 0) & (ck < shape[k])
        yf = np.where(ok, px[:, None] + (offs @ strides)[None, :], 0)
        ly = flat[yf]
        v = image_flat[px]
        acc = np.zeros(len(px))
        for side, sg in ((pa, -1.0), (pb, 1.0)):
            rr, cidx = np.nonzero(ok & (ly == side[:, None]))
            y = yf[rr, cidx]
            lab = side[rr]
            cy, sy, iy = C2[lab, y], S2[lab, y], image_flat[y]
            d = rho(iy, (sy + sg * v[rr]) / (cy + sg), noise) - rho(iy, sy / cy, noise)
            acc += np.bincount(rr, weights=d, minlength=len(px))
        acc += rho(v, (S2[pb, px] + v) / (C2[pb, px] + 1), noise)
        acc -= rho(v, S2[pa, px] / C2[pa, px], noise)
        out[s0:s0 + step] = acc
    return out


def ps_flip(C, S, shape, x: int, a: int, b: int, v: float, r: int) -> None:
    """Shift the ball counts/sums of regions a and b (energy.py:381-408)."""
    m = ball_mask(len(shape), r)
    coord = np.unravel_index(x, shape)
    win, cut = [], []
    for k, c in enumerate(coord):
        lo, hi = c - r, c + r + 1
        win.append(slice(max(0, lo), min(shape[k], hi)))
        cut.append(slice(max(0, -lo), m.shape[k] - max(0, hi - shape[k])))
    mm = m[tuple(cut)]
    w = tuple(win)
    C[(a,) + w] -= mm
    S[(a,) + w] -= v * mm
    C[(b,) + w] += mm
    S[(b,) + w] += v * mm


# ---------------------------------------------------------------------------
# energy oracle (energy.py:233-257)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Energy:
    total: float
    external: float
    internal: int


def evaluate_total(labels, image, region: str, noise: str, lam: float, r: int) -> Energy:
    nl = int(labels.max()) + 1
    if region == "pc":
        st = Stats(labels, image, nl)
        per = _g_gauss(st.count, st.total, st.total_sq) if noise == "gauss" \
            else _g_poisson(st.count, st.total)
        ext = math.fsum(per.tolist())
    else:
        C, S = smooth_fields(labels, image, r, nl)
        flat = labels.ravel()
        ii = np.arange(flat.size)
        th = S.reshape(nl, -1)[flat, ii] / C.reshape(nl, -1)[flat, ii]
        ext = math.fsum(rho(image.ravel(), th, noise).tolist())
    p = perimeter(labels)
    return Energy(ext + lam * p, ext, p)


# ---------------------------------------------------------------------------
# Sobolev kernel and filter (sobolev.py:34-49, 137-174; Appendix B5)
# ---------------------------------------------------------------------------

def kernel_eval(r, E: float, eps: float):
    """K(r) = (1 + (u^2 - u + 1/6)/(2 eps))/E, u = |r|/E (sobolev.py:34-49)."""
    r = np.asarray(r, np.float64)
    if np.any(np.abs(r) > E / 2.0):
        raise ValueError("kernel evaluated outside its support")
    u = np.abs(r) / E
    return (1.0 + (u * u - u + 1.0 / 6.0) / (2.0 * eps)) / E


def weight_table(E: float, eps: float) -> np.ndarray:
    """w[d2] for every integer d2 < cutoff^2 (strict, sobolev.py:121)."""
    c2 = (E / 2.0) ** 2
    n = int(math.ceil(c2))
    d2 = np.arange(n, dtype=np.int64)
    d2 = d2[d2 < c2]
    return np.asarray(kernel_eval(np.sqrt(d2.astype(np.float64)), E, eps), np.float64).reshape(-1)


def stencil(ndim: int, E: float):
    """Lattice offsets with |off|^2 < (E/2)^2, lexicographic, and their d2."""
    c2 = (E / 2.0) ** 2
    r = int(math.ceil(E / 2.0))
    b = box_offsets(ndim, r)
    d2 = (b * b).sum(axis=1)
    keep = d2 < c2
    return b[keep], d2[keep]


def sobolev_filter(coords, owners, comps, raw, E: float = 12.0, eps: float = 1.0 / 24.0):
    """Two-sided kernel-weighted means over partners within the cutoff.
    For each p the partners q are summed in ascending (flat q, comp q, index q)
    order with flat taken over the coordinate bounding box (sobolev.py:155-171)."""
    coords = np.asarray(coords, np.int64)
    owners = np.asarray(owners, np.int64)
    comps = np.asarray(comps, np.int64)
    raw = np.asarray(raw, np.float64)
    n = len(raw)
    if n == 0:
        return np.zeros(0)
    nd = coords.shape[1]
    dims = tuple(int(coords[:, k].max()) + 1 for k in range(nd))
    flat = np.ravel_multi_index(tuple(coords[:, k] for k in range(nd)), dims)
    canon = np.lexsort((np.arange(n), comps, flat))        # q in canonical order
    sflat = flat[canon]
    offs, d2 = stencil(nd, E)
    wt = weight_table(E, eps)
    P, Q, W = [], [], []
    for off, dd in zip(offs, d2):
        nb = coords + off[None, :]
        ok = np.all((nb >= 0) & (nb < np.array(dims)[None, :]), axis=1)
        p_ok = np.flatnonzero(ok)
        if p_ok.size == 0:
            continue
        nf = np.ravel_multi_index(tuple(nb[p_ok, k] for k in range(nd)), dims)
        lo = np.searchsorted(sflat, nf, "left")
        hi = np.searchsorted(sflat, nf, "right")
        cnt = hi - lo
        if cnt.sum() == 0:
            continue
        pp = np.repeat(p_ok, cnt)
        start = np.repeat(lo, cnt)
        within = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        P.append(pp)
        Q.append(start + within)            # canonical position of q
        W.append(np.full(pp.size, wt[dd]))
    if not P:
        return np.zeros(n)
    P = np.concatenate(P)
    Qc = np.concatenate(Q)
    W = np.concatenate(W)
    o = np.lexsort((Qc, P))
    P, Qc, W = P[o], Qc[o], W[o]
    q = canon[Qc]
    contrib = W * raw[q]
    same = owners[q] == owners[P]
    opp = comps[q] == owners[P]
    ss = np.zeros(n)
    so = np.zeros(n)
    np.add.at(ss, P[same], contrib[same])
    np.add.at(so, P[opp], contrib[opp])
    cs = np.bincount(P[same], minlength=n)
    co = np.bincount(P[opp], minlength=n)
    out = np.where(cs > 0, ss / np.maximum(cs, 1), 0.0)
    out -= np.where(co > 0, so / np.maximum(co, 1), 0.0)
    return out


def pair_count(coords, E: float) -> int:
    """Number of ordered interacting pairs including p == q (the
    particle-interaction count of BASELINE.md §4)."""
    coords = np.asarray(coords, np.int64)
    n = len(coords)
    if n == 0:
        return 0
    nd = coords.shape[1]
    dims = tuple(int(coords[:, k].max()) + 1 for k in range(nd))
    flat = np.sort(np.ravel_multi_index(tuple(coords[:, k] for k in range(nd)), dims))
    offs, _ = stencil(nd, E)
    tot = 0
    for off in offs:
        nb = coords + off[None, :]
        ok = np.all((nb >= 0) & (nb < np.array(dims)[None, :]), axis=1)
        nf = np.ravel_multi_index(tuple(nb[ok, k] for k in range(nd)), dims)
        tot += int((np.searchsorted(flat, nf, "right") - np.searchsorted(flat, nf, "left")).sum())
    return tot


def detect_oscillation(energies, moves, window: int = 10, tol: float = 1e-6) -> bool:
    """sobolev.py:177-192"""
    if len(energies) < window or window < 2:
        return False
    e = list(energies[-window:])
    if min(list(moves[-window:])) <= 0:
        return False
    return (e[0] - e[-1]) <= tol * abs(e[-1])


# ---------------------------------------------------------------------------
# ranking (optimizer.py:80-87, 135-147; Appendix B6)
# ---------------------------------------------------------------------------

def tie_keys(xs, comps, seed: int) -> np.ndarray:
    m1 = np.uint64(0x9E3779B97F4A7C15)
    m2 = np.uint64(0xBF58476D1CE4E5B9)
    m3 = np.uint64(0x94D049BB133111EB)
    z = np.asarray(xs).astype(np.uint64) * m1
    z ^= np.asarray(comps).astype(np.uint64) * m2
    z ^= np.uint64(seed & _MASK64)
    z = (z ^ (z >> np.uint64(30))) * m2
    z = (z ^ (z >> np.uint64(27))) * m3
    return z ^ (z >> np.uint64(31))


def rank_order(rank, ties, xs, comps) -> np.ndarray:
    return np.lexsort((comps, xs, ties, rank))


# ---------------------------------------------------------------------------
# topology-safe acceptance (contour.py:128-207; Appendix B7)
# ---------------------------------------------------------------------------

def local_component_count(labels, x: int, a: int, conn: Conn) -> int:
    """0: no same-label cell in the punctured box; 1: every fg-adjacent
    same-label cell is connected inside the box; 2: inconclusive
    (contour.py:128-162)."""
    shape = labels.shape
    coord = np.unravel_index(x, shape)
    cells = set()
    for off in box_offsets(labels.ndim):
        if not off.any():
            continue
        nb = tuple(int(c + o) for c, o in zip(coord, off))
        if _inb(nb, shape) and labels[nb] == a:
            cells.add(tuple(int(o) for o in off))
    if not cells:
        return 0
    fg = [tuple(int(o) for o in off) for off in conn.fg]
    fgset = set(fg)
    seeds = [c for c in cells if c in fgset]
    if not seeds:
        return 2
    seen = {seeds[0]}
    stack = [seeds[0]]
    while stack:
        cur = stack.pop()
        for off in fg:
            nx = tuple(c + o for c, o in zip(cur, off))
            if nx in cells and nx not in seen:
                seen.add(nx)
                stack.append(nx)
    return 1 if all(s in seen for s in seeds) else 2


def admissible(labels, x: int, b: int, conn: Conn, allow_fusion: bool,
               allow_vanish: bool, count_a=None) -> bool:
    """contour.py:171-207"""
    flat = labels.ravel()
    a = int(flat[x])
    if a == b:
        return False
    coord = np.unravel_index(x, labels.shape)
    if a > 0:
        cnt = int(np.count_nonzero(flat == a)) if count_a is None else count_a
        if cnt == 1:
            if not allow_vanish:
                return False
        elif local_component_count(labels, x, a, conn) != 1:
            mask = labels == a
            mask.ravel()[x] = False
            if ndimage.label(mask, structure=conn.fg_structure)[1] != 1:
                return False
    if b > 0 and not allow_fusion:
        for off in conn.fg:
            nb = tuple(int(c + o) for c, o in zip(coord, off))
            if _inb(nb, labels.shape):
                l = int(labels[nb])
                if l > 0 and l != a and l != b:
                    return False
    return True


# ---------------------------------------------------------------------------
# the engine (optimizer.py:36-279)
# ---------------------------------------------------------------------------

@dataclass
class OptimizerConfig:
    gradient: str = "sobolev"
    max_iterations: int = 2000
    oscillation_window: int = 10
    oscillation_tol: float = 1e-6
    move_budget: float = 1.0
    seed: int = 0
    allow_fusion: bool = False
    allow_vanish: bool = True
    vanish_grace: int = 0
    resync_every: int = 10
    drift_tolerance: float = 1e-6


@dataclass
class IterationRecord:
    iteration: int
    energy: float
    moves: int
    particles: int
    mode: str
    seconds: float
    accepted: list = field(default_factory=list)   # [(x, a, b)] in acceptance order


class OracleEngine:
    """Sequential RC engine (optimizer.py:90-270) over the functions above."""

    def __init__(self, image, init_labels, region="pc", noise="gauss", lam=0.0,
                 smooth_radius=8, length_scale=12.0, epsilon=1.0 / 24.0,
                 config: OptimizerConfig | None = None, conn: Conn | None = None):
        self.image = np.ascontiguousarray(image, np.float64)
        self.labels = np.ascontiguousarray(init_labels, np.int32).copy()
        self.region, self.noise, self.lam, self.r = region, noise, float(lam), int(smooth_radius)
        self.E, self.eps = float(length_scale), float(epsilon)
        self.config = config or OptimizerConfig()
        self.conn = conn or Conn(self.image.ndim)
        self.mode = self.config.gradient
        self.n_labels = int(self.labels.max()) + 1
        self.flat_image = self.image.ravel()
        self._refresh()
        self.iteration = 0
        self.fallback_iteration = None
        self.trace: list[IterationRecord] = []
        self.last_candidates = None
        self._energy = self.evaluate().total
        self._mode_start = 0

    def _refresh(self):
        self.stats = Stats(self.labels, self.image, self.n_labels)
        if self.region == "ps":
            self.C, self.S = smooth_fields(self.labels, self.image, self.r, self.n_labels)

    def evaluate(self) -> Energy:
        return evaluate_total(self.labels, self.image, self.region, self.noise, self.lam, self.r)

    def delta_ext(self, xs, owners, comps):
        if self.region == "pc":
            return delta_pc(self.flat_image, self.stats, xs, owners, comps, self.noise)
        return delta_ps(self.labels, self.flat_image, self.C, self.S, xs, owners, comps,
                        self.r, self.noise)

    def particle_count(self) -> int:
        return len(scan_particles(self.labels, self.conn)[0])

    def iterate(self) -> IterationRecord:
        t0 = time.perf_counter()
        self.iteration += 1
        cfg = self.config
        xs, owners, comps = scan_particles(self.labels, self.conn)
        n = len(xs)
        accepted = []
        if n:
            raw_ext = self.delta_ext(xs, owners, comps)
            raw_int = delta_internal_batch(self.labels, xs, owners, comps)
            if self.mode == "sobolev":
                coords = np.stack(np.unravel_index(xs, self.labels.shape), axis=1)
                sm = sobolev_filter(coords, owners, comps, raw_ext, self.E, self.eps)
                rank = sm + self.lam * raw_int
            else:
                rank = raw_ext + self.lam * raw_int
            self.last_candidates = (xs, owners, comps, rank)
            order = rank_order(rank, tie_keys(xs, comps, cfg.seed), xs, comps)
            budget = int(math.ceil(cfg.move_budget * n))
            accepted = self._execute(order, xs, owners, comps, rank, budget)
        else:
            self.last_candidates = (xs, owners, comps, np.empty(0))
        if self.iteration % cfg.resync_every == 0:
            self._refresh()
            ref = self.evaluate().total
            drift = abs(ref - self._energy)
            if drift > cfg.drift_tolerance:
                raise RuntimeError(f"incremental energy drifted {drift:.3e} from the oracle "
                                   f"at iteration {self.iteration}")
            self._energy = ref
        rec = IterationRecord(self.iteration, self._energy, len(accepted), self.particle_count(),
                              self.mode, time.perf_counter() - t0, accepted)
        self.trace.append(rec)
        return rec

    def _execute(self, order, xs, owners, comps, rank, budget):
        cfg = self.config
        flat = self.labels.ravel()
        vanish_ok = cfg.allow_vanish and self.iteration > cfg.vanish_grace
        moved = set()
        acc = []
        for i in order:
            if not rank[i] < 0.0:
                break
            if len(acc) >= budget:
                break
            x, a, b = int(xs[i]), int(owners[i]), int(comps[i])
            if x in moved or int(flat[x]) != a:
                continue
            if b not in site_competitors(self.labels, x, self.conn):
                continue
            cnt = int(self.stats.count[a]) if a > 0 else None
            if not admissible(self.labels, x, b, self.conn, cfg.allow_fusion, vanish_ok, cnt):
                continue
            d = float(self.delta_ext(np.array([x]), np.array([a]), np.array([b]))[0]) \
                + self.lam * delta_internal(self.labels, x, b)
            if self.mode == "l2" and not d < 0.0:
                continue
            v = float(self.flat_image[x])
            flat[x] = b
            self.stats.move(a, b, v)
            if self.region == "ps":
                ps_flip(self.C, self.S, self.labels.shape, x, a, b, v, self.r)
            self._energy += d
            moved.add(x)
            acc.append((x, a, b))
        return acc

    def run(self, on_iteration=None):
        cfg = self.config
        status = "max-iter"
        for _ in range(cfg.max_iterations):
            prev_labels = self.labels.copy()
            prev_e = self._energy
            rec = self.iterate()
            if on_iteration is not None:
                on_iteration(self, rec)
            if rec.moves == 0:
                status = "fallback-then-converged" if self.fallback_iteration is not None \
                    else "converged"
                break
            recent = self.trace[self._mode_start:]
            if detect_oscillation([t.energy for t in recent], [t.moves for t in recent],
                                  cfg.oscillation_window, cfg.oscillation_tol):
                if self.mode == "sobolev":
                    self.mode = "l2"
                    self.fallback_iteration = self.iteration
                    self._mode_start = len(self.trace)
                else:
                    status = "oscillation-halt"
                    if prev_e < self._energy:
                        self.labels[...] = prev_labels
                        self._refresh()
                        self._energy = prev_e
                    break
        final = self.evaluate()
        self._energy = final.total
        regions = int(np.count_nonzero(self.stats.count[1:] > 0))
        return status, final, regions
