"""Integer-image fast paths against the general kernels they replace.

* ``k_fields_band3d_int`` (prefix-sum ball runs, 16x8x8 tiles; band refresh,
  full rebuild and K5 site-record maintenance) against ``k_fields_band3d`` /
  ``k_fields_tile3d`` + the per-iteration ``k_pack_sites`` pass
  (``RCB_NO_BANDINT=1``, ``RCB_PACK_ALWAYS=1``);
* the 5^3 window tier of the dataflow acceptance against the 9^3 window alone
  (``RCB_DF_WIN5=0``).

Both engines run the same seeded 3-D PS/Poisson scene whose sides are NOT
multiples of the tile extents (clipped tiles, halos across the lattice
faces) for several iterations, through a resync; accepted moves in order,
labels, particle counts and ledger energies must be identical (the fast
paths are exact, not approximate: integer sums in another order).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _scene(shape, seed, radius):
    """Two Poisson-noised blobs on a ramp, integer counts < 4096; bubbles as
    initial labels (several labels per tile)."""
    rng = np.random.default_rng(seed)
    nz, ny, nx = shape
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    mean = 4.0 + 6.0 * x / nx
    for c, r, v in (((nz * 0.35, ny * 0.4, nx * 0.3), min(shape) * 0.28, 25.0),
                    ((nz * 0.65, ny * 0.6, nx * 0.7), min(shape) * 0.22, 18.0)):
        d2 = (z - c[0]) ** 2 + (y - c[1]) ** 2 + (x - c[2]) ** 2
        mean = np.where(d2 < r * r, v, mean)
    img = rng.poisson(mean).astype(np.float64)
    lab = np.zeros(shape, np.int32)
    k = 1
    step = max(8, min(shape) // 2)
    for cz in range(step // 2, nz, step):
        for cy in range(step // 2, ny, step):
            for cx in range(step // 2, nx, step):
                d2 = (z - cz) ** 2 + (y - cy) ** 2 + (x - cx) ** 2
                lab[d2 < radius * radius] = k
                k += 1
    return img, lab


def _run(P, img, lab, smooth_radius, iters, env, gradient="sobolev"):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        eng = P.RegionCompetition(
            img, lab, P.EnergyConfig("ps", "poisson", 0.0, smooth_radius), P.SobolevParams(6.0),
            P.OptimizerConfig(gradient, vanish_grace=5, resync_every=3, drift_tolerance=1e-3))
        out = []
        for _ in range(iters):
            rec = eng.iterate()
            out.append((rec.moves, rec.particles, rec.energy,
                        np.asarray(eng.last_accepted).copy(), eng.labels.copy()))
        return out
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _same(a, b):
    assert len(a) == len(b)
    for it, (x, y) in enumerate(zip(a, b), 1):
        assert x[0] == y[0] and x[1] == y[1], f"iteration {it}: counts {x[:2]} vs {y[:2]}"
        assert np.array_equal(x[3], y[3]), f"iteration {it}: accepted moves differ"
        assert np.array_equal(x[4], y[4]), f"iteration {it}: labels differ"
        assert x[2] == y[2], f"iteration {it}: ledger {x[2]!r} vs {y[2]!r}"


@pytest.mark.parametrize("shape,R", [((23, 29, 37), 3), ((20, 41, 50), 4), ((9, 17, 33), 2)])
def test_int_band_refresh_equals_general_kernels(shape, R):
    import paper_1403_0240_b200 as P
    img, lab = _scene(shape, seed=7 + R, radius=4.5)
    fast = _run(P, img, lab, R, 7, {})
    slow = _run(P, img, lab, R, 7, {"RCB_NO_BANDINT": "1", "RCB_PACK_ALWAYS": "1"})
    assert sum(r[0] for r in fast) > 0
    _same(fast, slow)


def test_site_records_kept_current_equal_the_packing_pass():
    import paper_1403_0240_b200 as P
    img, lab = _scene((24, 40, 48), seed=3, radius=5.0)
    _same(_run(P, img, lab, 4, 6, {}), _run(P, img, lab, 4, 6, {"RCB_PACK_ALWAYS": "1"}))


def test_window5_tier_decides_like_the_9_window():
    import paper_1403_0240_b200 as P
    img, lab = _scene((32, 40, 48), seed=11, radius=6.0)
    a = _run(P, img, lab, 4, 6, {})
    b = _run(P, img, lab, 4, 6, {"RCB_DF_WIN5": "0"})
    _same(a, b)


def test_int_band_in_l2_mode():
    import paper_1403_0240_b200 as P
    img, lab = _scene((21, 30, 35), seed=5, radius=4.5)
    _same(_run(P, img, lab, 3, 4, {}, "l2"),
          _run(P, img, lab, 3, 4, {"RCB_NO_BANDINT": "1", "RCB_PACK_ALWAYS": "1"}, "l2"))
