"""fp32 mode (BASELINE north_star): gradients within rtol 1e-4 of the fp64
path, final labels Dice >= 0.999.

The tolerance on a gradient value g (raw increment or Sobolev output) is
|g32 - g64| <= 1e-4 |g64| + 1e-5 * mean|g64|: the absolute floor is the
single-precision rounding of the O(mean|g|) terms that make up g, which
matters when g itself is a near-cancellation (e.g. equal same/opposite means).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pair(P, sc, gradient, iters=1, **kw):
    ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
    out = []
    for prec in ("fp64", "fp32"):
        eng = P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale),
                                  P.OptimizerConfig(gradient, precision=prec,
                                                    vanish_grace=sc.vanish_grace, **kw))
        for _ in range(iters):
            eng.iterate()
        out.append(eng)
    return out


def _close(g32, g64):
    floor = 1e-5 * max(np.mean(np.abs(g64)), 1e-300)
    return np.abs(g32 - g64) <= 1e-4 * np.abs(g64) + floor


@pytest.mark.parametrize("name", ["cfg1", "cfg2_small", "cfg3_small"])
@pytest.mark.parametrize("gradient", ["l2", "sobolev"])
def test_fp32_gradients(name, gradient):
    import paper_1403_0240_b200 as P
    import scenes
    sc = scenes.cfg3(n=40) if name == "cfg3_small" else getattr(scenes, name)()
    e64, e32 = _pair(P, sc, gradient)
    x64, _, c64, r64 = e64.last_candidates
    x32, _, c32, r32 = e32.last_candidates
    assert np.array_equal(x64, x32) and np.array_equal(c64, c32)
    ok = _close(r32, r64)
    assert ok.mean() == 1.0, (name, gradient, ok.mean(), np.max(np.abs(r32 - r64)))


def _dice(a, b):
    labs = [l for l in np.union1d(np.unique(a), np.unique(b)) if l > 0]
    d = []
    for l in labs:
        A, B = a == l, b == l
        s = A.sum() + B.sum()
        d.append(1.0 if s == 0 else 2.0 * np.logical_and(A, B).sum() / s)
    return float(np.mean(d)) if d else 1.0


@pytest.mark.parametrize("name,iters", [("cfg1", 50), ("cfg2_small", 30)])
def test_fp32_final_labels_dice(name, iters):
    import paper_1403_0240_b200 as P
    import scenes
    sc = getattr(scenes, name)()
    ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
    res = {}
    for prec in ("fp64", "fp32"):
        res[prec] = P.run(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale),
                          P.OptimizerConfig("sobolev", precision=prec, max_iterations=iters,
                                            vanish_grace=sc.vanish_grace, drift_tolerance=1e-3))
    dice = _dice(res["fp32"].labels, res["fp64"].labels)
    assert dice >= 0.999, dice
