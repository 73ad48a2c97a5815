"""Every BASELINE config pinned to runs of the REFERENCE itself.

Fixtures (tests/golden/make_golden.py ``big_runs``; the unmodified ``rcseg``
engine run in the build container, every accepted move captured in
acceptance order):

* ``run_cfg2_full``  cfg2 1024^2 PS/Poisson R=4, E=6, iterations 1-26
  (covers bench.py's timed window, iterations 6-25);
* ``run_cfg3``       cfg3 128^3 PC/Gauss, E=4, iterations 1-3;
* ``run_cfg4s``      cfg4' 128^3, 8 ellipsoids, bubbles:2:15, PS/Poisson R=4,
  E=6, iterations 1-6 (cfg4 itself needs a 1 TiB oracle);
* ``run_cfg5_{0..3}`` cfg5 images 0-3, 512^2 PC/Gauss, E=4, 50 iterations;
* ``run_cfg2s_l2`` / ``run_cfg4s_l2``  the scaled cfg2 (256^2) and cfg4' in l2
  mode: the PS d_tot < 0 gate of the dataflow acceptance (4 / 3 iterations).

The scenes are regenerated here by ``scenes.py`` through the DEVICE synth
pipeline (render, blur, poissonize); their sha-256 must equal the images the
reference consumed.  Contract per iteration: accepted moves in order and the
label hash bit-exact, particle and move counts exact, ledger energy bit-exact
for PC/Gauss and within rtol 1e-12 for Poisson (CUDA's and numpy's ``log``
may differ by an ulp).
"""
import hashlib

import numpy as np
import pytest

from tests.conftest import golden

pytestmark = pytest.mark.gpu


def sha(a, dtype=None):
    a = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype))
    return hashlib.sha256(a.tobytes()).hexdigest()[:16]


def _cfgs(P, g, drift):
    ps, pois, r, lam, E, eps, sob, grace, seed, fusion, vanish, budget = g["cfg"]
    ocfg = P.OptimizerConfig(gradient="sobolev" if sob else "l2", vanish_grace=int(grace),
                             seed=int(seed), allow_fusion=bool(fusion), allow_vanish=bool(vanish),
                             move_budget=float(budget), drift_tolerance=drift)
    ecfg = P.EnergyConfig("ps" if ps else "pc", "poisson" if pois else "gauss", float(lam),
                          int(r))
    return ecfg, P.SobolevParams(float(E), float(eps)), ocfg, bool(pois)


def _scene(name):
    import scenes
    if name == "cfg2s_l2":
        return scenes.cfg2_small()
    if name == "cfg4s_l2":
        return scenes.cfg4_small()
    if name == "cfg2_full":
        return scenes.cfg2()
    if name == "cfg3":
        return scenes.cfg3()
    if name == "cfg4s":
        return scenes.cfg4_small()
    return scenes.cfg5_image(int(name.split("_")[1]))


def _replay(eng, g, approx, name):
    off = 0
    for it in range(len(g["moves"])):
        rec = eng.iterate()
        n = int(g["acc_len"][it])
        got = eng.last_accepted
        want = g["acc"][off:off + n]
        off += n
        assert got.shape == want.shape and np.array_equal(got, want), \
            (name, it + 1, len(got), n)
        assert sha(eng.labels, np.int32) == str(g["hashes"][it]), (name, it + 1)
        assert rec.particles == int(g["particles"][it]), (name, it + 1)
        assert rec.moves == int(g["moves"][it]), (name, it + 1)
        want_e = float(g["energy"][it])
        if approx:
            assert abs(rec.energy - want_e) <= 1e-12 * abs(want_e), (name, it + 1, rec.energy,
                                                                     want_e)
        else:
            assert rec.energy == want_e, (name, it + 1, rec.energy, want_e)


@pytest.fixture(scope="module")
def P():
    import paper_1403_0240_b200 as P
    from paper_1403_0240_b200 import _lib
    if _lib.device_count() < 1:
        pytest.fail("no CUDA device visible to librcseg_b200")
    return P


@pytest.mark.parametrize("name", ["cfg2_full", "cfg3", "cfg4s", "cfg5_0", "cfg5_1", "cfg5_2",
                                  "cfg5_3", "cfg2s_l2", "cfg4s_l2"])
def test_config_vs_reference_run(P, name):
    g = golden(f"run_{name}.npz")
    sc = _scene(name)
    assert sha(sc.image) == str(g["image_sha"][0]), f"{name}: device scene != reference scene"
    assert sha(sc.labels, np.int32) == str(g["init_sha"][0]), name
    drift = 1e-3 if name in ("cfg2_full", "cfg4s", "cfg2s_l2", "cfg4s_l2") else 1e-6
    ecfg, scfg, ocfg, approx = _cfgs(P, g, drift)
    eng = P.RegionCompetition(sc.image, sc.labels, ecfg, scfg, ocfg)
    _replay(eng, g, approx, name)


def test_cfg5_batch_vs_reference_runs(P):
    """cfg5 through the batched path (several engines in flight): images 0-3
    after 50 iterations equal the reference's label hashes and energies."""
    from paper_1403_0240_b200.batch import run_batch
    gs = [golden(f"run_cfg5_{i}.npz") for i in range(4)]
    scs = [_scene(f"cfg5_{i}") for i in range(4)]
    ecfg, scfg, ocfg, _ = _cfgs(P, gs[0], 1e-6)
    ocfg.max_iterations = 50
    out = dict(run_batch([s.image for s in scs], [s.labels for s in scs], ecfg, scfg, ocfg,
                         rank=0, world=1, in_flight=4))
    for i, g in enumerate(gs):
        res = out[i]
        n = min(len(res.trace), len(g["moves"]))
        assert [r.moves for r in res.trace[:n]] == [int(m) for m in g["moves"][:n]], i
        assert [r.energy for r in res.trace[:n]] == [float(e) for e in g["energy"][:n]], i
        if len(res.trace) == len(g["moves"]):
            assert sha(res.labels, np.int32) == str(g["hashes"][-1]), i
