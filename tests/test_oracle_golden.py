"""Pin the CPU oracle against fixtures produced by the reference itself.

Every fixture under tests/golden/ was made by tests/golden/make_golden.py,
which runs the unmodified reference (rcseg) in the build container.  The
oracle must reproduce them bit for bit (Gaussian models; Poisson on
integer-valued data with the same numpy ``log``) — otherwise it cannot serve
as the checker of the CUDA path.
"""
import numpy as np
import pytest

from oracle import rc_oracle as O
from tests.conftest import golden


def test_kernel_values_and_known_answers():
    g = golden("kernel.npz")
    k = 0
    while f"E{k}" in g:
        E, eps = g[f"E{k}"]
        assert np.array_equal(O.weight_table(E, eps), g[f"w{k}"])
        k += 1
    # reference known answers (test_sobolev.py:58-64)
    assert abs(O.kernel_eval(0.0, 12.0, 1 / 24) - 0.25) < 1e-12
    assert abs(O.kernel_eval(3.0, 12.0, 1 / 24) - 0.0625) < 1e-12
    assert abs(O.kernel_eval(6.0 - 1e-13, 12.0, 1 / 24)) < 1e-12
    with pytest.raises(ValueError):
        O.kernel_eval(6.1, 12.0, 1 / 24)


def test_sobolev_filter_bitwise():
    g = golden("sobolev.npz")
    for k in range(int(g["n"][0])):
        got = O.sobolev_filter(g[f"c{k}"], g[f"o{k}"], g[f"m{k}"], g[f"r{k}"], float(g[f"E{k}"][0]))
        assert np.array_equal(got, g[f"y{k}"]), k
        assert O.pair_count(g[f"c{k}"], float(g[f"E{k}"][0])) == int(g[f"p{k}"][0])


def test_sobolev_known_answers():
    # single particle -> 0.5 (test_sobolev.py:137-144)
    out = O.sobolev_filter(np.array([[4, 4]]), [1], [0], [2.0])
    assert abs(out[0] - 0.5) < 1e-12
    # empty opposing side contributes zero (test_sobolev.py:207-223)
    c = np.array([[0, 0], [2, 0]])
    a = O.sobolev_filter(c, [1, 1], [2, 2], [1.0, 3.0])
    b = O.sobolev_filter(c, [1, 1], [0, 0], [1.0, 3.0])
    assert np.array_equal(a, b)


def test_contour_particles():
    g = golden("contour.npz")
    for k in range(int(g["n"][0])):
        lab = g[f"l{k}"]
        conn = O.Conn(lab.ndim, bool(g[f"f{k}"][0]))
        xs, ow, cm = O.scan_particles(lab, conn)
        keys = np.stack([xs, cm], axis=1) if len(xs) else np.zeros((0, 2), np.int64)
        assert np.array_equal(keys, g[f"k{k}"]), k
        assert np.array_equal(ow, lab.ravel()[xs])


def test_energy_increments_and_totals():
    g = golden("energy.npz")
    for k in range(int(g["n"][0])):
        ps, pois, r, lam = g[f"cfg{k}"]
        region = "ps" if ps else "pc"
        noise = "poisson" if pois else "gauss"
        lab, img = g[f"lab{k}"], g[f"img{k}"]
        xs, ow, cm = g[f"xs{k}"], g[f"ow{k}"], g[f"cm{k}"]
        eng = O.OracleEngine(img, lab, region, noise, lam, int(r))
        de = eng.delta_ext(xs, ow, cm)
        assert np.array_equal(de, g[f"de{k}"]), (k, region, noise)
        assert np.array_equal(O.delta_internal_batch(lab, xs, ow, cm), g[f"di{k}"])
        ev = O.evaluate_total(lab, img, region, noise, lam, int(r))
        assert [ev.total, ev.external, ev.internal] == list(g[f"ev{k}"]), k


def test_admissibility_verdicts():
    g = golden("admissible.npz")
    for k in range(int(g["n"][0])):
        lab = g[f"l{k}"]
        conn = O.Conn(lab.ndim, bool(g[f"f{k}"][0]))
        for x, c, fu, va, ok in g[f"v{k}"]:
            got = O.admissible(lab, int(x), int(c), conn, bool(fu), bool(va))
            assert got == bool(ok), (k, x, c, fu, va)


def _engine_from_run(g):
    ps, pois, r, lam, E, eps, sob, grace, seed, fusion, vanish, budget = g["cfg"]
    cfg = O.OptimizerConfig(gradient="sobolev" if sob else "l2", vanish_grace=int(grace),
                            seed=int(seed), allow_fusion=bool(fusion), allow_vanish=bool(vanish),
                            move_budget=float(budget))
    return O.OracleEngine(g["image"], g["init"], "ps" if ps else "pc",
                          "poisson" if pois else "gauss", float(lam), int(r), float(E),
                          float(eps), cfg)


RUNS = ["pc2d", "pc2d_l2", "pc3d", "ps2d", "ps2d_gauss"]


@pytest.mark.parametrize("name", RUNS)
def test_engine_iterations_bitwise(name):
    g = golden(f"run_{name}.npz")
    eng = _engine_from_run(g)
    off = 0
    for it in range(len(g["moves"])):
        rec = eng.iterate()
        n = int(g["acc_len"][it])
        want = [tuple(int(v) for v in row) for row in g["acc"][off:off + n]]
        off += n
        assert rec.accepted == want, (name, it)
        if "labels" in g:
            assert np.array_equal(eng.labels, g["labels"][it]), (name, it)
        assert rec.energy == g["energy"][it], (name, it)
        assert rec.particles == g["particles"][it]
        assert rec.mode == str(g["mode"][it])


@pytest.mark.parametrize("name", ["full_pc2d", "full_ps2d"])
def test_engine_full_run_status(name):
    g = golden(f"run_{name}.npz")
    eng = _engine_from_run(g)
    eng.config.max_iterations = 300
    status, final, regions = eng.run()
    assert status == str(g["status"][0])
    assert len(eng.trace) == int(g["iterations"][0])
    fb = int(g["fallback"][0])
    assert (eng.fallback_iteration if eng.fallback_iteration is not None else -1) == fb
    assert [final.total, final.external, final.internal] == list(g["final"])
    assert regions == int(g["regions"][0])
    assert [t.energy for t in eng.trace] == list(g["energy"])
    assert np.array_equal(eng.labels, g["labels"][-1]) or status == "oscillation-halt"


@pytest.mark.slow
@pytest.mark.parametrize("name,iters", [("cfg2_small", 4), ("cfg1", 8)])
def test_engine_config_runs(name, iters):
    import hashlib
    g = golden(f"run_{name}.npz")
    eng = _engine_from_run(g)
    off = 0
    for it in range(min(iters, len(g["moves"]))):
        rec = eng.iterate()
        n = int(g["acc_len"][it])
        want = [tuple(int(v) for v in row) for row in g["acc"][off:off + n]]
        off += n
        assert rec.accepted == want, (name, it)
        h = hashlib.sha256(np.ascontiguousarray(eng.labels, np.int32).tobytes()).hexdigest()[:16]
        assert h == str(g["hashes"][it])
        assert rec.energy == g["energy"][it]


@pytest.mark.slow
@pytest.mark.parametrize("name,iters", [("cfg5_0", 3), ("cfg3", 1)])
def test_oracle_on_baseline_configs(name, iters):
    """The oracle port against the reference's own cfg5 / cfg3 runs (the
    scenes regenerate on the host: no Poisson noise, numpy + scipy only)."""
    import hashlib

    import scenes
    g = dict(golden(f"run_{name}.npz"))
    sc = scenes.cfg5_image(0) if name == "cfg5_0" else scenes.cfg3()
    assert hashlib.sha256(np.ascontiguousarray(sc.image).tobytes()).hexdigest()[:16] == \
        str(g["image_sha"][0])
    g["image"], g["init"] = sc.image, sc.labels
    eng = _engine_from_run(g)
    off = 0
    for it in range(iters):
        rec = eng.iterate()
        n = int(g["acc_len"][it])
        want = [tuple(int(v) for v in row) for row in g["acc"][off:off + n]]
        off += n
        assert rec.accepted == want, (name, it)
        h = hashlib.sha256(np.ascontiguousarray(eng.labels, np.int32).tobytes()).hexdigest()[:16]
        assert h == str(g["hashes"][it])
        assert rec.energy == g["energy"][it]
