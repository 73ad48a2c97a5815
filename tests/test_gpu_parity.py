"""CUDA path vs the golden fixtures (made by the reference) and the oracle.

Contracts (BASELINE.json north_star):
* integer work (particles, ΔE_int, accepted moves, labels): bit-exact;
* fp64 Gaussian PC increments, Sobolev sums, region statistics, ledger: bit-exact;
* Poisson (``log``) and PS-on-float-data quantities: rtol 1e-12
  (RTOL below), because CUDA's and numpy's ``log`` may differ by 1 ulp and
  the own-label PS fields sum float data in a different order.
"""
import hashlib

import numpy as np
import pytest

from oracle import rc_oracle as O
from tests.conftest import golden

pytestmark = pytest.mark.gpu
RTOL = 1e-12


@pytest.fixture(scope="module")
def P():
    import paper_1403_0240_b200 as P
    from paper_1403_0240_b200 import _lib
    if _lib.device_count() < 1:
        pytest.fail("no CUDA device visible to librcseg_b200")
    return P


def close(a, b, rtol=RTOL, atol=0.0):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= atol + rtol * np.abs(b))


# ---- function level -------------------------------------------------------

def test_sobolev_filter_bitwise_vs_reference(P):
    g = golden("sobolev.npz")
    for k in range(int(g["n"][0])):
        E = float(g[f"E{k}"][0])
        out, pairs = P.sobolev_filter(g[f"c{k}"], g[f"o{k}"], g[f"m{k}"], g[f"r{k}"],
                                      P.SobolevParams(E), return_pairs=True)
        assert np.array_equal(out, g[f"y{k}"]), k
        assert pairs == int(g[f"p{k}"][0]), k


def test_sobolev_known_answers_and_properties(P):
    p = P.SobolevParams()
    out = P.sobolev_filter(np.array([[4, 4]]), np.array([1]), np.array([0]), np.array([2.0]), p)
    assert abs(out[0] - 0.5) < 1e-12
    rng = np.random.default_rng(23)
    coords = rng.integers(0, 30, size=(150, 2))
    ow = rng.integers(0, 3, size=150)
    cm = rng.integers(0, 3, size=150)
    raw = rng.normal(size=150)
    base = P.sobolev_filter(coords, ow, cm, raw, p)
    perm = rng.permutation(150)
    assert np.array_equal(P.sobolev_filter(coords[perm], ow[perm], cm[perm], raw[perm], p),
                          base[perm])
    # locality: far particles cannot change near outputs, bit for bit
    near = rng.integers(0, 10, size=(60, 2))
    far = rng.integers(100, 110, size=(40, 2))
    allc = np.vstack([near, far])
    ow = rng.integers(0, 3, size=100)
    cm = rng.integers(0, 3, size=100)
    raw = rng.normal(size=100)
    full = P.sobolev_filter(allc, ow, cm, raw, p)
    alone = P.sobolev_filter(near, ow[:60], cm[:60], raw[:60], p)
    assert np.array_equal(full[:60], alone)
    # empty input
    assert P.sobolev_filter(np.zeros((0, 2), np.int64), [], [], [], p).size == 0


def test_scan_contour_vs_reference(P):
    g = golden("contour.npz")
    from paper_1403_0240_b200.contour import scan_particles
    for k in range(int(g["n"][0])):
        lab = g[f"l{k}"]
        fg = {2: (8, 4), 3: (26, 6)}[lab.ndim][0 if g[f"f{k}"][0] else 1]
        xs, ow, cm = scan_particles(lab, P.Connectivity(lab.ndim, fg))
        keys = np.stack([xs, cm], 1) if len(xs) else np.zeros((0, 2), np.int64)
        assert np.array_equal(keys, g[f"k{k}"]), k
        assert np.array_equal(ow, lab.ravel()[xs])


@pytest.mark.parametrize("shape,nlab", [((131, 257), 7), ((1, 300), 3), ((300, 1), 3),
                                         ((23, 37, 41), 9), ((1, 1, 50), 2), ((17, 1, 19), 5)])
def test_scan_contour_face_path_vs_oracle(P, shape, nlab):
    """The face-adjacency contour kernels (full_fg, 32-bit coordinates,
    register sort) against the oracle on dense multi-label lattices, where
    most sites have several distinct competitors, and on degenerate extents."""
    from paper_1403_0240_b200.contour import scan_particles
    rng = np.random.default_rng(sum(shape) * 31 + nlab)
    lab = rng.integers(0, nlab, size=shape).astype(np.int32)
    lab[tuple(slice(0, max(1, d // 3)) for d in shape)] = nlab + 4  # a flat block
    xs, ow, cm = scan_particles(lab, P.Connectivity(lab.ndim, 8 if lab.ndim == 2 else 26))
    oxs, oow, ocm = O.scan_particles(lab, O.Conn(lab.ndim, True))
    assert np.array_equal(xs, oxs) and np.array_equal(ow, oow) and np.array_equal(cm, ocm)


def _term_magnitude(lab, img, xs, ow, cm, ps, pois, r):
    """Sum of |terms| of each particle's increment (energy.py:129-143 PC,
    :326-372 PS): the scale its fp64 rounding is relative to."""
    noise = "poisson" if pois else "gauss"
    img = np.asarray(img, np.float64)
    flat = img.ravel()
    if not ps:
        st = O.Stats(lab, img, int(lab.max()) + 1)
        def g(n, s_, q):
            return np.abs(q) + np.abs(s_ * s_ / np.maximum(n, 1)) if not pois else \
                np.abs(s_) + np.abs(s_ * np.log(np.maximum(s_ / np.maximum(n, 1), 1e-8)))
        na, sa, qa = st.count[ow].astype(float), st.total[ow], st.total_sq[ow]
        nb, sb, qb = st.count[cm].astype(float), st.total[cm], st.total_sq[cm]
        return g(na, sa, qa) + g(nb, sb, qb) + g(na - 1, sa, qa) + g(nb + 1, sb, qb)
    C, S = O.smooth_fields(lab, img, r, int(lab.max()) + 1)
    C2, S2 = C.reshape(C.shape[0], -1), S.reshape(S.shape[0], -1)
    offs = O.ball_offsets(lab.ndim, r)
    out = np.zeros(len(xs))
    for i, (x, a, b) in enumerate(zip(xs, ow, cm)):
        c0 = np.array(np.unravel_index(int(x), lab.shape))
        tot = 0.0
        for off in offs:
            y = c0 + off
            if np.any(y < 0) or np.any(y >= lab.shape):
                continue
            fy = int(np.ravel_multi_index(tuple(y), lab.shape))
            l = int(lab.ravel()[fy])
            if l not in (a, b):
                continue
            for ll in (a, b):
                c, s_ = C2[ll, fy], S2[ll, fy]
                for cc, ss in ((c, s_), (c - 1, s_ - flat[x]), (c + 1, s_ + flat[x])):
                    if cc > 0:
                        tot += abs(float(O.rho(flat[fy], ss / cc, noise)))
        out[i] = tot
    return out


def test_energy_increments_vs_reference(P):
    g = golden("energy.npz")
    for k in range(int(g["n"][0])):
        ps, pois, r, lam = g[f"cfg{k}"]
        cfg = P.EnergyConfig("ps" if ps else "pc", "poisson" if pois else "gauss", float(lam),
                             int(r))
        lab, img = g[f"lab{k}"], g[f"img{k}"]
        xs, ow, cm = g[f"xs{k}"], g[f"ow{k}"], g[f"cm{k}"]
        model = P.EnergyModel(img, lab, cfg)
        de = model.delta_external_batch(xs, ow, cm)
        if not ps and not pois:
            assert np.array_equal(de, g[f"de{k}"]), k
        else:
            # rtol 1e-12 per element (north_star) plus the increment's own
            # conditioning floor: 4 ulp of the sum of the absolute terms it is
            # formed from (CUDA's and numpy's log differ by <= 1 ulp; float
            # PS fields are summed in another order than the reference's
            # cumulative-sum windows, 1 ulp of each field)
            ref = g[f"de{k}"]
            floor = 4.0 * 2.0 ** -52 * _term_magnitude(lab, img, xs, ow, cm, bool(ps),
                                                        bool(pois), int(r))
            err = np.abs(de - ref)
            assert np.all(err <= 1e-12 * np.abs(ref) + floor), (k, float(np.max(err - 1e-12 * np.abs(ref) - floor)))
            assert np.mean(err <= 1e-12 * np.abs(ref)) > 0.9, k  # the floor is the exception
        assert np.array_equal(P.delta_internal_batch(lab, xs, ow, cm), g[f"di{k}"])
        ev = P.evaluate_total(lab, img, cfg)
        want = g[f"ev{k}"]
        assert ev.internal == int(want[2])
        if not ps and not pois:
            assert ev.external == want[1], k
        else:
            assert close(ev.external, want[1]), (k, ev.external, want[1])


def test_stats_rebuild_bitwise(P):
    rng = np.random.default_rng(5)
    lab = rng.integers(0, 7, size=(61, 67)).astype(np.int32)
    img = rng.normal(size=lab.shape)
    t = P.StatsTable.from_labels(lab, img)
    o = O.Stats(lab, img, 7)
    assert np.array_equal(t.count, o.count)
    assert np.array_equal(t.total, o.total)
    assert np.array_equal(t.total_sq, o.total_sq)


def test_evaluate_total_exact_rounding(P):
    # a sum that naive fp64 accumulation gets wrong: fsum semantics required
    lab = np.zeros((2, 3), np.int32)
    lab[0, :] = [0, 1, 2]
    lab[1, :] = [3, 4, 5]
    img = np.array([[1e16, 1.0, -1e16], [1.0, 3.0, 2.0]])
    for region, noise in (("pc", "gauss"), ("ps", "gauss")):
        cfg = P.EnergyConfig(region, noise, smooth_radius=1)
        want = O.evaluate_total(lab, img, region, noise, 0.0, 1)
        got = P.evaluate_total(lab, img, cfg)
        assert got.external == want.external


# ---- the engine -------------------------------------------------------------

def _engine(P, g):
    ps, pois, r, lam, E, eps, sob, grace, seed, fusion, vanish, budget = g["cfg"]
    cfg = P.OptimizerConfig(gradient="sobolev" if sob else "l2", vanish_grace=int(grace),
                            seed=int(seed), allow_fusion=bool(fusion), allow_vanish=bool(vanish),
                            move_budget=float(budget), max_iterations=300)
    ecfg = P.EnergyConfig("ps" if ps else "pc", "poisson" if pois else "gauss", float(lam),
                          int(r))
    return P.RegionCompetition(g["image"], g["init"], ecfg, P.SobolevParams(float(E), float(eps)),
                               cfg), bool(ps or pois)


@pytest.mark.parametrize("name", ["pc2d", "pc2d_l2", "pc3d", "ps2d", "ps2d_gauss"])
def test_engine_iterations_vs_reference(P, name):
    g = golden(f"run_{name}.npz")
    eng, approx = _engine(P, g)
    off = 0
    for it in range(len(g["moves"])):
        rec = eng.iterate()
        n = int(g["acc_len"][it])
        want = g["acc"][off:off + n]
        off += n
        got = eng.last_accepted
        assert np.array_equal(got, want), (name, it, len(got), n)
        if "labels" in g:
            assert np.array_equal(eng.labels, g["labels"][it]), (name, it)
        assert rec.particles == int(g["particles"][it])
        assert rec.moves == int(g["moves"][it])
        if approx:
            assert close(rec.energy, g["energy"][it], 1e-12), (name, it)
        else:
            assert rec.energy == g["energy"][it], (name, it)


@pytest.mark.parametrize("name", ["full_pc2d", "full_ps2d"])
def test_engine_full_run_vs_reference(P, name):
    g = golden(f"run_{name}.npz")
    eng, approx = _engine(P, g)
    res = eng.run()
    assert res.status == str(g["status"][0])
    assert res.iterations == int(g["iterations"][0])
    fb = -1 if res.fallback_iteration is None else res.fallback_iteration
    assert fb == int(g["fallback"][0])
    assert res.region_count == int(g["regions"][0])
    assert res.final_energy.internal == int(g["final"][2])
    assert close(res.final_energy.total, g["final"][0], 1e-12)
    if not approx:
        assert [r.energy for r in res.trace] == list(g["energy"])


@pytest.mark.parametrize("name,iters", [("cfg1", 50), ("cfg2_small", 4)])
def test_engine_config_runs_vs_reference(P, name, iters):
    g = golden(f"run_{name}.npz")
    eng, approx = _engine(P, g)
    off = 0
    for it in range(iters):
        rec = eng.iterate()
        n = int(g["acc_len"][it])
        assert np.array_equal(eng.last_accepted, g["acc"][off:off + n]), (name, it)
        off += n
        h = hashlib.sha256(np.ascontiguousarray(eng.labels, np.int32).tobytes()).hexdigest()[:16]
        assert h == str(g["hashes"][it]), (name, it)
        if approx:
            assert close(rec.energy, g["energy"][it], 1e-12)
        else:
            assert rec.energy == g["energy"][it], (name, it)


def test_engine_candidates_match_oracle(P):
    """last_candidates (particles and rank values) against the oracle's
    particle set and filtered ranks on the same raster."""
    g = golden("run_pc2d.npz")
    eng, _ = _engine(P, g)
    o = O.OracleEngine(g["image"], g["init"], "pc", "gauss", 0.0, 8, 4.0)
    for it in range(5):
        eng.iterate()
        o.iterate()
        xs, ow, cm, rk = eng.last_candidates
        ox, oo, oc, orank = o.last_candidates
        assert np.array_equal(xs, ox) and np.array_equal(ow, oo) and np.array_equal(cm, oc)
        assert np.array_equal(rk, orank)


@pytest.mark.parametrize("mode", ["dataflow", "rounds"])
def test_rank_ties_noiseless_vs_oracle(P, mode, monkeypatch):
    """A noiseless piecewise-constant image with straight edges gives long
    runs of exactly equal rank values, so the acceptance order inside each
    run comes from the tie keys and particle order alone (lexsort's later
    keys): accepted moves and labels must match the oracle exactly."""
    monkeypatch.setenv("RCB_ACCEPT", mode)
    img = np.zeros((96, 96))
    img[20:70, 16:60] = 1.0
    img[50:90, 50:92] = 0.5
    lab = np.zeros((96, 96), np.int32)
    lab[8:88, 8:88] = 1
    lab[40:60, 40:60] = 2
    cfg = P.OptimizerConfig("sobolev")
    eng = P.RegionCompetition(img, lab, P.EnergyConfig("pc", "gauss"), P.SobolevParams(4.0), cfg)
    o = O.OracleEngine(img, lab, "pc", "gauss", 0.0, 8, 4.0)
    longest = 0
    for it in range(8):
        rec = eng.iterate()
        orec = o.iterate()
        rk = eng.last_candidates[3]
        _, cnt = np.unique(rk[rk < 0], return_counts=True)
        longest = max(longest, int(cnt.max()) if cnt.size else 0)
        want = np.asarray(orec.accepted, np.int64).reshape(-1, 3)
        assert np.array_equal(eng.last_accepted, want), (mode, it)
        assert np.array_equal(eng.labels, o.labels), (mode, it)
        assert rec.energy == orec.energy, (mode, it)
    assert longest > 32  # exercises the long-run (block bitonic) fix-up too


@pytest.mark.parametrize("gradient", ["l2", "sobolev"])
def test_rank_tie_run_beyond_block_sort(P, gradient):
    """One run of > 4096 exactly equal rank values (a straight 6000-pixel
    edge of a noiseless two-level image): the block merge sort of K7 must
    give lexsort's (rank, tie, x, comp) order -- accepted moves in order and
    labels equal to the oracle's."""
    img = np.zeros((12, 6000))
    img[:8] = 1.0
    lab = np.zeros((12, 6000), np.int32)
    lab[:4] = 1
    cfg = P.OptimizerConfig(gradient)
    eng = P.RegionCompetition(img, lab, P.EnergyConfig("pc", "gauss"), P.SobolevParams(4.0), cfg)
    o = O.OracleEngine(img, lab, "pc", "gauss", 0.0, 8, 4.0,
                       config=O.OptimizerConfig(gradient))
    longest = 0
    for it in range(3):
        rec = eng.iterate()
        orec = o.iterate()
        rk = eng.last_candidates[3]
        _, cnt = np.unique(rk[rk < 0], return_counts=True)
        longest = max(longest, int(cnt.max()) if cnt.size else 0)
        want = np.asarray(orec.accepted, np.int64).reshape(-1, 3)
        assert np.array_equal(eng.last_accepted, want), (gradient, it)
        assert np.array_equal(eng.labels, o.labels), (gradient, it)
        assert rec.energy == orec.energy, (gradient, it)
    assert longest > 4096


def test_engine_invariants_at_full_cfg2_size(P):
    """Size-independent properties on the 1024^2 PS-Poisson config: the
    device contour equals a fresh scan, the ledger agrees with the from-scratch
    energy, no region is split, moves never exceed the candidates."""
    import scenes
    from scipy import ndimage
    sc = scenes.cfg2()
    cfg = P.OptimizerConfig("sobolev", vanish_grace=5)
    ecfg = P.EnergyConfig("ps", "poisson", smooth_radius=4)
    eng = P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(6.0), cfg)
    conn = P.Connectivity.default(2)
    for it in range(3):
        rec = eng.iterate()
        assert 0 < rec.moves <= eng.last_negative
        lab = eng.labels
        xs, _, cs = O.scan_particles(lab, O.Conn(2))
        assert rec.particles == len(xs)
        ev = eng._evaluate().total
        assert abs(ev - rec.energy) <= 1e-6 * max(1.0, abs(ev))
    lab = eng.labels
    for l in np.unique(lab):
        if l > 0:
            assert ndimage.label(lab == l, structure=conn.fg_structure)[1] == 1


@pytest.mark.parametrize("which", ["cfg2", "cfg1", "cfg3_small", "cfg4_small"])
def test_parallel_acceptance_equals_sequential(P, which, monkeypatch):
    """K8 v3 (dataflow) and K8 v2 (cooperative rounds) against K8 v1 (one
    thread, the literal sequential greedy) on the same inputs: accepted moves
    in order, labels and ledger must be identical.  The dataflow runs cover
    each topology-test tier: the bounding-box map BFS (default), the hash
    BFS (box tier off), the large global-memory box tier (3-D, hash capped
    at 8 sites) and the grid-wide union-find assist jobs (hash capped, large
    tier off)."""
    import scenes
    if which == "cfg2":
        sc, iters = scenes.cfg2(), 3
    elif which == "cfg1":
        sc, iters = scenes.cfg1(), 6
    elif which == "cfg3_small":
        sc, iters = scenes.cfg3(n=48), 3
    else:
        sc, iters = scenes.cfg4(n=64, n_obj=8, per_axis=2), 3
    ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
    ocfg = P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace)
    runs = []
    for force, mode, cap, box, big in (("0", "dataflow", "0", "-1", "1"),
                                       ("0", "rounds", "0", "-1", "1"),
                                       ("1", "dataflow", "0", "-1", "1"),
                                       ("0", "dataflow", "0", "0", "1"),
                                       ("0", "dataflow", "8", "0", "1"),
                                       ("0", "dataflow", "8", "0", "0")):
        monkeypatch.setenv("RCB_FORCE_SEQUENTIAL", force)
        monkeypatch.setenv("RCB_ACCEPT", mode)
        monkeypatch.setenv("RCB_DF_MAXINSERT", cap)
        monkeypatch.setenv("RCB_DF_BOXCAP", box)
        monkeypatch.setenv("RCB_DF_BIGBOX", big)
        eng = P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale), ocfg)
        out = []
        for _ in range(iters):
            rec = eng.iterate()
            out.append((rec.moves, rec.energy, eng.last_accepted.copy(), eng.labels))
        runs.append(out)
    # 3-D PS and 2-D PS/Poisson: the dataflow/rounds kernels keep the ledger
    # with the exact band change per iteration, the sequential kernel with
    # per-move terms
    band = sc.region == "ps" and (sc.image.ndim == 3 or sc.noise == "poisson")
    for other in runs[1:]:
        for it, (a, b) in enumerate(zip(runs[0], other)):
            assert a[0] == b[0], (which, it)
            assert np.array_equal(a[2], b[2]), (which, it)
            assert np.array_equal(a[3], b[3]), (which, it)
            if band:
                assert close(a[1], b[1]), (which, it, a[1], b[1])
            else:
                assert a[1] == b[1], (which, it, a[1], b[1])


def test_ps3d_band_ledger_vs_oracle(P):
    """3-D PS/Poisson: accepted moves and labels bit-exact against the oracle,
    the ledger (exact band change per iteration) within rtol 1e-12."""
    import scenes
    rng = np.random.default_rng(11)
    shape = (24, 28, 32)
    img = np.full(shape, 4.0)
    scenes._paint(img, (12, 14, 16), (7, 9, 8), 12.0)
    scenes._paint(img, (6, 8, 24), (4, 5, 4), 20.0)
    img = rng.poisson(img).astype(np.float32)
    lab = scenes.bubbles(shape, 2, 5.0)
    cfg = P.OptimizerConfig("sobolev", vanish_grace=5)
    eng = P.RegionCompetition(img, lab, P.EnergyConfig("ps", "poisson", smooth_radius=3),
                              P.SobolevParams(6.0), cfg)
    ocfg = O.OptimizerConfig("sobolev", vanish_grace=5)
    o = O.OracleEngine(img, lab, "ps", "poisson", 0.0, 3, 6.0, config=ocfg)
    for it in range(4):
        rec = eng.iterate()
        orec = o.iterate()
        want = np.asarray(orec.accepted, np.int64).reshape(-1, 3)
        assert np.array_equal(eng.last_accepted, want), it
        assert np.array_equal(eng.labels, o.labels), it
        assert close(rec.energy, orec.energy), (it, rec.energy, orec.energy)


def _adversarial_sequences():
    rng = np.random.default_rng(77)
    seqs = [
        rng.normal(size=20000),                                  # sign changes, small binades
        rng.poisson(6.0, size=30000).astype(np.float64),          # integers (exact)
        np.concatenate([[2.0 ** 53], np.ones(3000), [3.0] * 500, [-1.0] * 700]),  # ties at u=2
        np.concatenate([[2.0 ** 52 + 1.0], np.full(2000, 0.5), np.full(2000, 1.5)]),  # ties, u=1
        np.cumprod(np.full(600, 1.07)) * rng.choice([-1, 1], 600),  # binade sweeps
        np.concatenate([[-0.0, 0.0, -0.0], rng.normal(size=50), [1e300, -1e300], rng.normal(size=50)]),
        np.tile([1e16, 1.0, -1e16, 2.0 ** -30], 2000),
        rng.normal(size=5000) * 10.0 ** rng.integers(-20, 20, size=5000),
    ]
    return seqs


def test_ordered_sum_exact_vs_sequential(P):
    """The parallel replay of s = fl(s + v) (stats rebuild, label chains,
    ledger) must equal numpy's sequential bincount accumulation bit for bit."""
    for k, seq in enumerate(_adversarial_sequences()):
        img = np.ascontiguousarray(seq, np.float64).reshape(1, -1)
        lab = np.zeros(img.shape, np.int32)
        lab[0, ::7] = 1  # a second interleaved label
        t = P.StatsTable.from_labels(lab, img)
        o = O.Stats(lab, img, 2)
        assert np.array_equal(t.count, o.count), k
        assert np.array_equal(t.total, o.total, equal_nan=True), (k, t.total, o.total)
        assert np.array_equal(t.total_sq, o.total_sq, equal_nan=True), (k, t.total_sq, o.total_sq)


@pytest.mark.parametrize("cap,box,iters", [("0", "-1", 30), ("8", "0", 12)])
def test_deferred_registry_equals_full_union_find(P, monkeypatch, cap, box, iters):
    """Dataflow assist jobs through the deferred-candidate registry (one
    union-find of a minus the registered sites, brought forward by scans,
    queried per candidate on the contracted graph) against one full
    union-find per deferred candidate: identical moves in order, labels and
    ledger on cfg3 (64^3, the stage where tubes join the spheres), both with
    the default tiers and with most non-simple candidates forced to defer."""
    import scenes
    sc = scenes.cfg3(n=64)
    ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
    ocfg = P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace)
    monkeypatch.setenv("RCB_DF_MAXINSERT", cap)
    monkeypatch.setenv("RCB_DF_BOXCAP", box)
    monkeypatch.setenv("RCB_DF_BIGBOX", "0")  # every overflow defers (exercise the jobs)
    runs, deferred = [], []
    for q in ("1", "0"):
        monkeypatch.setenv("RCB_DF_QJOB", q)
        eng = P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale), ocfg)
        out, dsum = [], 0
        for _ in range(iters):
            rec = eng.iterate()
            dsum += eng.counters()["deferred"]
            out.append((rec.moves, rec.energy, eng.last_accepted.copy()))
        out.append(eng.labels)
        runs.append(out)
        deferred.append(dsum)
    assert min(deferred) > 0  # (a timing-dependent count: BFS retries on pending sites)
    for it, (a, b) in enumerate(zip(runs[0][:-1], runs[1][:-1])):
        assert a[0] == b[0] and a[1] == b[1], it
        assert np.array_equal(a[2], b[2]), it
    assert np.array_equal(runs[0][-1], runs[1][-1])


@pytest.mark.parametrize("which,iters", [("cfg1", 8), ("cfg3_small", 5), ("cfg5_0", 6)])
def test_l2_dataflow_equals_sequential(P, monkeypatch, which, iters):
    """l2 mode (PC): the dataflow kernel with every label sequenced and the
    d_tot < 0 gate on running statistics against K8 v1 (one thread, the
    literal sequential greedy): moves in order, labels and ledger identical."""
    import scenes
    sc = {"cfg1": scenes.cfg1, "cfg3_small": lambda: scenes.cfg3(n=48),
          "cfg5_0": lambda: scenes.cfg5_image(0)}[which]()
    ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
    ocfg = P.OptimizerConfig("l2")
    runs = []
    for force in ("0", "1"):
        monkeypatch.setenv("RCB_FORCE_SEQUENTIAL", force)
        eng = P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale), ocfg)
        out = []
        for _ in range(iters):
            rec = eng.iterate()
            out.append((rec.moves, rec.energy, eng.last_accepted.copy(), eng.counters()["parallel"]))
        out.append(eng.labels)
        runs.append(out)
    assert all(r[3] == 1 for r in runs[0][:-1]) and all(r[3] == 0 for r in runs[1][:-1])
    for it, (a, b) in enumerate(zip(runs[0][:-1], runs[1][:-1])):
        assert a[0] == b[0] and a[1] == b[1], (which, it, a[0], b[0])
        assert np.array_equal(a[2], b[2]), (which, it)
    assert np.array_equal(runs[0][-1], runs[1][-1])


@pytest.mark.parametrize("which", ["cfg1", "cfg4_small"])
def test_dataflow_wide_site_words(P, monkeypatch, which):
    """The 27-bit-position / 10-bit-label site-word layout (used above 2^24
    candidates) decides exactly like the default layout."""
    import scenes
    sc = scenes.cfg1() if which == "cfg1" else scenes.cfg4(n=64, n_obj=8, per_axis=2)
    ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
    ocfg = P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace)
    runs = []
    for wide in ("0", "1"):
        monkeypatch.setenv("RCB_DF_WP27", wide)
        eng = P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale), ocfg)
        out = [(r.moves, r.energy, eng.last_accepted.copy()) for r in (eng.iterate() for _ in range(6))]
        runs.append((out, eng.labels))
    for (a, b) in zip(runs[0][0], runs[1][0]):
        assert a[0] == b[0] and a[1] == b[1] and np.array_equal(a[2], b[2])
    assert np.array_equal(runs[0][1], runs[1][1])


def test_engine_input_validation_on_device(P):
    """grid.py:24-39 / optimizer.py:100-101 semantics, checked on the device
    in rcb_engine_create: the same ValueErrors, and the label count."""
    img = np.full((20, 24), 2.0)
    lab = np.zeros((20, 24), np.int32)
    lab[5:12, 6:15] = 3
    ecfg = P.EnergyConfig("pc", "gauss")
    eng = P.RegionCompetition(img, lab, ecfg)
    assert eng.n_labels == 4
    bad = img.copy()
    bad[3, 4] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        P.RegionCompetition(bad, lab, ecfg)
    neg = lab.copy()
    neg[0, 0] = -1
    with pytest.raises(ValueError, match="negative labels"):
        P.RegionCompetition(img, neg, ecfg)
    with pytest.raises(ValueError, match="nonnegative"):
        P.RegionCompetition(img - 3.0, lab, P.EnergyConfig("pc", "poisson"))
    with pytest.raises(ValueError):
        P.RegionCompetition(img, lab.astype(np.float64), ecfg)


def test_ps_deferred_stats_chains(P, monkeypatch):
    """PS runs replay the per-label total / total_sq chains when the stats are
    read: identical to the eager chains before and after a resync, and to
    the oracle's sequential StatsTable updates."""
    import scenes
    sc = scenes.cfg2_small()
    ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
    ocfg = P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace, drift_tolerance=1e-3)
    out = []
    for d in ("1", "0"):
        monkeypatch.setenv("RCB_DEFER_STATS", d)
        eng = P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale), ocfg)
        snaps = []
        for it in range(13):
            eng.iterate()
            if it in (0, 6, 8, 12):
                st = eng.model.stats
                snaps.append((st.count.copy(), st.total.copy(), st.total_sq.copy()))
        out.append(snaps)
    for a, b in zip(out[0], out[1]):
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
    ref = O.OracleEngine(sc.image, sc.labels, "ps", "poisson", 0.0, sc.smooth_radius,
                         sc.length_scale, config=O.OptimizerConfig(vanish_grace=sc.vanish_grace,
                                                                   drift_tolerance=1e-3))
    for _ in range(7):
        ref.iterate()
    assert np.array_equal(out[0][1][0], ref.stats.count)
    assert np.array_equal(out[0][1][1], ref.stats.total)
    assert np.array_equal(out[0][1][2], ref.stats.total_sq)


@pytest.mark.parametrize("shape", [(72, 80), (20, 22, 24)])
def test_sobolev_site_kernel_multilabel_vs_oracle(P, shape):
    """w = 1 (E = 2): K6 is the warp-cooperative site-run kernel.  Touching
    bubbles make sites with 2-4 competitors (runs of equal px that cross warp
    edges, too): accepted moves, labels and ledger equal the oracle's."""
    import scenes
    rng = np.random.default_rng(31)
    per = 4 if len(shape) == 2 else 2
    lab = scenes.bubbles(shape, per, (shape[0] / per) * 0.62)
    img = rng.normal(0.0, 1.0, size=shape) + (lab % 3).astype(np.float64)
    eng = P.RegionCompetition(img, lab, P.EnergyConfig("pc", "gauss"), P.SobolevParams(2.0),
                              P.OptimizerConfig("sobolev"))
    o = O.OracleEngine(img, lab, "pc", "gauss", 0.0, 8, 2.0)
    for it in range(4):
        rec = eng.iterate()
        orec = o.iterate()
        want = np.asarray(orec.accepted, np.int64).reshape(-1, 3)
        assert np.array_equal(eng.last_accepted, want), it
        assert np.array_equal(eng.labels, o.labels), it
        assert rec.energy == orec.energy, it
        xs, ow, cm, rk = eng.last_candidates
        _, cnt = np.unique(xs, return_counts=True)
        assert cnt.max() >= 2


@pytest.mark.parametrize("flipcap", ["default", "0"])
@pytest.mark.parametrize("which,iters", [("ps2d", 4), ("ps3d", 3)])
def test_ps_l2_dataflow_equals_sequential(P, monkeypatch, which, iters, flipcap):
    """l2 mode (PS/Poisson): the dataflow kernel's d_tot < 0 gate on own-label
    fields corrected by the earlier flips within 2R, against K8 v1 (one
    thread, incremental fields): moves in order, labels and ledger identical."""
    import scenes
    if which == "ps2d":
        sc = scenes.cfg2_small(n=128)
    else:
        sc = scenes.cfg4(n=40, n_obj=5, per_axis=2, radius=9.0)
    ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
    ocfg = P.OptimizerConfig("l2", vanish_grace=sc.vanish_grace, drift_tolerance=1e-3)
    if flipcap != "default":  # every field from the view-label bitmaps (dense flips)
        monkeypatch.setenv("RCB_PS_L2_FLIPCAP", flipcap)
    runs = []
    for mode in ("df", "seq"):
        monkeypatch.setenv("RCB_PS_L2", mode)
        eng = P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale), ocfg)
        out = []
        for _ in range(iters):
            rec = eng.iterate()
            out.append((rec.moves, rec.energy, eng.last_accepted.copy(), eng.counters()["parallel"]))
        out.append(eng.labels)
        runs.append(out)
    assert all(r[3] == 1 for r in runs[0][:-1]) and all(r[3] == 0 for r in runs[1][:-1])
    for it, (a, b) in enumerate(zip(runs[0][:-1], runs[1][:-1])):
        assert a[0] == b[0], (which, it, a[0], b[0])
        assert np.array_equal(a[2], b[2]), (which, it)
        # 3-D PS keeps the exact band ledger (K8 v1 sums d_tot in order): the
        # two ledgers agree to rounding, the moves and labels bit for bit
        assert abs(a[1] - b[1]) <= 1e-12 * abs(b[1]), (which, it, a[1], b[1])
    assert np.array_equal(runs[0][-1], runs[1][-1])


@pytest.mark.parametrize("shape", [(40, 44, 48), (37, 29, 41)])
def test_k5_tiles_equal_scalar_kernel(P, monkeypatch, shape):
    """K5 on shared-memory tiles (integer 3-D images) against the per-particle
    kernel: every raw PS increment bit-identical (l2 mode exposes them as the
    rank values), also on lattices that are not multiples of the 8^3 tile."""
    import scenes
    sc = scenes.cfg4(n=shape[0], n_obj=5, per_axis=2, radius=9.0)
    img = np.ascontiguousarray(sc.image[:, :shape[1], :shape[2]])
    lab = np.ascontiguousarray(sc.labels[:, :shape[1], :shape[2]])
    ecfg = P.EnergyConfig("ps", "poisson", 0.0, 4)
    runs = []
    for k5 in ("tile", "scalar"):
        monkeypatch.setenv("RCB_K5", k5)
        eng = P.RegionCompetition(img, lab, ecfg, P.SobolevParams(6.0),
                                  P.OptimizerConfig("l2", vanish_grace=5, drift_tolerance=1e-3))
        out = []
        for _ in range(3):
            eng.iterate()
            out.append(eng.last_candidates[3].copy())
        runs.append(out)
    for it, (a, b) in enumerate(zip(*runs)):
        assert a.shape == b.shape and np.array_equal(a, b), it


@pytest.mark.parametrize("shape", [(40, 44, 48), (37, 29, 41), (2, 300, 257)])
def test_k5_packed_records_equal_gather_kernel(P, monkeypatch, shape):
    """K5 over packed 16-byte site records with the {theta, log theta} table
    (integer Poisson images, the default) against the five-array gather
    kernel (RCB_NO_K5REC=1): every raw PS increment bit-identical over three
    l2 iterations (labels move, so the records are re-packed from refreshed
    fields), in 3-D and 2-D, on lattices that are not tile multiples."""
    import scenes
    if shape[0] == 2:
        sc = scenes.cfg4(n=shape[2], n_obj=5, per_axis=2, radius=9.0)
        img = np.ascontiguousarray(sc.image[shape[2] // 2, :shape[1], :shape[2]])
        lab = np.ascontiguousarray(sc.labels[shape[2] // 2, :shape[1], :shape[2]])
    else:
        sc = scenes.cfg4(n=shape[0], n_obj=5, per_axis=2, radius=9.0)
        img = np.ascontiguousarray(sc.image[:, :shape[1], :shape[2]])
        lab = np.ascontiguousarray(sc.labels[:, :shape[1], :shape[2]])
    ecfg = P.EnergyConfig("ps", "poisson", 0.0, 4)
    runs = []
    for norec in ("0", "1"):
        if norec == "1":
            monkeypatch.setenv("RCB_NO_K5REC", "1")
        else:
            monkeypatch.delenv("RCB_NO_K5REC", raising=False)
        eng = P.RegionCompetition(img, lab, ecfg, P.SobolevParams(6.0),
                                  P.OptimizerConfig("l2", vanish_grace=5, drift_tolerance=1e-3))
        out = []
        for _ in range(3):
            eng.iterate()
            out.append(eng.last_candidates[3].copy())
        out.append(eng.labels.copy())
        runs.append(out)
    for it, (a, b) in enumerate(zip(*runs)):
        assert a.shape == b.shape and np.array_equal(a, b), it
