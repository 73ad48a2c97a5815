"""Generate the golden fixtures by running the REFERENCE itself (rcseg).

Run in the build container only (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py [--skip-cfg1]

It imports ``rcseg`` from ``/root/reference/pkg/src`` (read-only, unmodified),
feeds it the seeded inputs of ``scenes.py`` / local generators, and stores
inputs and outputs as compressed ``.npz`` files next to this script.  The
fixtures pin both the CPU oracle (tests/test_oracle_golden.py) and the CUDA
path (tests/test_gpu_*.py).
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import rcseg  # noqa: E402
from rcseg import contour as rc_contour  # noqa: E402
from rcseg import energy as rc_energy  # noqa: E402
from rcseg import optimizer as rc_opt  # noqa: E402
from rcseg import sobolev as rc_sob  # noqa: E402
from rcseg.grid import Connectivity  # noqa: E402

import scenes  # noqa: E402
from rcseg import synth as rc_synth  # noqa: E402

# The BASELINE scenes blur and noise through the REFERENCE's own pipeline here
# (SURVEY Appendix A); on the GPU box scenes.py uses the device pipeline,
# which tests/test_gpu_fixtures.py checks against these images bit for bit.
scenes.use_backend(
    blur=rc_synth.blur,
    poissonize=lambda img, psnr, seed: rc_synth.poissonize(img, rc_synth.NoiseSpec(psnr, seed)))


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: {os.path.getsize(path) / 1024:.1f} KiB")


def connected_random_labels(rng, shape, n_blobs, conn):
    from scipy import ndimage
    labels = np.zeros(shape, np.int32)
    g = np.indices(shape)
    for _ in range(n_blobs):
        c = [rng.integers(0, s) for s in shape]
        r = rng.integers(1, 4)
        d2 = sum((gi - ci) ** 2 for gi, ci in zip(g, c))
        labels[d2 <= r * r] = labels.max() + 1
    out = np.zeros_like(labels)
    nxt = 1
    for l in np.unique(labels):
        if l == 0:
            continue
        comp, n = ndimage.label(labels == l, structure=conn.fg_structure)
        for k in range(1, n + 1):
            out[comp == k] = nxt
            nxt += 1
    return out


# --------------------------------------------------------------------------

def gen_kernel():
    out = {}
    cases = [(12.0, 1 / 24), (4.0, 1 / 24), (6.0, 1 / 24), (2.0, 1 / 24), (8.0, 1 / 24),
             (16.0, 1 / 24), (5.0, 0.1), (12.0, 0.5)]
    for k, (E, eps) in enumerate(cases):
        p = rc_sob.SobolevParams(E, eps)
        c2 = p.cutoff ** 2
        d2 = np.arange(int(np.ceil(c2)))
        d2 = d2[d2 < c2]
        out[f"E{k}"] = np.array([E, eps])
        out[f"w{k}"] = np.asarray(rc_sob.kernel_eval(np.sqrt(d2.astype(np.float64)), p))
    save("kernel.npz", **out)


def gen_sobolev():
    rng = np.random.default_rng(101)
    out = {}
    k = 0
    for ndim in (2, 3):
        for E in (2.0, 4.0, 6.0, 12.0, 8.0):
            for n, ext in ((1, 5), (60, 8), (400, 30), (1500, 40)):
                coords = rng.integers(0, ext, size=(n, ndim)).astype(np.int64)
                owners = rng.integers(0, 4, size=n).astype(np.int64)
                comps = rng.integers(0, 4, size=n).astype(np.int64)   # may equal owner
                raw = rng.normal(size=n)
                got = rc_sob.sobolev_filter(coords, owners, comps, raw,
                                            rc_sob.SobolevParams(E))
                pi, _, _ = rc_sob.build_cell_list(coords, rc_sob.SobolevParams(E)).pairs(E / 2)
                out[f"c{k}"] = coords
                out[f"o{k}"] = owners
                out[f"m{k}"] = comps
                out[f"r{k}"] = raw
                out[f"E{k}"] = np.array([E])
                out[f"y{k}"] = got
                out[f"p{k}"] = np.array([len(pi)])
                k += 1
    # a contour-shaped case: particles of a real label image (2-D and 3-D)
    for shape in ((64, 64), (20, 20, 20)):
        conn = Connectivity.default(len(shape))
        lab = connected_random_labels(rng, shape, 12, conn)
        xs, owners, comps = rc_contour.scan_contour(lab, conn).as_arrays(lab)
        coords = np.stack(np.unravel_index(xs, shape), axis=1)
        raw = rng.normal(size=len(xs))
        for E in (4.0, 6.0):
            got = rc_sob.sobolev_filter(coords, owners, comps, raw, rc_sob.SobolevParams(E))
            out[f"c{k}"], out[f"o{k}"], out[f"m{k}"] = coords, owners, comps
            out[f"r{k}"], out[f"E{k}"], out[f"y{k}"] = raw, np.array([E]), got
            pi, _, _ = rc_sob.build_cell_list(coords, rc_sob.SobolevParams(E)).pairs(E / 2)
            out[f"p{k}"] = np.array([len(pi)])
            k += 1
    out["n"] = np.array([k])
    save("sobolev.npz", **out)


def gen_contour():
    rng = np.random.default_rng(202)
    out = {}
    k = 0
    for ndim, shape in ((2, (12, 11)), (3, (6, 7, 5)), (2, (1, 9)), (2, (30, 31))):
        for fg_full in (True, False):
            conn = Connectivity(ndim, {2: 8, 3: 26}[ndim] if fg_full else {2: 4, 3: 6}[ndim])
            for _ in range(3):
                lab = rng.integers(0, 4, size=shape).astype(np.int32)
                keys = sorted(rc_contour.scan_contour(lab, conn).as_key_set())
                out[f"l{k}"] = lab
                out[f"f{k}"] = np.array([int(fg_full)])
                out[f"k{k}"] = np.array(keys, np.int64).reshape(-1, 2)
                k += 1
    out["n"] = np.array([k])
    save("contour.npz", **out)


def gen_energy():
    """ΔE_ext / ΔE_int for every particle, and evaluate_total, on small rasters."""
    rng = np.random.default_rng(303)
    out = {}
    k = 0
    for shape in ((24, 26), (9, 10, 8)):
        conn = Connectivity.default(len(shape))
        lab = connected_random_labels(rng, shape, 6, conn)
        img_g = rng.normal(1.0, 0.5, size=shape)
        img_p = rng.poisson(6.0, size=shape).astype(np.float64)
        xs, owners, comps = rc_contour.scan_contour(lab, conn).as_arrays(lab)
        o = np.lexsort((comps, xs))
        xs, owners, comps = xs[o], owners[o], comps[o]
        for region, noise, r in (("pc", "gauss", 8), ("pc", "poisson", 8),
                                 ("ps", "gauss", 2), ("ps", "poisson", 3), ("ps", "poisson", 4)):
            img = img_g if noise == "gauss" else img_p
            cfg = rc_energy.EnergyConfig(region, noise, lam=0.3, smooth_radius=r)
            model = rc_energy.EnergyModel(img, lab, cfg)
            out[f"lab{k}"] = lab
            out[f"img{k}"] = img
            out[f"cfg{k}"] = np.array([region == "ps", noise == "poisson", r, 0.3])
            out[f"xs{k}"], out[f"ow{k}"], out[f"cm{k}"] = xs, owners, comps
            out[f"de{k}"] = model.delta_external_batch(xs, owners, comps)
            out[f"di{k}"] = rc_energy.delta_internal_batch(lab, xs, owners, comps)
            ev = rc_energy.evaluate_total(lab, img, cfg)
            out[f"ev{k}"] = np.array([ev.total, ev.external, ev.internal])
            k += 1
    out["n"] = np.array([k])
    save("energy.npz", **out)


def gen_admissible():
    rng = np.random.default_rng(404)
    out = {}
    k = 0
    for ndim, shape, nb in ((2, (14, 14), 5), (3, (7, 7, 6), 4)):
        for fg_full in (True, False):
            conn = Connectivity(ndim, {2: 8, 3: 26}[ndim] if fg_full else {2: 4, 3: 6}[ndim])
            for _ in range(3):
                lab = connected_random_labels(rng, shape, nb, conn)
                keys = sorted(rc_contour.scan_contour(lab, conn).as_key_set())
                rows = []
                for x, c in keys:
                    for fusion in (0, 1):
                        for vanish in (0, 1):
                            ok = rc_contour.is_move_admissible(lab, x, c, conn, bool(fusion),
                                                               bool(vanish))
                            rows.append((x, c, fusion, vanish, int(ok)))
                out[f"l{k}"] = lab
                out[f"f{k}"] = np.array([int(fg_full)])
                out[f"v{k}"] = np.array(rows, np.int64).reshape(-1, 5)
                k += 1
    out["n"] = np.array([k])
    save("admissible.npz", **out)


def label_hash(lab) -> str:
    return hashlib.sha256(np.ascontiguousarray(lab, np.int32).tobytes()).hexdigest()[:16]


def record_run(name, image, init, energy_cfg, sob, opt, iterations, keep_labels=True,
               use_run=False):
    """Run the reference engine; record per-iteration accepted moves (in
    acceptance order, captured by wrapping apply_move), labels and trace."""
    accepted = []
    real_apply = rc_opt.apply_move

    def spy(labels, contour, stats, img, pixel, owner, competitor, conn):
        accepted.append((int(pixel), int(owner), int(competitor)))
        return real_apply(labels, contour, stats, img, pixel, owner, competitor, conn)

    rc_opt.apply_move = spy
    try:
        eng = rc_opt.RegionCompetition(image, init, energy_cfg, sob, opt)
        per_iter_moves, per_iter_labels, per_iter_hash = [], [], []
        if use_run:
            marks = []

            def cb(e, rec):
                marks.append(len(accepted))
                per_iter_hash.append(label_hash(e.labels))
                if keep_labels:
                    per_iter_labels.append(e.labels.copy())
            res = eng.run(on_iteration=cb)
            starts = [0] + marks[:-1]
            per_iter_moves = [accepted[s:e] for s, e in zip(starts, marks)]
            status = res.status
            final = res.final_energy
            extra = dict(status=np.array([status]), iterations=np.array([res.iterations]),
                         fallback=np.array([-1 if res.fallback_iteration is None
                                            else res.fallback_iteration]),
                         final=np.array([final.total, final.external, final.internal]),
                         regions=np.array([res.region_count]))
        else:
            extra = {}
            for _ in range(iterations):
                s = len(accepted)
                eng.iterate()
                per_iter_moves.append(accepted[s:])
                per_iter_hash.append(label_hash(eng.labels))
                if keep_labels:
                    per_iter_labels.append(eng.labels.copy())
    finally:
        rc_opt.apply_move = real_apply
    tr = eng.trace
    out = dict(
        image=np.asarray(image, np.float32) if np.asarray(image).dtype == np.float32 else image,
        init=init,
        energy=np.array([r.energy for r in tr]),
        moves=np.array([r.moves for r in tr]),
        particles=np.array([r.particles for r in tr]),
        mode=np.array([r.mode for r in tr]),
        hashes=np.array(per_iter_hash),
        acc_len=np.array([len(m) for m in per_iter_moves]),
        acc=np.array([t for m in per_iter_moves for t in m], np.int64).reshape(-1, 3),
        cfg=np.array([energy_cfg.region_model == "ps", energy_cfg.noise_model == "poisson",
                      energy_cfg.smooth_radius, energy_cfg.lam, sob.length_scale, sob.epsilon,
                      opt.gradient == "sobolev", opt.vanish_grace, opt.seed,
                      opt.allow_fusion, opt.allow_vanish, opt.move_budget]),
        **extra,
    )
    if keep_labels:
        out["labels"] = np.array(per_iter_labels)
    save(f"run_{name}.npz", **out)


def gen_runs(skip_cfg1: bool):
    E = rc_energy.EnergyConfig
    S = rc_sob.SobolevParams
    O = rc_opt.OptimizerConfig
    sc = scenes.two_region_small((48, 48), seed=1)
    record_run("pc2d", sc.image, sc.labels, E("pc", "gauss"), S(4.0), O("sobolev"), 25)
    record_run("pc2d_l2", (np.abs(sc.image) + 0.1).astype(np.float32), sc.labels, E("pc", "poisson", lam=0.2), S(4.0), O("l2", seed=5),
               12)
    sc3 = scenes.cfg3(seed=3, n=20)
    record_run("pc3d", sc3.image, sc3.labels, E("pc", "gauss"), S(4.0), O("sobolev"), 8)
    # PS poisson, bubbles init, lam > 0 (the reference's two-blob style)
    img = scenes._cfg2_image(1024, 2)[:64, :64].copy()
    lab = scenes.bubbles(img.shape, 2, 10.0)
    record_run("ps2d", img, lab, E("ps", "poisson", lam=0.04, smooth_radius=4), S(6.0),
               O("sobolev", vanish_grace=5), 12)
    rng = np.random.default_rng(7)
    img_g = (scenes.two_region_small((40, 40), seed=3).image
             + rng.normal(0, 0.1, size=(40, 40))).astype(np.float64)
    lab_g = scenes.bubbles((40, 40), 3, 5.0)
    record_run("ps2d_gauss", img_g, lab_g, E("ps", "gauss", smooth_radius=2), S(6.0),
               O("sobolev"), 8)
    # full runs to a terminal status (statuses, fallback iteration, final energy)
    sc = scenes.two_region_small((32, 32), seed=4)
    record_run("full_pc2d", sc.image, sc.labels, E("pc", "gauss"), S(4.0),
               O("sobolev", max_iterations=300), 0, use_run=True)
    small = img[:40, :40].copy()
    record_run("full_ps2d", small, scenes.bubbles(small.shape, 2, 6.0),
               E("ps", "poisson", lam=0.04, smooth_radius=3), S(6.0),
               O("sobolev", max_iterations=300, vanish_grace=5), 0, use_run=True)
    # scaled cfg2 (256^2 crop, bubbles:4:10, PS poisson R=4, E=6) — 4 iterations
    s2 = scenes.cfg2_small()
    record_run("cfg2_small", s2.image, s2.labels, E("ps", "poisson", smooth_radius=4), S(6.0),
               O("sobolev", vanish_grace=5), 4, keep_labels=False)
    if not skip_cfg1:
        s1 = scenes.cfg1()
        record_run("cfg1", s1.image, s1.labels, E("pc", "gauss"), S(4.0), O("sobolev"), 50,
                   keep_labels=False)


# -- the BASELINE configs at their own sizes ("pin every config") --

def big_runs():
    E, S, O = rc_energy.EnergyConfig, rc_sob.SobolevParams, rc_opt.OptimizerConfig
    ps4 = dict(smooth_radius=4)

    def cfg2_full():
        # iterations 1..26 cover bench.py's timed window (6..25); the drift
        # tolerance is the bench's (the reference's own ledger
        # drifts ~1e-6 on cfg2 by the iteration-20 resync).
        s = scenes.cfg2()
        record_run("cfg2_full", s.image, s.labels, E("ps", "poisson", **ps4), S(6.0),
                   O("sobolev", vanish_grace=5, drift_tolerance=1e-3), 26, keep_labels=False)

    def cfg3():
        s = scenes.cfg3()
        record_run("cfg3", s.image, s.labels, E("pc", "gauss"), S(4.0), O("sobolev"), 3,
                   keep_labels=False)

    def cfg4s():
        s = scenes.cfg4_small()
        record_run("cfg4s", s.image, s.labels, E("ps", "poisson", **ps4), S(6.0),
                   O("sobolev", vanish_grace=5, drift_tolerance=1e-3), 6, keep_labels=False)

    def cfg5(i):
        s = scenes.cfg5_image(i)
        record_run(f"cfg5_{i}", s.image, s.labels, E("pc", "gauss"), S(4.0), O("sobolev"), 50,
                   keep_labels=False)

    def cfg4s_l2():
        # PS/Poisson in l2 mode (the d_tot < 0 gate with PS fields), 3-D
        s = scenes.cfg4_small()
        record_run("cfg4s_l2", s.image, s.labels, E("ps", "poisson", **ps4), S(6.0),
                   O("l2", vanish_grace=5, drift_tolerance=1e-3), 3, keep_labels=False)

    def cfg2s_l2():
        s = scenes.cfg2_small()
        record_run("cfg2s_l2", s.image, s.labels, E("ps", "poisson", **ps4), S(6.0),
                   O("l2", vanish_grace=5, drift_tolerance=1e-3), 4, keep_labels=False)

    jobs = {"cfg2_full": cfg2_full, "cfg3": cfg3, "cfg4s": cfg4s, "cfg4s_l2": cfg4s_l2,
            "cfg2s_l2": cfg2s_l2}
    for i in range(4):
        jobs[f"cfg5_{i}"] = (lambda i=i: cfg5(i))
    return jobs


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-cfg1", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    big = big_runs()
    if a.only in big:
        big[a.only]()
        sys.exit(0)
    todo = a.only.split(",") if a.only else ["kernel", "sobolev", "contour", "energy",
                                             "admissible", "runs"]
    for t in todo:
        if t == "runs":
            gen_runs(a.skip_cfg1)
        else:
            globals()[f"gen_{t}"]()
