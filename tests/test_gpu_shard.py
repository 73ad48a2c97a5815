"""z-slab sharded scoring on one GPU: G slab engines iterated in
lock step (shard.LocalSlabGroup: every engine scores its slab + halo, the
slabs' scores are copied into place, every engine finishes) must reproduce the
unsharded engine bit for bit — records, accepted moves in order, labels — for
every G, in 2-D and 3-D, PC and PS, Sobolev and l2 mode.  The slabs' phases
run one after another, so no kernel waits on another engine."""
import numpy as np
import pytest

import scenes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1403_0240_b200 as P
    from paper_1403_0240_b200 import _lib
    if _lib.device_count() < 1:
        pytest.fail("no CUDA device visible to librcseg_b200")
    return P


def _make(P, sc, gradient="sobolev"):
    ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
    ocfg = P.OptimizerConfig(gradient, vanish_grace=sc.vanish_grace, drift_tolerance=1e-3)
    return P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale), ocfg)


def _scene(which):
    if which == "cfg1":
        return scenes.cfg1()
    if which == "cfg2_small":
        return scenes.cfg2_small()
    if which == "cfg3_small":
        return scenes.cfg3(n=48)
    if which == "cfg4_small":
        return scenes.cfg4_small()
    raise KeyError(which)


@pytest.mark.parametrize("which,world,gradient,iters", [
    ("cfg1", 2, "sobolev", 12),
    ("cfg1", 5, "sobolev", 6),
    ("cfg1", 3, "l2", 6),
    ("cfg2_small", 3, "sobolev", 12),
    ("cfg3_small", 2, "sobolev", 8),
    ("cfg3_small", 4, "sobolev", 5),
    ("cfg4_small", 3, "sobolev", 5),
])
def test_slab_group_equals_single_engine(P, which, world, gradient, iters):
    from paper_1403_0240_b200.shard import LocalSlabGroup
    sc = _scene(which)
    ref = _make(P, sc, gradient)
    group = LocalSlabGroup([_make(P, sc, gradient) for _ in range(world)])
    for _ in range(iters):
        want = ref.iterate()
        got = group.iterate()
        acc = ref.last_accepted
        for g, eng in zip(got, group.engines):
            assert (g.iteration, g.energy, g.moves, g.particles) == \
                (want.iteration, want.energy, want.moves, want.particles)
            assert np.array_equal(eng.last_accepted, acc)
        if want.moves == 0:
            break
    lab = ref.labels
    for eng in group.engines:
        assert np.array_equal(eng.labels, lab)


def test_slab_engine_pairs_partition(P):
    """Each slab scores only its own particles: the Sobolev interaction counts
    of the slabs add up to the unsharded count."""
    from paper_1403_0240_b200.shard import LocalSlabGroup
    sc = scenes.cfg3(n=48)
    ref = _make(P, sc)
    group = LocalSlabGroup([_make(P, sc) for _ in range(3)])
    ref.iterate()
    group.iterate()
    assert sum(e.last_pairs for e in group.engines) == ref.last_pairs
    assert all(e.last_pairs < ref.last_pairs for e in group.engines)


def test_slab_band_refresh_through_resync_and_l2_switch(P):
    """3-D PS on integer data: each slab engine refreshes the own-label fields of
    its slab plus halo only and sums the band ledger over its slab; the shares
    are added exactly (int64 limbs) and rounded once.  Records must equal the
    unsharded engine's through a resync (full rebuild, iteration 10) and after
    the switch to l2 mode, whose acceptance reads the fields everywhere (the
    engines rebuild them in full first)."""
    from paper_1403_0240_b200.shard import LocalSlabGroup
    sc = scenes.cfg4(n=64, n_obj=8, per_axis=2)
    ref = _make(P, sc)
    group = LocalSlabGroup([_make(P, sc) for _ in range(3)])
    for it in range(14):
        if it == 11:
            ref.mode = "l2"
            for e in group.engines:
                e.mode = "l2"
        want = ref.iterate()
        got = group.iterate()
        acc = ref.last_accepted
        for g, eng in zip(got, group.engines):
            assert (g.iteration, g.energy, g.moves, g.particles) == \
                (want.iteration, want.energy, want.moves, want.particles), it
            assert np.array_equal(eng.last_accepted, acc), it
    lab = ref.labels
    for eng in group.engines:
        assert np.array_equal(eng.labels, lab)
