"""Batched images on the device: run_batch (several engines in flight on
separate streams) must give exactly the results of one-at-a-time runs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_run_batch_matches_single_runs():
    import paper_1403_0240_b200 as P
    import scenes
    from paper_1403_0240_b200.batch import gather_summaries, run_batch
    scs = [scenes.cfg5_image(i, n=160) for i in range(6)]
    imgs = [s.image for s in scs]
    inits = [s.labels for s in scs]
    ecfg = P.EnergyConfig("pc", "gauss")
    scfg = P.SobolevParams(4.0)
    ocfg = P.OptimizerConfig("sobolev", max_iterations=25)
    batch = run_batch(imgs, inits, ecfg, scfg, ocfg, rank=0, world=1, in_flight=3)
    assert [i for i, _ in batch] == list(range(6))
    for i, res in batch:
        ref = P.run(imgs[i], inits[i], ecfg, scfg, ocfg)
        assert np.array_equal(res.labels, ref.labels), i
        assert [r.energy for r in res.trace] == [r.energy for r in ref.trace], i
        assert res.status == ref.status
    summ = gather_summaries(batch)
    assert [s.index for s in summ] == list(range(6))


def test_compare_batch_matches_single_runs():
    """Batched L2-vs-Sobolev pairs (cli compare over several images, all pairs
    in flight at once) equal one-at-a-time runs."""
    import paper_1403_0240_b200 as P
    import scenes
    from paper_1403_0240_b200.batch import compare_batch
    scs = [scenes.cfg5_image(i, n=128) for i in range(3)]
    ecfg = P.EnergyConfig("pc", "gauss")
    scfg = P.SobolevParams(4.0)
    ocfg = P.OptimizerConfig("sobolev", max_iterations=20)
    out = compare_batch([s.image for s in scs], [s.labels for s in scs], ecfg, scfg, ocfg,
                        rank=0, world=1, in_flight=6)
    assert [i for i, _ in out] == [0, 1, 2]
    for i, pair in out:
        for g in ("l2", "sobolev"):
            ref = P.run(scs[i].image, scs[i].labels, ecfg, scfg,
                        P.OptimizerConfig(g, max_iterations=20))
            assert np.array_equal(pair[g].labels, ref.labels), (i, g)
            assert [r.energy for r in pair[g].trace] == [r.energy for r in ref.trace], (i, g)
