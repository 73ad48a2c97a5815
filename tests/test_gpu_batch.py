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
