import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1403_0240_b200 as P, scenes
sc = scenes.cfg2()
eng = P.RegionCompetition(sc.image, sc.labels, P.EnergyConfig("ps", "poisson", smooth_radius=4),
                          P.SobolevParams(6.0), P.OptimizerConfig("sobolev", vanish_grace=5, drift_tolerance=1e-3))
mx = 0
for it in range(100):
    eng.iterate()
    if it % 10 == 9:
        xs, ow, cm, rk = eng.last_candidates
        neg = rk[rk < 0]
        u, c = np.unique(neg, return_counts=True)
        print(it + 1, "neg", len(neg), "dup values", int((c > 1).sum()), "max run", int(c.max()), "in dups", int(c[c > 1].sum()))
