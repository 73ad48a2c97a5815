import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, scenes
import paper_1403_0240_b200 as P
sc = scenes.cfg2()
eng = P.RegionCompetition(sc.image, sc.labels, P.EnergyConfig("ps", "poisson", smooth_radius=4),
                          P.SobolevParams(6.0), P.OptimizerConfig("sobolev", vanish_grace=5, resync_every=1000))
for it in range(20):
    rec = eng.iterate()
    print(rec.iteration, rec.moves, rec.particles, repr(rec.energy), flush=True)
    if rec.iteration % 10 == 0:
        ref = eng._evaluate().total
        print("DRIFT", rec.iteration, abs(ref - rec.energy), repr(ref), flush=True)
        eng._energy = ref
        P._lib.lib.rcb_engine_set_energy(eng._h, ref)
