import os, sys
sys.path.insert(0, os.getcwd())
import paper_1403_0240_b200 as P, scenes
sc = scenes.cfg2()
ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
ocfg = P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace)
eng = P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale), ocfg)
for i in range(int(sys.argv[1])):
    r = eng.iterate(); print(i, r.moves, eng.counters()["deferred"], flush=True)
