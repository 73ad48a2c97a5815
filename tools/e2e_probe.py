import os, sys, time, json
sys.path.insert(0, os.getcwd())
os.environ["RCB_CTOR_LOG"] = "1"
import numpy as np, torch
import paper_1403_0240_b200 as P, scenes
from paper_1403_0240_b200 import optimizer as O
sc = scenes.cfg2()
ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
ocfg = P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace, drift_tolerance=1e-3)
main = P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale), ocfg)
for _ in range(25): main.iterate()
er = P.RegionCompetition(sc.image, sc.labels, ecfg, P.SobolevParams(sc.length_scale), ocfg)
for _ in range(25): er.iterate()
del er
img = torch.from_numpy(np.ascontiguousarray(sc.image)).pin_memory().numpy()
lab = torch.from_numpy(np.ascontiguousarray(sc.labels, np.int32)).pin_memory().numpy()
orig_eval = O.RegionCompetition._evaluate
def timed_eval(self):
    t = time.perf_counter(); r = orig_eval(self); print(f"  _evaluate {1e3*(time.perf_counter()-t):.2f} ms", file=sys.stderr); return r
O.RegionCompetition._evaluate = timed_eval
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2 = P.RegionCompetition(img, lab, ecfg, P.SobolevParams(sc.length_scale), ocfg)
    print(f"ctor {1e3*(time.perf_counter()-t0):.2f} ms", file=sys.stderr)
    for _ in range(25): e2.iterate()
    del e2
