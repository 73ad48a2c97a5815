"""Constructor cost of RegionCompetition on cfg2 (the e2e term outside the
iterations): wall time of each phase, repeated (first = cold)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402

sc = scenes.cfg2()
img = torch.from_numpy(np.ascontiguousarray(sc.image, np.float64)).pin_memory().numpy()
lab = torch.from_numpy(np.ascontiguousarray(sc.labels, np.int32)).pin_memory().numpy()
ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
ocfg = P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace, drift_tolerance=1e-3)
for rep in range(4):
    t0 = time.perf_counter()
    eng = P.RegionCompetition(img, lab, ecfg, P.SobolevParams(sc.length_scale), ocfg)
    t1 = time.perf_counter()
    eng.iterate()
    t2 = time.perf_counter()
    for _ in range(4):
        eng.iterate()
    t3 = time.perf_counter()
    out = eng.labels
    t4 = time.perf_counter()
    print(f"ctor {1e3*(t1-t0):.2f} ms  first iterate {1e3*(t2-t1):.2f} ms  next 4 {1e3*(t3-t2)/4:.2f} ms/it  labels {1e3*(t4-t3):.2f} ms")
    del eng
