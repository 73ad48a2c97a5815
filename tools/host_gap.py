"""Host enqueue time per iteration (RCB_HOST_LOG) against device time on cfg2."""
import os
import sys
import time
os.environ["RCB_HOST_LOG"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402
sc = scenes.cfg2()
eng = P.RegionCompetition(sc.image, sc.labels, P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius),
                          P.SobolevParams(sc.length_scale), P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace, drift_tolerance=1e-3))
for i in range(12):
    w0 = time.perf_counter()
    eng.iterate()
    w = time.perf_counter() - w0
    t, n = eng.timings()
    print(f"iter {i+1}: wall {1e6*w:.1f} us, device {1e3*t[5]:.1f} us, launches {n}",
          file=sys.stderr)
