"""Three cfg4 engines in sequence (as bench.py creates them), 26 iterations
each, with RCB_ALLOC_LOG: which iteration stalls and which allocation."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402

sc = scenes.cfg4()
for run in range(3):
    eng = P.RegionCompetition(sc.image, sc.labels,
                              P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius),
                              P.SobolevParams(sc.length_scale),
                              P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace,
                                                drift_tolerance=1e-3))
    ms = []
    for it in range(26):
        print(f"== run {run} it {it + 1}", file=sys.stderr, flush=True)
        eng.iterate()
        t, _ = eng.timings()
        ms.append([round(x, 1) for x in t])
    print(json.dumps({"run": run, "ms": [m[5] for m in ms],
                      "spikes": [(i + 1, m) for i, m in enumerate(ms) if m[5] > 1.6 * ms[i - 1][5] and i]}),
          flush=True)
    del eng
