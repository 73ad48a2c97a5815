"""Time l2-mode iterations (the PS d_tot < 0 gate in the dataflow kernel) on a
BASELINE config after K Sobolev iterations -- the state the oscillation
fallback hands to l2 mode.

  python tools/ps_l2_probe.py --config cfg4 --sobolev 30 --l2 2
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--sobolev", type=int, default=30)
    ap.add_argument("--l2", type=int, default=2)
    a = ap.parse_args()
    sc = scenes.CONFIGS[a.config]()
    eng = P.RegionCompetition(sc.image, sc.labels,
                              P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius),
                              P.SobolevParams(sc.length_scale),
                              P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace,
                                                drift_tolerance=1e-3))
    for _ in range(a.sobolev):
        eng.iterate()
    eng.mode = "l2"
    for _ in range(a.l2):
        t0 = time.time()
        rec = eng.iterate()
        t, _ = eng.timings()
        print(json.dumps({"it": rec.iteration, "mode": rec.mode, "wall_s": round(time.time() - t0, 3),
                          "ms": round(t[5], 2), "phases": [round(x, 2) for x in t[:5]],
                          "moves": rec.moves, "particles": rec.particles,
                          "parallel": eng.counters()["parallel"]}), flush=True)


if __name__ == "__main__":
    main()
