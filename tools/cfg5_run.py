"""BASELINE configs[4] first part on this GPU: 256 independent 512x512
PC/Gauss images (seeds 1000 + i), Sobolev w = 2, 50 iterations each, through
the batched data-parallel runner (several engines in flight on separate
streams).  Under torchrun the images are split over ranks.

  python tools/cfg5_run.py [--images 256] [--in-flight 8]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402
from paper_1403_0240_b200.batch import run_batch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=256)
    ap.add_argument("--in-flight", type=int, default=8)
    a = ap.parse_args()
    t0 = time.time()
    scs = [scenes.cfg5_image(i) for i in range(a.images)]
    gen = time.time() - t0
    sc = scs[0]
    ecfg = P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius)
    ocfg = P.OptimizerConfig("sobolev", max_iterations=sc.iterations)
    t0 = time.time()
    out = run_batch([s.image for s in scs], [s.labels for s in scs], ecfg,
                    P.SobolevParams(sc.length_scale), ocfg, in_flight=a.in_flight)
    wall = time.time() - t0
    iters = sum(r.iterations for _, r in out)
    status = {}
    for _, r in out:
        status[r.status] = status.get(r.status, 0) + 1
    print(json.dumps({"images": len(out), "gen_s": round(gen, 2), "wall_s": round(wall, 3),
                      "images_per_s": len(out) / wall, "iterations": iters,
                      "iterations_per_s": iters / wall, "statuses": status}))


if __name__ == "__main__":
    main()
