"""Sobolev-kernel sweep (BASELINE configs[4], second part) on one GPU.

For each (lattice, sphere count) giving ~1e4..1e8 contour particles and each
width w in {1, 2, 4, 8} (E = 2w): K6 device time with CUDA events (L2 flushed
between launches), particle-interactions/s and the HBM roofline fraction of
SURVEY §8(d)'s algorithmic 28 B/particle (record 12 + raw 8 + out 8).
Prints one JSON line per point."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1403_0240_b200.sweep import SobolevSweep  # noqa: E402

POINTS = {
    "1e4": ((64, 64, 64), 3),
    "1e5": ((128, 128, 128), 24),
    "1e6": ((256, 256, 256), 240),
    "1e7": ((512, 512, 512), 2400),
    "1e8": ((512, 2048, 2048), 24000),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", default="1e4,1e5,1e6,1e7,1e8")
    ap.add_argument("--widths", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        "MEASURED_PEAKS.json") else 6650.0
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for pt in a.points.split(","):
        shape, nsph = POINTS[pt]
        for w in (int(x) for x in a.widths.split(",")):
            sw = SobolevSweep(shape, nsph, w, seed=11)
            for _ in range(2):
                sw.run()
            tot_ms, pairs = 0.0, 0
            for _ in range(a.reps):
                flush.zero_()
                torch.cuda.synchronize()
                pairs, ms = sw.run()
                tot_ms += ms
            ms = tot_ms / a.reps
            n = sw.n_particles
            gbs = 28.0 * n / (ms / 1e3) / 1e9
            print(json.dumps({"point": pt, "lattice": list(shape), "spheres": nsph, "width": w,
                              "particles": n, "pairs": pairs, "pairs_per_particle": pairs / max(n, 1),
                              "k6_ms": round(ms, 4), "interactions_per_s": pairs / (ms / 1e3),
                              "alg_GBs": round(gbs, 1), "hbm_frac": round(gbs / peak, 4)}),
                  flush=True)
            del sw
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
