"""Run a BASELINE config to iteration W (unprofiled), then bracket K
iterations with cudaProfilerStart/Stop, for
``ncu --profile-from-start off`` launch lists and ``--set full`` captures of
exactly the bench window's kernels.

  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
      python tools/profile_window.py --config cfg4 --warm 24 --iters 1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1403_0240_b200 as P  # noqa: E402
import scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--warm", type=int, default=24)
    ap.add_argument("--iters", type=int, default=1)
    a = ap.parse_args()
    sc = scenes.CONFIGS[a.config]()
    eng = P.RegionCompetition(sc.image, sc.labels,
                              P.EnergyConfig(sc.region, sc.noise, sc.lam, sc.smooth_radius),
                              P.SobolevParams(sc.length_scale),
                              P.OptimizerConfig("sobolev", vanish_grace=sc.vanish_grace,
                                                drift_tolerance=1e-3))
    for _ in range(a.warm):
        eng.iterate()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(a.iters):
        rec = eng.iterate()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("iteration", rec.iteration, "particles", eng.last_candidates[0].size, "moves", rec.moves,
          "timings", eng.timings())


if __name__ == "__main__":
    main()
