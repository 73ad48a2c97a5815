"""Device synthetic-data pipeline throughput: a 512^3
scene of 64 balls, blur sigma 1.5, Poisson peak 30, generated in one device
pass (wall clock incl. the labels + image download); beside it the
reference's per-voxel CPU pipeline (the pinned restatement of synth.py) timed
on a 32^3 sample and scaled per voxel.

  python tools/synth_bench.py [--n 512]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import synth_oracle as SO  # noqa: E402
from paper_1403_0240_b200 import synth as S  # noqa: E402


def scene(n, seed=4):
    rng = np.random.default_rng(seed)
    shapes = [S.Shape(kind="disk", center=tuple(rng.uniform(0, n, 3)),
                      radius=float(rng.uniform(10, 50) * n / 512), intensity=float(rng.uniform(0.5, 1.0)))
              for _ in range(64)]
    return S.SceneSpec(dims=(n, n, n), background=0.2, shapes=shapes, blur_sigma=1.5,
                       noise=S.NoiseSpec(psnr=float(np.sqrt(30.0)), seed=seed))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=512)
    a = ap.parse_args()
    spec = scene(a.n)
    S.generate(scene(64))  # warm-up (module load, context)
    t0 = time.perf_counter()
    labels, image = S.generate(spec)
    dev_s = time.perf_counter() - t0
    small = scene(32)
    d = S.scene_to_dict(small)
    t0 = time.perf_counter()
    _, clean = SO.render_scene(d)
    noisy = SO.poissonize(SO.blur(clean, 1.5), small.noise.psnr, small.noise.seed)
    cpu_s = time.perf_counter() - t0
    vox = a.n ** 3
    print(json.dumps({"dims": [a.n] * 3, "device_wall_s": round(dev_s, 3),
                      "voxels_per_s": vox / dev_s, "mean_count": float(image.mean()),
                      "cpu_reference_voxels_per_s": 32 ** 3 / cpu_s,
                      "cpu_sample": "32^3, reference algorithm restated (oracle/synth_oracle.py), 1 core",
                      "labels_max": int(labels.max()), "nonzero": int(np.count_nonzero(noisy))}))


if __name__ == "__main__":
    main()
