"""Golden fixtures of the reference's synthetic-data pipeline (rcseg.synth:
render_scene, blur, poissonize, generate), made by running the REFERENCE
itself in the build container:

    python tests/golden/make_golden_synth.py

Scenes cover every shape kind (disk/ball, rect/box, annulus/shell, later shapes
overwriting earlier ones), 2-D and 3-D, blur sigma 0 / 0.7 / 1.5 / 2.0 on
lattices smaller than the kernel (mirror padding wraps), and Poisson noise on
both sampler branches (CDF inversion below mean 30, PTRS above).  The stock
benchmark scenes (desk, two_blob, two_sphere) are included as-is.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from rcseg import synth as S  # noqa: E402


def specs():
    out = {
        "desk": S.desk_scene(),
        "two_blob": S.two_blob_scene(),
        "two_sphere": S.two_sphere_scene(),
    }
    out["shapes2d"] = S.SceneSpec(
        dims=(37, 41), background=0.25,
        shapes=[S.Shape(kind="rect", origin=(3, 4), size=(20, 30), intensity=2.0),
                S.Shape(kind="disk", center=(18.5, 20.25), radius=9.5, intensity=7.0),
                S.Shape(kind="annulus", center=(25, 12), inner=3.0, outer=6.5, intensity=1.5)],
        blur_sigma=0.7, noise=S.NoiseSpec(psnr=9.0, seed=123))      # peak mean 81: PTRS
    out["shapes3d"] = S.SceneSpec(
        dims=(13, 17, 11), background=1.0,
        shapes=[S.Shape(kind="annulus", center=(6, 8, 5), inner=2.0, outer=5.0, intensity=4.0),
                S.Shape(kind="rect", origin=(0, 2, 3), size=(5, 6, 20), intensity=3.0),
                S.Shape(kind="disk", center=(9, 4, 7), radius=3.2, intensity=6.0)],
        blur_sigma=1.5, noise=S.NoiseSpec(psnr=4.0, seed=99))       # peak mean 16: inversion
    out["tiny"] = S.SceneSpec(
        dims=(3, 5), background=0.0,
        shapes=[S.Shape(kind="disk", center=(1, 2), radius=1.0, intensity=50.0)],
        blur_sigma=2.0, noise=S.NoiseSpec(psnr=20.0, seed=5))       # kernel wider than the image
    out["noblur"] = S.SceneSpec(
        dims=(16, 16), background=0.3,
        shapes=[S.Shape(kind="disk", center=(8, 8), radius=5.0, intensity=0.9)],
        blur_sigma=0.0, noise=S.NoiseSpec(psnr=7.0, seed=2 ** 40 + 17))
    return out


def main():
    arrays = {}
    meta = {}
    for name, spec in specs().items():
        labels, clean = S.render_scene(spec)
        blurred = S.blur(clean, spec.blur_sigma)
        noisy = S.poissonize(blurred, spec.noise)
        arrays[f"{name}_labels"] = labels
        arrays[f"{name}_clean"] = clean
        arrays[f"{name}_blurred"] = blurred
        arrays[f"{name}_noisy"] = noisy
        meta[name] = S.scene_to_dict(spec)
    arrays["specs_json"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    path = os.path.join(HERE, "synth.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote synth.npz: {os.path.getsize(path) / 1024:.1f} KiB")


if __name__ == "__main__":
    main()
