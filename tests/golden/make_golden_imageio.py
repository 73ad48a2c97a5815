"""Golden files written by the REFERENCE's rcseg.imageio for fixed inputs,
made in the build container:

    python tests/golden/make_golden_imageio.py

Covers write_labels (2-D P5 16-bit, 3-D NRRD ushort), write_pgm (binary and
plain, 8- and 16-bit), write_nrrd (float/ushort/uchar, 2-D and 3-D),
write_image (.pgm scaled, float NRRD) and write_overlay (2-D PGM, 3-D NRRD
uchar; the reference's host contour scan) on seeded label rasters with
several regions touching each other, the border and background.
"""
from __future__ import annotations

import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "imageio")
sys.path.insert(0, "/root/reference/pkg/src")
_mpl = types.ModuleType("matplotlib")
_mpl.use = lambda *a, **k: None
_mpl.pyplot = types.ModuleType("matplotlib.pyplot")
sys.modules.setdefault("matplotlib", _mpl)
sys.modules.setdefault("matplotlib.pyplot", _mpl.pyplot)

from rcseg import imageio as IO  # noqa: E402


def inputs():
    rng = np.random.default_rng(1403)
    lab2 = np.zeros((23, 31), np.int32)
    lab2[3:12, 4:15] = 1
    lab2[8:20, 12:28] = 2
    lab2[0:5, 25:31] = 3
    lab2[15:23, 0:6] = 700
    lab2[10, 20] = 0
    lab3 = np.zeros((9, 11, 13), np.int32)
    lab3[1:6, 2:8, 3:10] = 1
    lab3[4:9, 5:11, 0:6] = 2
    lab3[0:3, 0:3, 10:13] = 4
    img2 = rng.poisson(30.0, (17, 19)).astype(np.float64)
    img3 = rng.normal(5.0, 2.0, (5, 6, 7))
    big = rng.integers(0, 65536, (7, 9)).astype(np.float64)
    return lab2, lab3, img2, img3, big


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    lab2, lab3, img2, img3, big = inputs()
    p = lambda n: os.path.join(OUT, n)  # noqa: E731
    IO.write_labels(lab2, p("labels2.pgm"))
    IO.write_labels(lab3, p("labels3.nrrd"))
    IO.write_pgm(img2, p("img2.pgm"))
    IO.write_pgm(img2, p("img2_plain.pgm"), plain=True)
    IO.write_pgm(big, p("big16.pgm"))
    IO.write_pgm(big, p("big16_plain.pgm"), plain=True)
    IO.write_nrrd(img3, p("img3_float.nrrd"))
    IO.write_nrrd(img2, p("img2_ushort.nrrd"), dtype="ushort")
    IO.write_nrrd(img2, p("img2_uchar.nrrd"), dtype="uchar")
    IO.write_image(img3[0] * 1.37, p("scaled.pgm"), scale=True)
    IO.write_image(img3, p("image3.nrrd"))
    IO.write_overlay(lab2, p("overlay2.pgm"))
    IO.write_overlay(lab3, p("overlay3.nrrd"))
    np.savez_compressed(p("inputs.npz"), lab2=lab2, lab3=lab3, img2=img2, img3=img3, big=big)


if __name__ == "__main__":
    main()
