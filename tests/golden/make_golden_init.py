"""Golden outputs of the REFERENCE's rcseg.optimizer.initialize and of a
small `rcseg compare` / `rcseg segment` run, made in the build container:

    python tests/golden/make_golden_init.py

init.npz: every scheme (rect, bubbles with default and explicit radius,
otsu, maxima) on seeded 2-D and 3-D images.  cli/: the reference CLI's
label files, trace, report and compare CSV for a 40x48 two-disk image
(pc/gauss and ps/poisson), to be reproduced by the device CLI
(tests/test_gpu_cli.py); wall-clock fields are not compared.
"""
from __future__ import annotations

import os
import shutil
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
_mpl = types.ModuleType("matplotlib")
_mpl.use = lambda *a, **k: None
_mpl.pyplot = types.ModuleType("matplotlib.pyplot")
sys.modules.setdefault("matplotlib", _mpl)
sys.modules.setdefault("matplotlib.pyplot", _mpl.pyplot)

from rcseg import cli, imageio, optimizer  # noqa: E402
from rcseg import report as R  # noqa: E402

R.render_energy_figure = lambda *a, **k: None
cli.render_energy_figure = lambda *a, **k: None

SCHEMES = ["rect", "bubbles:3", "bubbles:2:5.5", "otsu", "maxima:2.0:3"]


def images():
    rng = np.random.default_rng(240)
    yy, xx = np.mgrid[0:40, 0:48]
    img2 = 10.0 + 40.0 * (((yy - 14) ** 2 + (xx - 15) ** 2) < 64) \
        + 25.0 * (((yy - 26) ** 2 + (xx - 33) ** 2) < 81)
    img2 = rng.poisson(img2).astype(np.float64)
    zz, yy, xx = np.mgrid[0:14, 0:16, 0:18]
    img3 = rng.poisson(8.0 + 30.0 * (((zz - 7) ** 2 + (yy - 8) ** 2 + (xx - 9) ** 2) < 20)).astype(np.float64)
    return img2, img3


def main() -> None:
    img2, img3 = images()
    out = {"img2": img2, "img3": img3, "schemes": np.array(SCHEMES)}
    for nd, img in ((2, img2), (3, img3)):
        for i, s in enumerate(SCHEMES):
            out[f"init{nd}_{i}"] = optimizer.initialize(img, s)
    np.savez_compressed(os.path.join(HERE, "init.npz"), **out)
    d = os.path.join(HERE, "cli")
    shutil.rmtree(d, ignore_errors=True)
    os.makedirs(d)
    imageio.write_pgm(img2, os.path.join(d, "in.pgm"))
    os.chdir(d)
    common = ["--input", "in.pgm", "--max-iter", "60", "--lambda", "0.5"]
    rc = cli.main(["compare", *common, "--init", "bubbles:3", "--output-prefix", "cmp",
                   "--report", "cmp.json"])
    rc2 = cli.main(["segment", *common, "--model", "ps", "--noise", "poisson", "--smooth-radius", "3",
                    "--init", "otsu", "--output", "seg.pgm", "--overlay", "seg_overlay.pgm",
                    "--trace", "seg.jsonl", "--report", "seg.json"])
    cli.main(["segment", "--input", "in.pgm", "--max-iter", "3", "--lambda", "0.5", "--init",
              "bubbles:3", "--output", "p.pgm", "--particles-csv", "particles.csv"])
    os.unlink("p.pgm")
    cli.render_kernel_figure = lambda *a, **k: None
    cli.main(["kernel-table", "--E", "9", "--epsilon", "1/30", "--samples", "101", "--out", "kernel.csv"])
    with open("exit_codes.txt", "w") as fh:
        fh.write(f"{rc} {rc2}\n")
    for f in os.listdir("."):
        if f.endswith(".png"):
            os.unlink(f)


if __name__ == "__main__":
    main()
