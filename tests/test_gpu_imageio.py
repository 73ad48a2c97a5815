"""Overlay masks from the device particle scan vs the reference's files
(imageio.py:308-327; tests/golden/imageio/overlay*.{pgm,nrrd} were written
by the reference's host contour walk)."""
import os

import numpy as np
import pytest

from tests.test_gpu_parity import P  # noqa: F401

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "imageio")


def test_write_overlay_matches_reference_bytes(P, tmp_path):
    from paper_1403_0240_b200 import imageio as IO
    inp = np.load(os.path.join(GOLD, "inputs.npz"))
    for lab, name in ((inp["lab2"], "overlay2.pgm"), (inp["lab3"], "overlay3.nrrd")):
        IO.write_overlay(lab, tmp_path / name)
        with open(os.path.join(GOLD, name), "rb") as fh:
            assert (tmp_path / name).read_bytes() == fh.read(), name
        m = IO.read_image(tmp_path / name)
        assert set(np.unique(m)) <= {0.0, 255.0} and np.all(lab[m > 0] > 0)


def test_overlay_mask_is_foreground_particles(P):
    from paper_1403_0240_b200 import imageio as IO
    from paper_1403_0240_b200.contour import scan_contour
    from paper_1403_0240_b200.grid import Connectivity
    lab = np.load(os.path.join(GOLD, "inputs.npz"))["lab2"]
    want = np.zeros(lab.size, np.uint8)
    for x, _ in scan_contour(lab, Connectivity.default(2)).as_key_set():
        if lab.flat[x] > 0:
            want[x] = 255
    assert np.array_equal(IO.overlay_mask(lab), want.reshape(lab.shape))
