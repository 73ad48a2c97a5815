"""Stage the reference's own test modules for replay against the drop-in.

Test infrastructure (VERDICT r01 "Close the boundary"): copies the
unmodified test files of the reference package (``pkg/tests/test_*.py`` for
grid, sobolev, energy, contour, optimizer and imageio, plus its conftest)
from ``/root/reference`` into ``oracle/_ref/reftests/`` — git-ignored like
every other reference-derived artefact under ``oracle/_ref``, but not
gpurun-ignored, so the staged copy travels to the GPU box, where
``tests/test_gpu_reference_suite.py`` runs them with ``rcseg`` rebound to
``paper_1403_0240_b200``.  Nothing here is product code and nothing is
committed.  ``test_synth.py`` (private scalar samplers ``_Stream`` /
``_poisson_draw``), ``test_cli.py`` and ``test_acceptance.py`` (matplotlib)
are not staged.
"""
from __future__ import annotations

import os
import shutil

REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
DEST = os.path.join(HERE, "_ref", "reftests")
FILES = ("conftest.py", "test_grid.py", "test_sobolev.py", "test_energy.py", "test_contour.py",
         "test_optimizer.py", "test_imageio.py")


def stage() -> bool:
    if not os.path.isdir(REF_TESTS):
        return False
    os.makedirs(DEST, exist_ok=True)
    for f in FILES:
        shutil.copyfile(os.path.join(REF_TESTS, f), os.path.join(DEST, f))
    return True


if __name__ == "__main__":
    print("staged" if stage() else "reference absent; nothing staged", DEST)
