"""The reference's own test suite, replayed against the drop-in.

``oracle/stage_reftests.py`` (run by ``__graft_entry__.build()`` where the
reference exists) stages the unmodified ``pkg/tests`` modules under
``oracle/_ref/reftests``; this test runs them in a fresh interpreter with
``rcseg`` and its submodules bound to ``paper_1403_0240_b200`` — the module
rebinding a user switching packages would do.  Every function they touch
(engine, energy, Sobolev filter, cell list, contour, admissibility,
components, initialisation, image I/O) runs on the B200 through the C ABI.
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGED = os.path.join(ROOT, "oracle", "_ref", "reftests")
MODULES = ("test_grid", "test_sobolev", "test_energy", "test_contour", "test_optimizer",
           "test_imageio")

BOOT = r"""
import importlib, sys
sys.path.insert(0, {root!r})
import paper_1403_0240_b200 as P
sys.modules["rcseg"] = P
for sub in ("grid", "energy", "sobolev", "contour", "optimizer", "synth", "imageio", "report"):
    m = importlib.import_module("paper_1403_0240_b200." + sub)
    sys.modules["rcseg." + sub] = m
    setattr(P, sub, m)
import pytest
sys.exit(pytest.main([{path!r}, "-q", "-p", "no:cacheprovider", "-x", "--rootdir", {staged!r}]))
"""


@pytest.mark.gpu
@pytest.mark.parametrize("module", MODULES)
def test_reference_module_passes_on_drop_in(module):
    path = os.path.join(STAGED, module + ".py")
    if not os.path.exists(path):
        pytest.skip("reference tests not staged (oracle/stage_reftests.py runs in build())")
    code = BOOT.format(root=ROOT, path=path, staged=STAGED)
    r = subprocess.run([sys.executable, "-c", code], cwd=STAGED, capture_output=True, text=True,
                       timeout=1800)
    tail = (r.stdout + r.stderr)[-4000:]
    print(tail)
    assert r.returncode == 0, tail
