"""The CPU restatement of the synthetic-data pipeline (oracle/synth_oracle.py)
against the reference's own outputs (tests/golden/synth.npz): bit for bit."""
import json

import numpy as np
import pytest

from oracle import synth_oracle as SO
from tests.conftest import golden


def _specs(g):
    return json.loads(bytes(g["specs_json"]).decode())


def test_oracle_synth_matches_reference():
    g = golden("synth.npz")
    for name, spec in _specs(g).items():
        labels, clean = SO.render_scene(spec)
        assert np.array_equal(labels, g[f"{name}_labels"]), name
        assert np.array_equal(clean, g[f"{name}_clean"]), name
        blurred = SO.blur(clean, spec["blur_sigma"])
        assert np.array_equal(blurred, g[f"{name}_blurred"]), name
        noisy = SO.poissonize(blurred, spec["noise"]["psnr"], spec["noise"]["seed"])
        assert np.array_equal(noisy, g[f"{name}_noisy"]), name


def test_oracle_synth_errors():
    with pytest.raises(ValueError):
        SO.blur(np.zeros((4, 4)), -1.0)
    with pytest.raises(ValueError):
        SO.poissonize(-np.ones((2, 2)), 3.0, 0)
    assert not SO.poissonize(np.zeros((3, 3)), 3.0, 0).any()
