"""Device synthetic-data pipeline (paper_1403_0240_b200/synth.py, csrc/synth.cu)
against the reference's own outputs (tests/golden/synth.npz): render, blur,
poissonize and generate bit for bit; plus a 128^3 scene checked against the
CPU restatement (blur in full, Poisson draws on a random sample of voxels)."""
import json

import numpy as np
import pytest

from oracle import synth_oracle as SO
from tests.conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_1403_0240_b200 import _lib, synth
    if _lib.device_count() < 1:
        pytest.fail("no CUDA device visible to librcseg_b200")
    return synth


def test_synth_matches_reference_golden(S):
    g = golden("synth.npz")
    specs = json.loads(bytes(g["specs_json"]).decode())
    for name, d in specs.items():
        spec = S.scene_from_dict(d)
        labels, image = S.generate(spec)
        assert np.array_equal(labels, g[f"{name}_labels"]), name
        assert np.array_equal(image, g[f"{name}_noisy"]), name
        lab2, clean = S.render_scene(spec)
        assert np.array_equal(lab2, g[f"{name}_labels"]) and np.array_equal(clean, g[f"{name}_clean"])
        assert np.array_equal(S.blur(clean, spec.blur_sigma), g[f"{name}_blurred"]), name
        assert np.array_equal(S.poissonize(g[f"{name}_blurred"], spec.noise), g[f"{name}_noisy"])
        assert S.scene_to_dict(spec) == d


def test_synth_errors(S):
    with pytest.raises(ValueError):
        S.poissonize(-np.ones((4, 4)), S.NoiseSpec(3.0, 1))
    with pytest.raises(ValueError):
        S.blur(np.zeros((4, 4)), -0.5)
    with pytest.raises(ValueError):
        S.generate(S.SceneSpec(dims=(8, 8), shapes=[S.Shape(kind="star", intensity=1.0)]))
    with pytest.raises(ValueError):
        S.generate(S.SceneSpec(dims=(8,)))
    with pytest.raises(ValueError):
        S.NoiseSpec(0.0, 1)
    assert not S.poissonize(np.zeros((5, 5)), S.NoiseSpec(3.0, 1)).any()


def test_synth_large_volume_vs_oracle(S):
    rng = np.random.default_rng(17)
    shapes = [S.Shape(kind="disk", center=tuple(rng.uniform(10, 118, 3)), radius=float(rng.uniform(5, 25)),
                      intensity=float(rng.uniform(0.5, 1.0))) for _ in range(12)]
    shapes.append(S.Shape(kind="annulus", center=(64, 64, 64), inner=20.0, outer=26.5, intensity=0.8))
    shapes.append(S.Shape(kind="rect", origin=(0, 100, 5), size=(30, 20, 60), intensity=0.6))
    spec = S.SceneSpec(dims=(128, 128, 128), background=0.1, shapes=shapes, blur_sigma=1.5,
                       noise=S.NoiseSpec(psnr=float(np.sqrt(30.0)), seed=4))
    d = S.scene_to_dict(spec)
    labels, clean = S.render_scene(spec)
    ol, oc = SO.render_scene(d)
    assert np.array_equal(labels, ol) and np.array_equal(clean, oc)
    blurred = S.blur(clean, 1.5)
    assert np.array_equal(blurred, SO.blur(oc, 1.5))
    noisy = S.poissonize(blurred, spec.noise)
    _, gen = S.generate(spec)
    assert np.array_equal(gen, noisy)
    scale = 30.0 / float(blurred.max())
    idx = rng.choice(blurred.size, 3000, replace=False)
    flat_b, flat_n = blurred.ravel(), noisy.ravel()
    for i in idx:
        assert flat_n[i] == SO.poisson_draw(float(flat_b[i] * scale), SO.Stream(4, int(i))), i
