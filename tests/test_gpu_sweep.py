"""Sweep workload: K6 on device-generated sphere-union contours against the
oracle (bit-exact outputs and interaction counts)."""
import numpy as np
import pytest

from oracle import rc_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,nsph,width", [((48, 40, 44), 6, 1), ((48, 40, 44), 6, 2),
                                              ((40, 36, 32), 4, 4), ((128, 120), 20, 3),
                                              ((32, 32, 32), 3, 8)])
def test_sweep_k6_matches_oracle(shape, nsph, width):
    from paper_1403_0240_b200.sweep import SobolevSweep
    sw = SobolevSweep(shape, nsph, width, seed=3)
    assert sw.n_particles > 100
    pairs, ms = sw.run()
    xs, ow, cm, raw, out = sw.get()
    coords = np.stack(np.unravel_index(xs, shape), axis=1)
    want = O.sobolev_filter(coords, ow, cm, raw, 2.0 * width)
    assert np.array_equal(out, want)
    assert pairs == O.pair_count(coords, 2.0 * width)
    # the particle set is the contour of the painted volume
    assert np.all(np.diff(xs) >= 0)
