"""Initial labelings vs the reference's initialize (tests/golden/init.npz,
make_golden_init.py; optimizer.py:284-405) and CLI usage errors (cli.py:33-38)."""
import numpy as np
import pytest

from paper_1403_0240_b200.init import initialize, otsu_threshold, split_disjoint_labels
from paper_1403_0240_b200.grid import Connectivity
from tests.conftest import golden

HOST_SCHEMES = [0, 1, 2, 3]  # rect, bubbles x2, otsu; maxima blurs on the device (test_gpu_cli)


@pytest.mark.gpu  # split_disjoint_labels labels components on the device
@pytest.mark.parametrize("nd", [2, 3])
@pytest.mark.parametrize("i", HOST_SCHEMES)
def test_initialize_matches_reference(nd, i):
    g = golden("init.npz")
    got = initialize(g[f"img{nd}"], str(g["schemes"][i]))
    assert got.dtype == np.int32
    assert np.array_equal(got, g[f"init{nd}_{i}"])


@pytest.mark.gpu
def test_otsu_and_split_edges():
    assert otsu_threshold(np.zeros(256)) is None
    h = np.zeros(256)
    h[[10, 200]] = 5
    assert 10 <= otsu_threshold(h) < 200
    with pytest.raises(ValueError):
        otsu_threshold(np.zeros(10))
    lab = np.array([[1, 0, 1], [0, 0, 0], [2, 2, 0]])
    assert split_disjoint_labels(lab, Connectivity.default(2)).tolist() == \
        [[1, 0, 2], [0, 0, 0], [3, 3, 0]]
    with pytest.warns(UserWarning):
        assert not initialize(np.full((5, 5), 3.0), "otsu").any()
    for bad in ("bubbles:0", "bubbles:2:0", "bubbles:1:2:3", "maxima:1", "nope"):
        with pytest.raises(ValueError):
            initialize(np.ones((6, 6)), bad)


def test_cli_usage_errors_exit_1(capsys):
    from paper_1403_0240_b200 import cli
    for argv in (["segment"], ["compare", "--input", "x"], ["frobnicate"],
                 ["kernel-table", "--out", "k.csv", "--epsilon", "1/0"]):
        with pytest.raises(SystemExit) as e:
            cli.main(argv)
        assert e.value.code == 1, argv
    assert cli.main(["segment", "--input", "/nonexistent.pgm", "--output", "o.pgm"]) == 1
    assert "rcseg: error:" in capsys.readouterr().err


def test_cli_kernel_table_matches_reference(tmp_path):
    """`kernel-table` (cli.py:207-215) writes the reference's CSV byte for byte."""
    import os
    from paper_1403_0240_b200 import cli
    out = tmp_path / "k.csv"
    assert cli.main(["kernel-table", "--E", "9", "--epsilon", "1/30", "--samples", "101",
                     "--out", str(out)]) == 0
    with open(os.path.join(os.path.dirname(__file__), "golden", "cli", "kernel.csv"), "rb") as fh:
        assert out.read_bytes() == fh.read()
