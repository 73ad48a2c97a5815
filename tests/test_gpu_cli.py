"""The device CLI reproduces the reference CLI's files
(tests/golden/cli/, make_golden_init.py running rcseg.cli): `compare`
(pc/gauss, L2 vs Sobolev: label files, report, energy/moves CSV — SURVEY
8(f) row 4) and `segment` (ps/poisson, otsu init: labels, overlay, trace,
report).  Wall-clock fields are excluded; Poisson energies to rtol 1e-12."""
import json
import os
import shutil

import numpy as np
import pytest

from tests.conftest import golden
from tests.test_gpu_parity import P, close  # noqa: F401

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "cli")
TIMES = {"wall_seconds", "seconds_per_iteration", "seconds_per_iteration_ratio", "rc_threads",
         "seconds"}


def _strip(d):
    if isinstance(d, dict):
        return {k: _strip(v) for k, v in d.items() if k not in TIMES}
    return d


def _gold(name):
    with open(os.path.join(GOLD, name), "rb") as fh:
        return fh.read()


def test_initialize_maxima_matches_reference(P):
    from paper_1403_0240_b200.init import initialize
    g = golden("init.npz")
    for nd in (2, 3):
        assert np.array_equal(initialize(g[f"img{nd}"], str(g["schemes"][4])), g[f"init{nd}_4"])


def test_cli_compare_and_segment_match_reference(P, tmp_path, monkeypatch):
    from paper_1403_0240_b200 import cli
    shutil.copy(os.path.join(GOLD, "in.pgm"), tmp_path / "in.pgm")
    monkeypatch.chdir(tmp_path)
    common = ["--input", "in.pgm", "--max-iter", "60", "--lambda", "0.5"]
    rc = cli.main(["compare", *common, "--init", "bubbles:3", "--output-prefix", "cmp",
                   "--report", "cmp.json"])
    rc2 = cli.main(["segment", *common, "--model", "ps", "--noise", "poisson", "--smooth-radius", "3",
                    "--init", "otsu", "--output", "seg.pgm", "--overlay", "seg_overlay.pgm",
                    "--trace", "seg.jsonl", "--report", "seg.json"])
    assert f"{rc} {rc2}\n" == _gold("exit_codes.txt").decode()
    for f in ("cmp-l2.pgm", "cmp-sobolev.pgm", "cmp.csv", "seg.pgm", "seg_overlay.pgm"):
        assert (tmp_path / f).read_bytes() == _gold(f), f
    got, want = json.loads((tmp_path / "cmp.json").read_text()), json.loads(_gold("cmp.json"))
    assert _strip(got) == _strip(want)
    got, want = json.loads((tmp_path / "seg.json").read_text()), json.loads(_gold("seg.json"))
    ge, we = got.pop("final_energy"), want.pop("final_energy")
    assert _strip(got) == _strip(want)
    assert ge["internal"] == we["internal"]
    assert close(ge["total"], we["total"]) and close(ge["external"], we["external"])
    lines = (tmp_path / "seg.jsonl").read_text().splitlines()
    wlines = _gold("seg.jsonl").decode().splitlines()
    assert len(lines) == len(wlines)
    for a, b in zip(lines, wlines):
        a, b = json.loads(a), json.loads(b)
        assert close(a.pop("energy"), b.pop("energy"))
        assert _strip(a) == _strip(b)


def test_cli_particles_csv_matches_reference(P, tmp_path, monkeypatch):
    """--particles-csv (cli.py:117-127): every iteration's candidates with
    their filtered rank values, same rows as the reference's (pc/gauss:
    bit-exact values); compared per iteration as row sets."""
    from paper_1403_0240_b200 import cli
    shutil.copy(os.path.join(GOLD, "in.pgm"), tmp_path / "in.pgm")
    monkeypatch.chdir(tmp_path)
    assert cli.main(["segment", "--input", "in.pgm", "--max-iter", "3", "--lambda", "0.5", "--init",
                     "bubbles:3", "--output", "p.pgm", "--particles-csv", "particles.csv"]) == 2
    got = (tmp_path / "particles.csv").read_text().splitlines()
    want = _gold("particles.csv").decode().splitlines()
    assert got[0] == want[0] and len(got) == len(want)
    assert sorted(got[1:]) == sorted(want[1:])
