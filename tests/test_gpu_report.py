"""A device run's trace and report written through report.py
(report.py:28-59): the emitted JSON carries the run's values unchanged and
agrees with the reference's golden run (run_full_*.npz)."""
import json

import numpy as np
import pytest

from tests.conftest import golden
from tests.test_gpu_parity import P, _engine, close  # noqa: F401

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["full_pc2d", "full_ps2d"])
def test_device_run_report_and_trace(P, tmp_path, name):
    from paper_1403_0240_b200 import report as R
    g = golden(f"run_{name}.npz")
    eng, approx = _engine(P, g)
    res = eng.run()
    R.write_trace(res.trace, tmp_path / "t.jsonl")
    R.write_json(R.build_report(res, {"case": name}, "in.pgm", None), tmp_path / "r.json")
    lines = (tmp_path / "t.jsonl").read_text().splitlines()
    assert len(lines) == res.iterations == int(g["iterations"][0])
    for line, rec in zip(lines, res.trace):
        d = json.loads(line)
        assert list(d) == ["iteration", "energy", "moves", "particles", "mode", "seconds"]
        assert (d["iteration"], d["energy"], d["moves"], d["particles"], d["mode"]) == \
            (rec.iteration, rec.energy, rec.moves, rec.particles, rec.mode)
    if not approx:
        assert [json.loads(s)["energy"] for s in lines] == list(g["energy"])
    rep = json.loads((tmp_path / "r.json").read_text())
    assert rep["status"] == str(g["status"][0])
    fb = -1 if rep["fallback_iteration"] is None else rep["fallback_iteration"]
    assert fb == int(g["fallback"][0])
    assert rep["region_count"] == int(g["regions"][0])
    assert rep["final_energy"]["internal"] == int(g["final"][2])
    assert close(rep["final_energy"]["total"], g["final"][0], 1e-12)
    assert rep["seconds_per_iteration"] == res.wall_seconds / res.iterations
    assert np.isfinite(rep["wall_seconds"]) and rep["input"] == "in.pgm" and rep["output"] is None
