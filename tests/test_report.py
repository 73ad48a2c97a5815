"""Report / trace emission vs the reference's own bytes (tests/golden/report/,
made by make_golden_report.py running rcseg.report; report.py:21-71)."""
import json
import os
from dataclasses import dataclass

import pytest

from paper_1403_0240_b200 import report as R
from paper_1403_0240_b200.energy import EnergyValue
from paper_1403_0240_b200.optimizer import IterationRecord, RunResult

GOLD = os.path.join(os.path.dirname(__file__), "golden", "report")


def _read(name):
    with open(os.path.join(GOLD, name), "rb") as fh:
        return fh.read()


def _cases():
    trace = [IterationRecord(0, 1234.5678901234, 311, 4021, "sobolev", 0.0012345),
             IterationRecord(1, 1100.0, 250, 3980, "sobolev", 0.001),
             IterationRecord(2, -3.25e-7, 0, 17, "l2", 1e-5),
             IterationRecord(3, 99.99999999999999, 1, 2, "l2", 0.5)]
    yield ("mixed", RunResult(None, trace, "converged", 4, 0.0312345678,
                              EnergyValue(99.99999999999999, 80.5, 19.499999999999993), 3, 2),
           {"seed": 0, "gradient": "sobolev", "radius": 4, "lambda": 0.04}, "in.pgm", "out.pgm")
    yield ("empty", RunResult(None, [], "max_iterations", 0, 0.0, EnergyValue(0.0, 0.0, 0.0), 1, None),
           {"seed": 7}, None, None)


@pytest.mark.parametrize("case", list(_cases()), ids=lambda c: c[0])
def test_trace_and_report_bytes_match_reference(tmp_path, case):
    name, result, echo, inp, outp = case
    R.write_trace(result.trace, tmp_path / "t.jsonl")
    R.write_json(R.build_report(result, echo, inp, outp), tmp_path / "r.json")
    assert (tmp_path / "t.jsonl").read_bytes() == _read(f"{name}.trace.jsonl")
    assert (tmp_path / "r.json").read_bytes() == _read(f"{name}.report.json")
    assert not [p for p in os.listdir(tmp_path) if p.startswith(".tmp-rcseg-")]


def test_csv_and_figure_path_match_reference(tmp_path):
    R.write_csv(tmp_path / "t.csv", ["gradient", "iterations", "seconds", "energy"],
                [["sobolev", 40, 0.125, 1234.5678901234], ["l2", 1000, 3.0, -0.0],
                 ["x y", 0, 1e-9, 1e20]])
    assert (tmp_path / "t.csv").read_bytes() == _read("table.csv")
    manifest = json.loads(_read("manifest.json"))
    for p, want in manifest["figure_path"].items():
        assert R.figure_path(p) == want


def test_atomic_write_leaves_target_on_failure(tmp_path):
    target = tmp_path / "r.json"
    target.write_text("old\n")

    class Bad:
        pass
    with pytest.raises(TypeError):
        R.write_json({"x": Bad()}, target)
    assert target.read_text() == "old\n"
    assert not [p for p in os.listdir(tmp_path) if p.startswith(".tmp-rcseg-")]
