"""Golden fixtures of the reference's run-report / trace emission
(rcseg.report: write_trace, build_report + write_json, write_csv), made by
running the REFERENCE itself in the build container:

    python tests/golden/make_golden_report.py

matplotlib is absent from this image, so a stub module stands in for it; the
functions fixed here never touch it (only the render_* figure helpers do).
Cases: a mixed sobolev/l2 trace with a fallback, an empty trace (zero
iterations: seconds_per_iteration 0.0, file is one newline), a CSV table with
ints, floats and strings, and figure_path on a few names.
"""
from __future__ import annotations

import json
import os
import sys
import types
from dataclasses import dataclass

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "report")
sys.path.insert(0, "/root/reference/pkg/src")

_mpl = types.ModuleType("matplotlib")
_mpl.use = lambda *a, **k: None
_mpl.pyplot = types.ModuleType("matplotlib.pyplot")
sys.modules.setdefault("matplotlib", _mpl)
sys.modules.setdefault("matplotlib.pyplot", _mpl.pyplot)

from rcseg import report as R  # noqa: E402


@dataclass
class Rec:
    iteration: int
    energy: float
    moves: int
    particles: int
    mode: str
    seconds: float


@dataclass
class Energy:
    total: float
    external: float
    internal: float


@dataclass
class Result:
    trace: list
    status: str
    iterations: int
    wall_seconds: float
    final_energy: Energy
    region_count: int
    fallback_iteration: object = None


def cases():
    trace = [Rec(0, 1234.5678901234, 311, 4021, "sobolev", 0.0012345),
             Rec(1, 1100.0, 250, 3980, "sobolev", 0.001),
             Rec(2, -3.25e-7, 0, 17, "l2", 1e-5),
             Rec(3, 99.99999999999999, 1, 2, "l2", 0.5)]
    yield "mixed", Result(trace, "converged", 4, 0.0312345678, Energy(99.99999999999999, 80.5, 19.499999999999993), 3, 2), \
        {"seed": 0, "gradient": "sobolev", "radius": 4, "lambda": 0.04}, "in.pgm", "out.pgm"
    yield "empty", Result([], "max_iterations", 0, 0.0, Energy(0.0, 0.0, 0.0), 1, None), \
        {"seed": 7}, None, None


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    manifest = {"figure_path": {}}
    for name, result, echo, inp, outp in cases():
        R.write_trace(result.trace, os.path.join(OUT, f"{name}.trace.jsonl"))
        R.write_json(R.build_report(result, echo, inp, outp), os.path.join(OUT, f"{name}.report.json"))
    R.write_csv(os.path.join(OUT, "table.csv"), ["gradient", "iterations", "seconds", "energy"],
                [["sobolev", 40, 0.125, 1234.5678901234], ["l2", 1000, 3.0, -0.0], ["x y", 0, 1e-9, 1e20]])
    for p in ["run.json", "dir/run.report.json", "noext", "a.b/c"]:
        manifest["figure_path"][p] = R.figure_path(p)
    with open(os.path.join(OUT, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)


if __name__ == "__main__":
    main()
