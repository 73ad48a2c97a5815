"""Run reports and iteration traces (mirror of rcseg.report, report.py:21-71).

A run's ``RunResult`` (optimizer.py) becomes a JSON report with a config echo
and a JSON-lines trace, one record per iteration, in exactly the reference's
byte format: ``json.dumps`` with default separators, a 2-space indented report
and a trailing newline, written atomically (temp file in the target directory,
then ``os.replace``; imageio.py:42-55).  ``tests/golden/report/`` holds the
reference's own output for a fixed trace (``make_golden_report.py``).

Not mirrored: the companion PNG figures (``render_energy_figure`` and
friends, report.py:74+) — matplotlib is not in this image; ``figure_path``
is kept so callers can name them.
"""
from __future__ import annotations

import json
import os
import tempfile

ARTIFACT_VERSION = "0.1.0"


def _atomic_write_bytes(path, data: bytes) -> None:
    """imageio.py:42-55: write beside the target, then rename over it."""
    path = os.fspath(path)
    fd, tmp = tempfile.mkstemp(dir=os.path.dirname(path) or ".", prefix=".tmp-rcseg-")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(data)
        os.replace(tmp, path)
    except BaseException:
        try:
            os.unlink(tmp)
        except OSError:
            pass
        raise


def write_json(obj: dict, path) -> None:
    """report.py:24-25"""
    _atomic_write_bytes(path, (json.dumps(obj, indent=2) + "\n").encode())


def trace_records(trace) -> list[dict]:
    """report.py:28-31: one dict per IterationRecord, fields in this order."""
    keys = ("iteration", "energy", "moves", "particles", "mode", "seconds")
    return [{k: getattr(rec, k) for k in keys} for rec in trace]


def write_trace(trace, path) -> None:
    """report.py:34-36: JSON lines; an empty trace is a single newline."""
    body = "\n".join(json.dumps(rec) for rec in trace_records(trace))
    _atomic_write_bytes(path, (body + "\n").encode())


def build_report(result, config_echo: dict, input_path: str | None,
                 output_path: str | None) -> dict:
    """report.py:39-59; seconds_per_iteration is 0.0 for a zero-iteration run."""
    n = result.iterations
    energy = result.final_energy
    return {
        "artifact_version": ARTIFACT_VERSION,
        "status": result.status,
        "iterations": n,
        "fallback_iteration": result.fallback_iteration,
        "wall_seconds": result.wall_seconds,
        "seconds_per_iteration": result.wall_seconds / n if n else 0.0,
        "final_energy": {"total": energy.total, "external": energy.external,
                         "internal": energy.internal},
        "region_count": result.region_count,
        "input": input_path,
        "output": output_path,
        "config": config_echo,
    }


def write_csv(path, header: list[str], rows) -> None:
    """report.py:62-66: comma-joined ``str`` of each value, no quoting."""
    lines = [",".join(header)] + [",".join(str(v) for v in row) for row in rows]
    _atomic_write_bytes(path, ("\n".join(lines) + "\n").encode())


def figure_path(path) -> str:
    """report.py:69-71: the companion figure's name (same stem, .png)."""
    return os.path.splitext(os.fspath(path))[0] + ".png"
