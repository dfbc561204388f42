"""Trace output in the reference's JSON schema (reporting.py:50-75 of the reference).

Only the data half of the reference's reporting module: the figures need matplotlib, which
the reference's own import requires (and which is not part of the hot path).  The payload keys,
value types, ``indent=2, sort_keys=True`` formatting and the quarantined ``"timing"`` entry are
the reference's, so a trace written here diffs cleanly against one written by the reference
(apart from the wall times).
"""

from __future__ import annotations

import json
from pathlib import Path

from .mgrit import IterationTrace, convergence_factor

__all__ = ["trace_payload", "write_json", "write_trace"]


def write_json(path, payload) -> Path:
    """reporting.py:50-56: pretty-printed, sorted keys, trailing newline; parent directories created."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    with open(path, "w") as fh:
        json.dump(payload, fh, indent=2, sort_keys=True)
        fh.write("\n")
    return path


def trace_payload(trace: IterationTrace, config: dict) -> dict:
    """reporting.py:59-75: the iteration trace as JSON-ready data; timing is segregated."""
    payload = {
        "config": config,
        "seed": trace.seed,
        "converged": trace.converged,
        "iterations": trace.iterations,
        "residual_norms": [float(r) for r in trace.residual_norms],
        "spatial_solves": [int(v) for v in trace.spatial_solves],
        "cg_iterations": [int(v) for v in trace.cg_iterations],
        "timing": {"wall_times": [float(t) for t in trace.wall_times]},
    }
    if len(trace.residual_norms) >= 6:
        payload["convergence_factor"] = float(convergence_factor(trace))
    return payload


def write_trace(path, trace: IterationTrace, config: dict) -> Path:
    """The JSON half of the reference's ``solve_report`` (reporting.py:86-97)."""
    return write_json(path, trace_payload(trace, config))
