"""Bench / trace report formats of the reference CLI:
the per-iteration JSONL trace records (REF/cli.py:74-86) and the CSV summary
row of ``gadi-mp bench`` (REF/cli.py:320-338), both with
``schema_version = 1`` so existing tooling reads them, plus optional GPU
columns appended after the reference's."""

from __future__ import annotations

import csv
import json
from pathlib import Path

SCHEMA_VERSION = 1

SUMMARY_COLUMNS = ["schema_version", "problem", "n", "alpha", "omega", "u_s", "u", "u_r", "status",
                   "outer_iterations", "inner_iterations", "final_relative_residual", "final_backward_error",
                   "final_forward_error", "wall_time_s", "repeat_index"]
GPU_COLUMNS = ["n_gpus", "device_time_s", "achieved_gbs", "roofline_frac"]

__all__ = ["SCHEMA_VERSION", "SUMMARY_COLUMNS", "GPU_COLUMNS", "history_records", "write_trace", "append_summary"]


def history_records(report) -> list[dict]:
    """One dict per outer iteration, the keys of REF/cli.py:74-86."""
    return [{"schema_version": SCHEMA_VERSION, "k": h.k, "residual_norm": h.residual_norm,
             "relative_residual": h.relative_residual, "backward_error": h.backward_error,
             "forward_error": h.forward_error, "mu": h.mu, "inner_h_iterations": h.inner_h_iterations,
             "inner_s_iterations": h.inner_s_iterations, "inner_breakdown": h.inner_breakdown}
            for h in report.history]


def write_trace(path, report) -> Path:
    path = Path(path)
    with path.open("w") as f:
        for rec in history_records(report):
            f.write(json.dumps(rec) + "\n")
    return path


def append_summary(path, problem, cfg, report, wall_time_s: float, repeat_index: int = 0, gpu: dict | None = None):
    """Append one summary row (header written for a new file); ``gpu`` adds
    the GPU_COLUMNS after the reference's columns."""
    path = Path(path)
    new = not path.exists()
    h = report.history[-1]
    row = [SCHEMA_VERSION, problem.label, problem.n, cfg.alpha, cfg.omega, cfg.u_s.name, cfg.u.name, cfg.u_r.name,
           report.status, report.iterations, report.total_inner_iterations, h.relative_residual, h.backward_error,
           h.forward_error, wall_time_s, repeat_index]
    cols = SUMMARY_COLUMNS + (GPU_COLUMNS if gpu is not None else [])
    if gpu is not None:
        row += [gpu.get(k) for k in GPU_COLUMNS]
    with path.open("a", newline="") as f:
        w = csv.writer(f)
        if new:
            w.writerow(cols)
        w.writerow(row)
    return path
