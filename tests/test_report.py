"""Report formats (CPU): the JSONL trace / CSV summary layouts of the
reference CLI (REF/cli.py:74-86, 320-338) built from a SolveReport."""

import csv
import json

import numpy as np

from paper_2512_21164_b200 import GadiConfig, IterationRecord, SolveReport
from paper_2512_21164_b200 import report as R


class _P:
    label, n = "cd3d", 8


def _rep():
    hist = [IterationRecord(k, 1.0 / (k + 1), 0.1 / (k + 1), 1e-3, 1e-2, 0.5, 3, 2, False) for k in range(3)]
    return SolveReport(x=np.ones(8), status="Converged", history=hist, wallclock={})


def test_trace_records_keys(tmp_path):
    p = R.write_trace(tmp_path / "t.jsonl", _rep())
    recs = [json.loads(line) for line in p.read_text().splitlines()]
    assert len(recs) == 3 and recs[0]["schema_version"] == 1
    assert set(recs[0]) == {"schema_version", "k", "residual_norm", "relative_residual", "backward_error",
                            "forward_error", "mu", "inner_h_iterations", "inner_s_iterations", "inner_breakdown"}


def test_summary_csv(tmp_path):
    cfg = GadiConfig(alpha=0.5, u_s="bf16")
    path = tmp_path / "summary.csv"
    R.append_summary(path, _P(), cfg, _rep(), 1.25, 0)
    R.append_summary(path, _P(), cfg, _rep(), 1.5, 1, gpu={"n_gpus": 1, "device_time_s": 1.0})
    rows = list(csv.reader(path.open()))
    assert rows[0] == R.SUMMARY_COLUMNS
    assert rows[1][:9] == ["1", "cd3d", "8", "0.5", "1.0", "bf16", "fp64", "fp64", "Converged"]
    assert rows[2][-4:-2] == ["1", "1.0"]
