"""Outer-loop fixtures of the STORAGE MODEL (the paper's GPU arithmetic:
u_s storage, fp32 compute) from the CPU oracle's
restatement of it (oracle/gadi_oracle.py gadi_solve(..., rounding="storage")).

The reference package has no storage model -- it emulates every operation in
u_s (its rounding is what gadi_solve(..., rounding="reference") reproduces
bitwise, tests/golden/solves.json).  The storage-model GPU solves are
compared with these fixtures (status, outer count +-1, +-0 all-fp64,
backward error within 2x): same problems and configurations as
solves.json.

    python tests/golden/make_storage_golden.py   ->  tests/golden/solves_storage.json
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
from oracle import gadi_oracle as O  # noqa: E402


def run(c):
    cfg = dict(c["cfg"])
    op = O.build(c["family"], c["n_g"], **c.get("kw", {}))
    t0 = time.perf_counter()
    r = O.gadi_solve(op, O.rhs_ones(op), cfg["alpha"], omega=cfg.get("omega", 1.0), u=cfg.get("u", "fp64"),
                     u_r=cfg.get("u_r", "fp64"), u_s=cfg.get("u_s", "fp64"), outer_tol=cfg.get("outer_tol", 1e-10),
                     outer_maxit=cfg.get("outer_maxit", 2000), inner_tol=cfg.get("inner_tol", 1e-4),
                     strict=cfg.get("strict_model", True), exact=np.ones(op.n), norm_a=c["norm_A"],
                     rounding="storage")
    h = r.history
    return {"name": c["name"], "family": c["family"], "n_g": c["n_g"], "kw": c.get("kw", {}), "cfg": c["cfg"],
            "status": r.status, "outer": len(h), "inner_h": [x.inner_h for x in h], "inner_s": [x.inner_s for x in h],
            "relres": [x.relative_residual for x in h], "berr": [x.backward_error for x in h],
            "norm_A": c["norm_A"], "wall_s": time.perf_counter() - t0}


def main():
    cases = json.loads((HERE / "solves.json").read_text())
    out = []
    for c in cases:
        r = run(c)
        print(f"{r['name']}: {r['status']} outer={r['outer']} (reference {c['outer']}) {r['wall_s']:.1f}s", flush=True)
        out.append(r)
    (HERE / "solves_storage.json").write_text(json.dumps(out))


if __name__ == "__main__":
    main()
