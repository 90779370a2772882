"""Golden runs of the UNMODIFIED reference at the benchmark's parameters.

The bench workload (bench.py) is cd3d with alpha = 0.0125, u_s = bf16,
strict_model = False, inner_tol = 1e-2, omega = 1, u = u_r = fp64.  The
reference cannot hold n = 512^3, so it is run here at n_g = 32, 64 (400 outer
steps: MaxIt on both precisions) and at n_g = 128, 256 for the first outer
steps (outer_maxit caps the run), recording every per-step quantity the GPU
tests compare: relres / berr / ferr / mu, inner H and S counts, and a
SHA-256 of the final iterate's bytes (bitwise check of the fused
reference-rounding path).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_headline_golden.py --case headline_cd3d32_bf16

writes tests/golden/headline_<case>.json.  Slow: the reference emulates
bf16 per operation in numpy (64^3 takes about an hour, 256^3 several).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import gadimp  # noqa: E402
from gadimp import GadiConfig, build_cd_3d, gadi_solve  # noqa: E402

HERE = Path(__file__).resolve().parent

BENCH_CFG = {"alpha": 0.0125, "u_s": "bf16", "strict_model": False, "inner_tol": 1e-2, "omega": 1.0,
             "outer_tol": 1e-12}

CASES = {
    "headline_cd3d32_bf16": (32, {**BENCH_CFG, "outer_maxit": 400}),
    "headline_cd3d32_fp64": (32, {**BENCH_CFG, "u_s": "fp64", "outer_maxit": 400}),
    "headline_cd3d64_bf16": (64, {**BENCH_CFG, "outer_maxit": 400}),
    "headline_cd3d128_bf16": (128, {**BENCH_CFG, "outer_maxit": 30}),
    "headline_cd3d256_bf16": (256, {**BENCH_CFG, "outer_maxit": 4}),
}


def run(name):
    n_g, cfg = CASES[name]
    p = build_cd_3d(n_g)
    t0 = time.perf_counter()
    rep = gadi_solve(p, cfg=GadiConfig(**cfg))
    wall = time.perf_counter() - t0
    h = rep.history
    x = np.ascontiguousarray(rep.x, dtype=np.float64)
    return {
        "name": name, "family": "cd3d", "n_g": n_g, "cfg": cfg,
        "status": rep.status, "outer": rep.iterations, "inner": rep.total_inner_iterations,
        "inner_h": [r.inner_h_iterations for r in h], "inner_s": [r.inner_s_iterations for r in h],
        "relres": [r.relative_residual for r in h], "berr": [r.backward_error for r in h],
        "ferr": [r.forward_error for r in h], "mu": [r.mu for r in h],
        "residual_norm": [r.residual_norm for r in h],
        "norm_A": rep.norm_A, "wall_s": wall,
        "x_sha256": hashlib.sha256(x.tobytes()).hexdigest(), "x_head": x[:8].tolist(),
        "x_norm": float(np.linalg.norm(x)), "gadimp": gadimp.__version__,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", choices=sorted(CASES), required=True)
    a = ap.parse_args()
    r = run(a.case)
    (HERE / f"{a.case}.json").write_text(json.dumps(r))
    print(f"{a.case}: {r['status']} outer={r['outer']} inner={r['inner']} relres={r['relres'][-1]:.3e} "
          f"{r['wall_s']:.0f}s", flush=True)


if __name__ == "__main__":
    main()
