"""Drop-in fixtures from the UNMODIFIED reference: the divergence-guard case
of its own test suite (TST/test_gadi.py:83-97) and reference-built problems
(cd3d / cdr2d / crd via gadimp.problems) with their CSR arrays' digests, run
through gadimp.gadi_solve.

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_dropin_golden.py   ->  tests/golden/dropin.json
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from gadimp import GadiConfig, Problem, SparseMatrix, build_cd_3d, build_cdr_2d, build_complex_rd, gadi_solve  # noqa

HERE = Path(__file__).resolve().parent


def digest(a):
    h = hashlib.sha256()
    for arr in (a.row_offsets, a.col_indices, a.values):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


out = {}
# TST/test_gadi.py:83-97 (same construction and seed)
rng = np.random.default_rng(0)
d = np.diag(rng.uniform(1.0, 2.0, 20)) + rng.standard_normal((20, 20))
g = rng.standard_normal((20, 20)) * 50.0
dense = 0.1 * np.eye(20) + 0.5 * (g - g.T)
cfg = {"alpha": 1e-3, "outer_tol": 1e-12, "outer_maxit": 300, "inner_tol": 1e-1}
rep = gadi_solve(Problem(A=SparseMatrix.from_dense(dense), b=np.ones(20), exact_solution=None, label="skewheavy",
                         params={}), cfg=GadiConfig(**cfg))
out["divergence"] = {"dense": dense.tolist(), "cfg": cfg, "status": rep.status, "outer": rep.iterations,
                     "relres": [h.relative_residual for h in rep.history]}
for fam, ng, build, c in (("cd3d", 12, build_cd_3d, {"alpha": 0.5, "u_s": "bf16", "outer_tol": 1e-6}),
                          ("cdr2d", 24, build_cdr_2d, {"alpha": 1.0, "u_s": "fp32", "outer_tol": 1e-10}),
                          ("crd", 12, build_complex_rd, {"alpha": 10.0, "u_s": "bf16", "outer_tol": 1e-6})):
    p = build(ng)
    rep = gadi_solve(p, cfg=GadiConfig(**c))
    out[f"{fam}{ng}"] = {"family": fam, "n_g": ng, "label": p.label, "params": p.params, "cfg": c,
                         "A_sha256": digest(p.A), "nnz": int(p.A.nnz), "status": rep.status, "outer": rep.iterations,
                         "inner_h": [h.inner_h_iterations for h in rep.history],
                         "inner_s": [h.inner_s_iterations for h in rep.history],
                         "x_sha256": hashlib.sha256(np.ascontiguousarray(rep.x).tobytes()).hexdigest()}
    print(fam, rep.status, rep.iterations)
(HERE / "dropin.json").write_text(json.dumps(out))
print("divergence:", out["divergence"]["status"], out["divergence"]["outer"])
