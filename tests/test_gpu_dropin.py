"""The drop-in boundary with objects built the reference's way
(tests/golden/dropin.json, make_dropin_golden.py: the unmodified gadimp).

* A problem whose A is a plain CSR (the reference's SparseMatrix layout) with
  the reference's label / params is recognised as the stencil after a
  whole-CSR bitwise check and solved by the fused kernels: the solve equals
  the reference's run bit for bit (default rounding = the reference's).
* The CSR arrays this package generates for cd3d / cdr2d / crd are the
  reference's (SHA-256 of row offsets, columns, value bits).
* The reference's own divergence-guard case (TST/test_gadi.py:83-97) ends the
  way the reference's run ends.
* The benchmark's parameters with the reference's arithmetic at 512^3: the
  bf16 per-operation emulation cannot resolve the H-system and the outer
  loop trips the divergence guard (relres > 1e3) -- pinned here.
"""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2512_21164_b200 as g
from paper_2512_21164_b200 import sparsemat as M
from paper_2512_21164_b200.problems import Problem
from paper_2512_21164_b200.stencil import recognise

pytestmark = pytest.mark.gpu

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "dropin.json").read_text())
BUILD = {"cd3d": g.build_cd_3d, "cdr2d": g.build_cdr_2d, "crd": g.build_complex_rd}


def _digest(a):
    h = hashlib.sha256()
    for arr in (a.row_offsets, a.col_indices, a.values):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", ["cd3d12", "cdr2d24", "crd12"])
def test_reference_built_problem_is_recognised_and_solved_bitwise(gpu, name):
    c = GOLD[name]
    sp = BUILD[c["family"]](c["n_g"])
    csr = M.SparseMatrix.from_scipy(sp.A.to_scipy())
    assert csr.nnz == c["nnz"] and _digest(csr) == c["A_sha256"], "generated CSR differs from the reference's"
    p = Problem(A=csr, b=sp.b.copy(), exact_solution=np.ones(csr.nrows), label=c["label"], params=c["params"])
    assert recognise(p) is not None
    rep = g.gadi_solve(p, cfg=g.GadiConfig(**c["cfg"]))
    assert rep.status == c["status"] and rep.iterations == c["outer"]
    assert [h.inner_h_iterations for h in rep.history] == c["inner_h"]
    assert [h.inner_s_iterations for h in rep.history] == c["inner_s"]
    assert hashlib.sha256(np.ascontiguousarray(rep.x).tobytes()).hexdigest() == c["x_sha256"]


def test_modified_csr_runs_on_the_csr_engine(gpu):
    c = GOLD["cd3d12"]
    sp = BUILD["cd3d"](12)
    csr = M.SparseMatrix.from_scipy(sp.A.to_scipy())
    v = csr.values.copy()
    v[100] = np.nextafter(v[100], np.inf)
    a = M.SparseMatrix(csr.row_offsets, csr.col_indices, v, csr.shape)
    p = Problem(A=a, b=a.to_scipy() @ np.ones(a.nrows), exact_solution=np.ones(a.nrows), label="cd3d",
                params=c["params"])
    assert recognise(p) is None
    rep = g.gadi_solve(p, cfg=g.GadiConfig(**c["cfg"]), rounding="storage")
    assert rep.status == "Converged" and abs(rep.iterations - c["outer"]) <= 1


def test_divergence_guard_case_matches_reference(gpu):
    c = GOLD["divergence"]
    a = M.SparseMatrix.from_dense(np.array(c["dense"]))
    p = Problem(A=a, b=np.ones(a.nrows), exact_solution=None, label="skewheavy", params={})
    rep = g.gadi_solve(p, cfg=g.GadiConfig(**c["cfg"]))
    assert rep.status == c["status"] and rep.iterations == c["outer"]
    assert rep.status in ("Diverged", "Stagnated", "MaxIt")  # TST/test_gadi.py:97
    np.testing.assert_allclose(rep.relative_residuals[:20], c["relres"][:20], rtol=1e-6)


def test_reference_arithmetic_diverges_at_the_bench_size(gpu):
    cfg = g.GadiConfig(alpha=0.0125, u_s="bf16", strict_model=False, inner_tol=1e-2, outer_tol=1e-12,
                       outer_maxit=12)
    rep = g.gadi_solve(g.build_cd_3d(512), cfg=cfg, rounding="reference", return_x=False, reuse_context=False)
    assert rep.status == "Diverged", rep.status
    assert rep.history[-1].relative_residual > 1e3
    assert rep.history[0].inner_h_iterations > 1000  # the first H-solve already struggles
