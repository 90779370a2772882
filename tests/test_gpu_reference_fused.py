"""The reference's per-operation rounding inside the fused passes
(gadi_solve(..., rounding="reference"), csrc/strict.cuh).

Bar: bitwise.  The fused passes restate gadimp's round-after-every-op
emulation (precision.py:176-220, sparsemat.py:178-199, inner.py:39-143) in
the streaming stencil kernels, with fl_dot's pairwise tree split at aligned
power-of-two blocks (lane vector, warp butterfly, tree finisher).  They are
compared against

* the per-operation form of the same emulation (rounding="reference_host",
  csrc/exact.cu: one launch per operation, the pairwise tree level by level),
  which is itself pinned bitwise to the reference's golden iterates
  (tests/test_gpu_solve.py);
* the unmodified reference run at the benchmark's own parameters
  (tests/golden/headline_*.json, tests/golden/make_headline_golden.py):
  every per-step inner count and the final iterate's SHA-256.

Shapes are chosen to hit every leaf granularity of the tree: one leaf per
element (rows that are not 16-byte aligned: register-path sweeps), per lane
vector, and per 2..32-lane warp block (G = min(2^v2(nz), 32 VZ)).
"""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2512_21164_b200 as g

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"
BUILD = {"cdr2d": g.build_cdr_2d, "cd3d": g.build_cd_3d, "crd": g.build_complex_rd}


def _bits(x):
    return np.asarray(x, dtype=np.float64).view(np.uint64)


CROSS = [
    # family, n_g, u_s, strict_model, alpha
    ("cd3d", 16, "bf16", False, 0.5),     # nz 16: 2-lane blocks
    ("cd3d", 64, "bf16", False, 0.0125),  # nz 64: 8-lane blocks, the headline regime
    ("cd3d", 64, "bf16", True, 0.5),      # bf16 dot tree (strict_model)
    ("cd3d", 32, "fp32", True, 0.5),      # fp32: VZ 4, 8-lane blocks
    ("cd3d", 12, "bf16", False, 0.5),     # 24-byte rows: register path, one leaf per element
    ("cd3d", 24, "fp16", False, 0.5),     # fp16, 48-byte rows: lane-vector leaves
    ("cdr2d", 256, "bf16", False, 1.0),   # 2-D rows of 64 lanes: 32-lane blocks
    ("cdr2d", 100, "fp32", True, 1.0),    # nz 100: 4-element leaves
    ("cdr2d", 37, "bf16", True, 1.0),     # odd rows
    ("crd", 32, "bf16", False, 10.0),     # interleaved complex H sweeps + pointwise S
    ("crd", 24, "fp32", True, 10.0),
]


@pytest.mark.parametrize("fam,ng,us,strict,alpha", CROSS)
def test_fused_reference_equals_per_operation(gpu, fam, ng, us, strict, alpha):
    cfg = g.GadiConfig(alpha=alpha, u_s=us, strict_model=strict, outer_tol=0.0, outer_maxit=6,
                       inner_tol=1e-2 if alpha < 0.1 else 1e-4)
    a = g.gadi_solve(BUILD[fam](ng), cfg=cfg, rounding="reference", reuse_context=False)
    b = g.gadi_solve(BUILD[fam](ng), cfg=cfg, rounding="reference_host", reuse_context=False)
    assert [h.inner_h_iterations for h in a.history] == [h.inner_h_iterations for h in b.history]
    assert [h.inner_s_iterations for h in a.history] == [h.inner_s_iterations for h in b.history]
    assert np.array_equal(a.x, b.x), "fused reference rounding differs from the per-operation form"
    np.testing.assert_array_equal(a.relative_residuals, b.relative_residuals)


@pytest.mark.parametrize("fam,ng,us", [("cd3d", 64, "bf16"), ("cdr2d", 256, "fp16"), ("crd", 32, "bf16")])
def test_fused_reference_inner_solvers(gpu, fam, ng, us):
    """cg_spd / cg_normal_skew with rounding="reference" (fused) equal the
    per-operation form bitwise on a random right-hand side."""
    p = BUILD[fam](ng)
    sp = g.make_hss_splitting(p.A, 0.5 if fam != "crd" else 10.0, us)
    rng = np.random.default_rng(5)
    rhs = g.quantize(rng.standard_normal(p.n) / 4.0, us)
    for strict in (True, False):
        z1, s1 = g.cg_spd(sp.H_low, rhs, 1e-4, 300, us, strict, rounding="reference")
        z2, s2 = g.cg_spd(sp.H_low, rhs, 1e-4, 300, us, strict, rounding="reference_host")
        assert s1.iterations == s2.iterations and np.array_equal(z1, z2)
        y1, t1 = g.cg_normal_skew(sp.S_low, rhs, 1e-4, 300, us, strict, sp.S_low_T, rounding="reference")
        y2, t2 = g.cg_normal_skew(sp.S_low, rhs, 1e-4, 300, us, strict, sp.S_low_T, rounding="reference_host")
        assert t1.iterations == t2.iterations and np.array_equal(y1, y2)


def test_packed_stencil_subnormals(gpu):
    """The packed bf16x2 / f16x2 reference stencil (strict.cuh, SASS HFMA2.BF16
    / HADD2) keeps subnormal products and sums: y = Op x on inputs scaled into
    the subnormal range equals the oracle's per-operation spmv."""
    from oracle import gadi_oracle as O

    for us, scale in (("bf16", 2.0 ** -128), ("fp16", 2.0 ** -16)):
        p = g.build_cd_3d(16)
        sp = g.make_hss_splitting(p.A, 0.75, us)
        rng = np.random.default_rng(11)
        x = g.quantize(rng.standard_normal(p.n) * scale, us)
        assert np.count_nonzero(np.abs(x) < (1.2e-38 if us == "bf16" else 6.1e-5)) > 0
        op = O.cd3d(16)
        H, S, ST = O.splitting(op, 0.75, us)
        for mat, ref in ((sp.H_low, H), (sp.S_low, S), (sp.S_low_T, ST)):
            y = g.spmv(mat, x, us)
            yo = O.stencil_apply(ref, x, us)
            assert np.array_equal(_bits(y), _bits(yo)) or np.array_equal(y, yo), us


# ---------------------------------------------------------------- headline regime vs the reference
HEADLINE = sorted(p.stem for p in GOLDEN.glob("headline_*.json"))


@pytest.mark.parametrize("name", HEADLINE)
def test_headline_regime_matches_reference(gpu, name):
    """The benchmark's parameters (alpha 0.0125, bf16, strict_model False,
    inner_tol 1e-2) on the unmodified reference at n_g = 32 .. 256: the fused
    reference-rounding solve reproduces every outer step -- inner counts,
    relres, status -- and the final iterate bit for bit."""
    c = json.loads((GOLDEN / f"{name}.json").read_text())
    rep = g.gadi_solve(g.build_cd_3d(c["n_g"]), cfg=g.GadiConfig(**c["cfg"]), rounding="reference")
    assert rep.status == c["status"]
    assert rep.iterations == c["outer"]
    assert [h.inner_h_iterations for h in rep.history] == c["inner_h"]
    assert [h.inner_s_iterations for h in rep.history] == c["inner_s"]
    np.testing.assert_allclose(rep.relative_residuals, c["relres"], rtol=1e-9, atol=0)
    if c["cfg"]["u_s"] != "fp64":  # fp64 dots are BLAS np.dot: order unpinned
        x = np.ascontiguousarray(rep.x, dtype=np.float64)
        assert hashlib.sha256(x.tobytes()).hexdigest() == c["x_sha256"]
    # berr = ||r|| / (||A||_2 ||x|| + ||b||): above HOST_START_MAX unknowns the
    # power iteration starts from the device generator instead of the
    # reference's numpy vector, so ||A||_2 agrees to the power-iteration
    # tolerance (1e-6 relative change per step), not to rounding
    big = c["n_g"] ** 3 > g.analysis.HOST_START_MAX
    np.testing.assert_allclose([h.backward_error for h in rep.history], c["berr"], rtol=1e-3 if big else 1e-9,
                               atol=0)
    assert rep.norm_A == pytest.approx(c["norm_A"], rel=1e-3 if big else 1e-10)


@pytest.mark.parametrize("name", HEADLINE)
def test_headline_regime_storage_model(gpu, name):
    """The storage model (fp32 arithmetic, rounded once per stored vector) at
    the same parameters: the north-star bar -- status, outer count within
    +-1, backward error within 2x -- where the run ends before outer_maxit;
    relres within 2x step by step over the first ten steps otherwise."""
    c = json.loads((GOLDEN / f"{name}.json").read_text())
    rep = g.gadi_solve(g.build_cd_3d(c["n_g"]), cfg=g.GadiConfig(**c["cfg"]), rounding="storage")
    assert rep.status == c["status"]
    if c["status"] == "Converged":
        assert abs(rep.iterations - c["outer"]) <= 1
        b, br = rep.history[-1].backward_error, c["berr"][-1]
        assert 0.5 * br <= b <= 2.0 * br
    k = min(10, len(c["relres"]), rep.iterations)
    rr = np.array(rep.relative_residuals[:k])
    ref = np.array(c["relres"][:k])
    assert np.all(rr <= 2 * ref) and np.all(ref <= 2 * rr), (rr, ref)
