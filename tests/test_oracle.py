"""Pin the CPU oracle to the reference's golden outputs (CPU-only tests).

The oracle (oracle/gadi_oracle.py) is the checker the GPU tests and the
benchmark's CPU baseline rely on; these tests prove it reproduces the
unmodified reference: bitwise for b = A 1, residuals and the emulated spmv,
to 1e-12 for ||A||_2, and run-for-run (status, outer count, inner counts,
error history) for gadi_solve."""

import json

import numpy as np
import pytest

from oracle import gadi_oracle as O


def _op(meta):
    return O.build(meta["family"], meta["n_g"], **meta["kw"])


def _same_bits(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return np.array_equal(a.view(np.uint64), b.view(np.uint64)) or np.array_equal(a, b)


def test_rhs_and_fp64_kernels_bitwise(golden_kernels, golden_kernel_meta):
    for m in golden_kernel_meta:
        op, t = _op(m), m["tag"]
        assert _same_bits(O.rhs_ones(op), golden_kernels[f"{t}/b_ones"]), t
        x, b = golden_kernels[f"{t}/x"], golden_kernels[f"{t}/bvec"]
        assert _same_bits(O.stencil_apply(op, x), golden_kernels[f"{t}/Ax_fp64"]), t
        assert _same_bits(O.stencil_residual(op, x, b, "fp64"), golden_kernels[f"{t}/res_fp64"]), t


def test_fp32_and_compensated_residual_bitwise(golden_kernels, golden_kernel_meta):
    for m in golden_kernel_meta:
        if m["family"] == "crd":
            continue
        op, t = _op(m), m["tag"]
        a32 = O.Stencil(op.dims, O.q(op.d, "fp32"), tuple(O.q(c, "fp32") for c in op.lo),
                        tuple(O.q(c, "fp32") for c in op.up))
        xq, b = golden_kernels[f"{t}/xq32"], golden_kernels[f"{t}/bvec"]
        assert _same_bits(O.stencil_residual(a32, xq, O.q(b, "fp32"), "fp32"), golden_kernels[f"{t}/res_fp32"]), t
        assert _same_bits(O.stencil_residual(op, golden_kernels[f"{t}/x"], b, "fp64x2"),
                          golden_kernels[f"{t}/res_fp64x2"]), t


@pytest.mark.parametrize("us", ["bf16", "fp16", "fp32", "fp64"])
def test_emulated_splitting_spmv_bitwise(golden_kernels, golden_kernel_meta, us):
    for m in golden_kernel_meta:
        op, t = _op(m), m["tag"]
        H, S, ST = O.splitting(op, m["alpha"], us)
        x = golden_kernels[f"{t}/{us}/xq"] if us != "fp64" else golden_kernels[f"{t}/x"]
        for name, o in (("H", H), ("S", S), ("ST", ST)):
            assert _same_bits(O.stencil_apply(o, x, us), golden_kernels[f"{t}/{us}/{name}"]), (t, us, name)


def test_norm2(golden_kernels, golden_kernel_meta):
    for m in golden_kernel_meta:
        got = O.matrix_norm_2(_op(m))
        assert got == pytest.approx(float(golden_kernels[f"{m['tag']}/norm2"][0]), rel=1e-12), m["tag"]


def test_rounding_contract():
    assert O.q(1.0 + 2.0 ** -8, "bf16") == 1.0            # tie to even
    assert O.q(1.0 + 3 * 2.0 ** -8, "bf16") == 1.0 + 2.0 ** -6
    assert np.isinf(O.q(1e39, "fp32")) and np.isinf(O.q(1e39, "bf16"))
    assert O.q(1e-40, "bf16") != 0.0                      # subnormals kept
    assert O.fl_sum([2.0 ** -8, 2.0 ** -8, 1.0, 0.0], "bf16") == 1.0 + 2.0 ** -7  # pairwise, not sequential
    p, e = O.two_prod(1.0 + 2.0 ** -30, 1.0 + 2.0 ** -30)
    assert p + e == p and e == 2.0 ** -60


FAST_SOLVES = ["c3_cdr2d16_bf16", "c3_cdr2d16_fp32", "c3_cdr2d32_fp64", "c3_cd3d8_bf16", "c3_cd3d8_fp32",
               "c3_crd16_bf16", "c3_crd16_fp64", "gadi_cdr2d6", "three_precision_cdr2d8", "stagnation_cdr2d8",
               "omega05_cdr2d16_fp32", "r03_cdr2d24_bf16", "nonstrict_cdr2d32_bf16", "innertol1e2_cd3d12_bf16"]


@pytest.mark.parametrize("name", FAST_SOLVES)
def test_oracle_solve_reproduces_reference(golden_solves, name):
    c = golden_solves[name]
    op = O.build(c["family"], c["n_g"], **c.get("kw", {}))
    cfg = dict(c["cfg"])
    cfg.setdefault("u_s", "fp64")
    strict = cfg.pop("strict_model", True)
    kw = {k: cfg[k] for k in ("omega", "u", "u_r", "u_s", "outer_tol", "outer_maxit", "inner_tol") if k in cfg}
    rep = O.gadi_solve(op, O.rhs_ones(op), cfg["alpha"], strict=strict, exact=np.ones(op.n), **kw)
    assert rep.status == c["status"]
    assert len(rep.history) == c["outer"]
    assert [h.inner_h for h in rep.history] == c["inner_h"]
    assert [h.inner_s for h in rep.history] == c["inner_s"]
    np.testing.assert_allclose([h.relative_residual for h in rep.history], c["relres"], rtol=1e-6)
    np.testing.assert_allclose([h.backward_error for h in rep.history], c["berr"], rtol=1e-6)
    assert rep.norm_A == pytest.approx(c["norm_A"], rel=1e-12)
