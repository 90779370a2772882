"""3-D complex reaction-diffusion (BASELINE config 5; the
reference has only the 2-D generator).  The 3-D operator is the reference's
2-D recipe (REF/problems.py:96-120) with the triple Kronecker sum, assembled
from the reference's own sparse operations by tests/golden/make_golden.py
--only crd3d; the reference's gadi_solve was run on it for the fixtures.

CPU: the stencil spec, its CSR view and the oracle equal that assembly
bitwise.  GPU: kernels bitwise, solves within the parity bar, and
rounding="reference" exactly."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2512_21164_b200 as g
from oracle import gadi_oracle as O

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def fx():
    return np.load(GOLDEN / "crd3d.npz"), {c["name"]: c for c in json.loads((GOLDEN / "crd3d.json").read_text())}


def _bits(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return np.array_equal(a.view(np.uint64), b.view(np.uint64)) or np.array_equal(a, b)


@pytest.mark.parametrize("ng", [6, 8])
def test_crd3d_operator_equals_reference_assembly(fx, ng):
    arr, _ = fx
    t = f"crd3d_{ng}"
    a = g.build_complex_rd_3d(ng).A
    assert np.array_equal(a.row_offsets, arr[f"{t}/rp"])
    assert np.array_equal(a.col_indices, arr[f"{t}/ci"])
    assert _bits(a.values, arr[f"{t}/v"])


@pytest.mark.parametrize("ng", [6, 8])
def test_crd3d_oracle_kernels(fx, ng):
    arr, _ = fx
    t = f"crd3d_{ng}"
    op = O.build("crd3d", ng)
    assert _bits(O.rhs_ones(op), arr[f"{t}/b_ones"])
    assert _bits(O.stencil_residual(op, arr[f"{t}/x"], arr[f"{t}/bvec"]), arr[f"{t}/res_fp64"])
    for us in ("bf16", "fp32"):
        H, S, ST = O.splitting(op, 10.0, us)
        xq = arr[f"{t}/{us}/xq"]
        for nm, m in (("H", H), ("S", S), ("ST", ST)):
            assert _bits(O.stencil_apply(m, xq, us), arr[f"{t}/{us}/{nm}"]), (us, nm)


@pytest.mark.gpu
@pytest.mark.parametrize("ng", [6, 8])
def test_crd3d_gpu_kernels_bitwise(gpu, fx, ng):
    from paper_2512_21164_b200 import device

    arr, _ = fx
    t = f"crd3d_{ng}"
    p = g.build_complex_rd_3d(ng)
    assert _bits(device.rhs_ones(p.A.spec), arr[f"{t}/b_ones"])
    assert _bits(g.residual(p.A, arr[f"{t}/x"], arr[f"{t}/bvec"], "fp64"), arr[f"{t}/res_fp64"])
    assert g.matrix_norm_2(p.A) == pytest.approx(float(arr[f"{t}/norm2"][0]), rel=1e-12)
    for us in ("bf16", "fp32"):
        sp = g.make_hss_splitting(p.A, 10.0, us)
        xq = arr[f"{t}/{us}/xq"]
        for nm, m in (("H", sp.H_low), ("S", sp.S_low), ("ST", sp.S_low_T)):
            assert _bits(g.spmv(m, xq, us), arr[f"{t}/{us}/{nm}"]), (us, nm)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["crd3d6_bf16", "crd3d6_fp32", "crd3d6_fp64", "crd3d8_bf16", "crd3d8_fp32",
                                  "crd3d8_fp64"])
def test_crd3d_solves(gpu, fx, name):
    _, runs = fx
    c = runs[name]
    cfg = g.GadiConfig(**c["cfg"])
    rep = g.gadi_solve(g.build_complex_rd_3d(c["n_g"]), cfg=cfg)
    assert rep.status == c["status"]
    assert 0.5 * c["berr"][-1] <= rep.history[-1].backward_error <= 2.0 * c["berr"][-1]
    # n_g = 6: every CGNR solve stops at maxit (104 iterations, kappa(S) ~ 1e3)
    # without converging, so the unpinned BLAS dot order of the reference (fp64)
    # and the storage model (bf16) move the outer count by up to 2; the
    # rounding="reference" run below is still exact.  n_g = 8 takes the bar.
    tol = 2 if c["n_g"] == 6 else (0 if c["cfg"]["u_s"] == "fp64" else 1)
    assert abs(rep.iterations - c["outer"]) <= tol, (rep.iterations, c["outer"])
    if c["cfg"]["u_s"] != "fp64":
        ex = g.gadi_solve(g.build_complex_rd_3d(c["n_g"]), cfg=cfg, rounding="reference")
        assert ex.iterations == c["outer"]
        assert [h.inner_h_iterations for h in ex.history] == c["inner_h"]
        assert [h.inner_s_iterations for h in ex.history] == c["inner_s"]
        assert np.array_equal(ex.x[:8], np.array(c["x_head"]))
