"""GPU kernel parity against the reference's golden outputs (bitwise where
the reference arithmetic is reproducible: fp64 ordered stencils, the strict
u_s spmv, the fp32 and fp64x2 residuals, b = A 1)."""

import numpy as np
import pytest

import paper_2512_21164_b200 as g
from paper_2512_21164_b200 import device
from paper_2512_21164_b200.stencil import spec_cd_3d, spec_cdr_2d, spec_complex_rd

pytestmark = pytest.mark.gpu


def _spec(meta):
    fam, n_g, kw = meta["family"], meta["n_g"], meta["kw"]
    if fam == "cdr2d":
        return spec_cdr_2d(n_g, **kw)
    if fam == "cd3d":
        return spec_cd_3d(n_g)
    return spec_complex_rd(n_g, **kw)


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def _assert_bitwise(got, want, what):
    got, want = np.asarray(got), np.asarray(want)
    bad = np.nonzero(_bits(got) != _bits(want))[0]
    # +0 / -0 differences are representation-only; everything else must match
    real_bad = [i for i in bad if not (got[i] == 0.0 and want[i] == 0.0)]
    assert not real_bad, f"{what}: {len(real_bad)} mismatches, first {real_bad[:5]} " \
                         f"got {got[real_bad[:3]]} want {want[real_bad[:3]]}"


def test_rhs_ones_bitwise(gpu, golden_kernels, golden_kernel_meta):
    for m in golden_kernel_meta:
        spec = _spec(m)
        _assert_bitwise(device.rhs_ones(spec), golden_kernels[f"{m['tag']}/b_ones"], m["tag"])


def test_residual_fp64_bitwise(gpu, golden_kernels, golden_kernel_meta):
    for m in golden_kernel_meta:
        p = g.StencilProblem(_spec(m))
        t = m["tag"]
        r = g.residual(p.A, golden_kernels[f"{t}/x"], golden_kernels[f"{t}/bvec"], "fp64")
        _assert_bitwise(r, golden_kernels[f"{t}/res_fp64"], t)


def test_spmv_A_fp64_bitwise(gpu, golden_kernels, golden_kernel_meta):
    for m in golden_kernel_meta:
        p = g.StencilProblem(_spec(m))
        t = m["tag"]
        _assert_bitwise(g.spmv(p.A, golden_kernels[f"{t}/x"], "fp64"), golden_kernels[f"{t}/Ax_fp64"], t)


def test_residual_fp32_and_compensated_bitwise(gpu, golden_kernels, golden_kernel_meta):
    for m in golden_kernel_meta:
        if m["family"] == "crd":
            continue
        p = g.StencilProblem(_spec(m))
        t = m["tag"]
        xq = golden_kernels[f"{t}/xq32"]
        r32 = g.residual(p.A, xq, golden_kernels[f"{t}/bvec"], "fp32")
        _assert_bitwise(r32, golden_kernels[f"{t}/res_fp32"], t + " fp32")
        r2 = g.residual(p.A, golden_kernels[f"{t}/x"], golden_kernels[f"{t}/bvec"], "fp64x2")
        _assert_bitwise(r2, golden_kernels[f"{t}/res_fp64x2"], t + " fp64x2")


@pytest.mark.parametrize("us", ["bf16", "fp16", "fp32", "fp64"])
def test_strict_spmv_splitting_bitwise(gpu, golden_kernels, golden_kernel_meta, us):
    for m in golden_kernel_meta:
        p = g.StencilProblem(_spec(m))
        t = m["tag"]
        sp = g.make_hss_splitting(p.A, m["alpha"], us)
        x = golden_kernels[f"{t}/{us}/xq"] if us != "fp64" else golden_kernels[f"{t}/x"]
        for name, op in (("H", sp.H_low), ("S", sp.S_low), ("ST", sp.S_low_T)):
            _assert_bitwise(g.spmv(op, x, us), golden_kernels[f"{t}/{us}/{name}"], f"{t} {us} {name}")


def test_norm2_matches_reference(gpu, golden_kernels, golden_kernel_meta):
    for m in golden_kernel_meta:
        p = g.StencilProblem(_spec(m))
        want = float(golden_kernels[f"{m['tag']}/norm2"][0])
        got = g.matrix_norm_2(p.A)
        assert got == pytest.approx(want, rel=1e-12), m["tag"]


@pytest.mark.parametrize("fam,ng", [("cdr2d", 37), ("cdr2d", 64), ("cdr2d", 100), ("cd3d", 19), ("cd3d", 20), ("cd3d", 34)])
def test_fused_power_iteration_equals_two_pass(gpu, fam, ng, monkeypatch):
    """The one-sweep A^T A step (csrc/norm_fused.cuh) computes every t and w
    value with the two-pass operations; only the grid (hence the summation
    order of ||w||^2) differs: same iteration count, sigma to rounding."""
    spec = spec_cdr_2d(ng) if fam == "cdr2d" else spec_cd_3d(ng)
    v0 = g.analysis.power_start_vector(spec.n)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("GADI_NORM_2PASS", mode)
        with device.open_context(device.make_desc(spec, 1.0, "fp64")) as ctx:
            out[mode] = ctx.norm2(v0)
    assert out["0"][1] == out["1"][1], out
    assert out["0"][0] == pytest.approx(out["1"][0], rel=1e-13), out


@pytest.mark.parametrize("ng,us", [(16, "bf16"), (40, "bf16"), (64, "bf16"), (48, "fp32"), (64, "fp16")])
def test_tensor_map_producer_bitwise(gpu, ng, us, monkeypatch):
    """The TMA tensor-map producer (csrc/tmap.cuh: HcgA / CgnrP1 haloed
    inputs as boxes, grid edges zero-filled by the hardware) feeds the
    consumers exactly the data the row-copy producer does: H- and S-solves
    bitwise equal with GADI_TMAP=1 and GADI_TMAP=0, iteration counts equal."""
    spec = spec_cd_3d(ng)
    rng = np.random.default_rng(ng)
    rhs = g.quantize(rng.uniform(-1.0, 1.0, spec.n), us)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("GADI_TMAP", mode)
        with device.open_context(device.make_desc(spec, 0.05, us)) as ctx:
            zh, sh = ctx.h_solve(rhs, 1e-6, 400)
            zs, ss = ctx.s_solve(rhs, 1e-6, 400)
        out[mode] = (zh, sh.iterations, zs, ss.iterations)
    assert out["0"][1] == out["1"][1] and out["0"][3] == out["1"][3]
    assert np.array_equal(out["0"][0], out["1"][0])
    assert np.array_equal(out["0"][2], out["1"][2])
