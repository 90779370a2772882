"""Generate the golden fixtures from the UNMODIFIED reference package.

Run in the build container (the reference is not present on GPU boxes):

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py [--quick]

Writes tests/golden/kernels.npz (bitwise kernel outputs: residuals, strict
spmv on the u_s splitting copies, b = A 1, ||A||_2) and
tests/golden/solves.json (gadi_solve / cg_spd / cg_normal_skew outcomes:
status, outer and inner counts, relres / berr / ferr / mu histories).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import gadimp  # noqa: E402
from gadimp import (GadiConfig, build_cd_3d, build_cdr_2d, build_complex_rd, cg_normal_skew,  # noqa: E402
                    cg_spd, gadi_solve, make_hss_splitting, matrix_norm_2, quantize, residual, spmv)

HERE = Path(__file__).resolve().parent


def build(family, n_g, **kw):
    return {"cdr2d": build_cdr_2d, "cd3d": build_cd_3d, "crd": build_complex_rd}[family](n_g, **kw)


KERNEL_CASES = [
    ("cdr2d", 37, {}), ("cdr2d", 20, {"r": 0.3}), ("cdr2d", 32, {}), ("cd3d", 19, {}), ("cd3d", 16, {}),
    ("crd", 12, {}), ("crd", 16, {"seed": 3, "laplacian_scaling": "nu"}),
]


def kernels(out):
    rng = np.random.default_rng(2024)
    arrays = {}
    meta = []
    for fam, n_g, kw in KERNEL_CASES:
        p = build(fam, n_g, **kw)
        tag = f"{fam}_{n_g}" + ("_" + "_".join(f"{k}{v}" for k, v in kw.items()) if kw else "")
        n = p.n
        x = rng.standard_normal(n)
        b = rng.standard_normal(n)
        arrays[f"{tag}/x"] = x
        arrays[f"{tag}/bvec"] = b
        arrays[f"{tag}/b_ones"] = p.b
        arrays[f"{tag}/res_fp64"] = residual(p.A, x, b, "fp64")
        arrays[f"{tag}/Ax_fp64"] = spmv(p.A, x, "fp64")
        if fam != "crd":
            xq32 = quantize(x, "fp32")
            arrays[f"{tag}/xq32"] = xq32
            arrays[f"{tag}/res_fp32"] = residual(p.A.quantized("fp32"), xq32, quantize(b, "fp32"), "fp32")
            arrays[f"{tag}/res_fp64x2"] = residual(p.A, x, b, "fp64x2")
        t0 = time.perf_counter()
        arrays[f"{tag}/norm2"] = np.array([matrix_norm_2(p.A)])
        tn = time.perf_counter() - t0
        for us in ("bf16", "fp16", "fp32"):
            sp = make_hss_splitting(p.A, 0.75, us)
            xq = quantize(x, us)
            arrays[f"{tag}/{us}/xq"] = xq
            arrays[f"{tag}/{us}/H"] = spmv(sp.H_low, xq, us)
            arrays[f"{tag}/{us}/S"] = spmv(sp.S_low, xq, us)
            arrays[f"{tag}/{us}/ST"] = spmv(sp.S_low_T, xq, us)
        sp = make_hss_splitting(p.A, 0.75, "fp64")
        arrays[f"{tag}/fp64/H"] = spmv(sp.H_low, x, "fp64")
        arrays[f"{tag}/fp64/S"] = spmv(sp.S_low, x, "fp64")
        arrays[f"{tag}/fp64/ST"] = spmv(sp.S_low_T, x, "fp64")
        meta.append({"tag": tag, "family": fam, "n_g": n_g, "kw": kw, "alpha": 0.75, "norm_s": tn})
    np.savez_compressed(out / "kernels.npz", **arrays)
    (out / "kernels_meta.json").write_text(json.dumps(meta, indent=1))


def run_case(case):
    fam, n_g, kw = case["family"], case["n_g"], case.get("kw", {})
    p = build(fam, n_g, **kw)
    cfg = GadiConfig(**case["cfg"])
    t0 = time.perf_counter()
    rep = gadi_solve(p, cfg=cfg)
    wall = time.perf_counter() - t0
    h = rep.history
    return {
        **case,
        "status": rep.status, "outer": rep.iterations, "inner": rep.total_inner_iterations,
        "inner_h": [r.inner_h_iterations for r in h], "inner_s": [r.inner_s_iterations for r in h],
        "relres": [r.relative_residual for r in h], "berr": [r.backward_error for r in h],
        "ferr": [r.forward_error for r in h], "mu": [r.mu for r in h],
        "residual_norm": [r.residual_norm for r in h],
        "norm_A": rep.norm_A, "wall_s": wall,
        "x_head": rep.x[:8].tolist(),
    }


def solve_cases(quick):
    cases = []
    for n_g in (16, 32, 64):
        for us in ("bf16", "fp32", "fp64"):
            cases.append({"name": f"c3_cdr2d{n_g}_{us}", "family": "cdr2d", "n_g": n_g,
                          "cfg": {"alpha": 1.0, "u_s": us, "outer_tol": 1e-10, "outer_maxit": 800}})
    for n_g in (8, 16):
        for us in ("bf16", "fp32", "fp64"):
            cases.append({"name": f"c3_cd3d{n_g}_{us}", "family": "cd3d", "n_g": n_g,
                          "cfg": {"alpha": 0.5, "u_s": us, "outer_tol": 1e-6, "outer_maxit": 800}})
    for n_g in (16, 32):
        for us in ("bf16", "fp32", "fp64"):
            cases.append({"name": f"c3_crd{n_g}_{us}", "family": "crd", "n_g": n_g,
                          "cfg": {"alpha": 10.0, "u_s": us, "outer_tol": 1e-6, "outer_maxit": 800}})
    cases += [
        {"name": "gadi_cdr2d6", "family": "cdr2d", "n_g": 6, "cfg": {"alpha": 1.0, "outer_tol": 1e-10}},
        {"name": "stagnation_cdr2d8", "family": "cdr2d", "n_g": 8,
         "cfg": {"alpha": 1.0, "u": "fp32", "u_r": "fp32", "u_s": "bf16", "outer_tol": 1e-14, "outer_maxit": 500}},
        {"name": "three_precision_cdr2d8", "family": "cdr2d", "n_g": 8,
         "cfg": {"alpha": 1.0, "u": "fp32", "u_r": "fp64x2", "u_s": "bf16", "outer_tol": 1e-6, "outer_maxit": 300}},
        {"name": "omega05_cdr2d16_fp32", "family": "cdr2d", "n_g": 16,
         "cfg": {"alpha": 1.0, "omega": 0.5, "u_s": "fp32", "outer_tol": 1e-10, "outer_maxit": 800}},
        {"name": "r03_cdr2d24_bf16", "family": "cdr2d", "n_g": 24, "kw": {"r": 0.3},
         "cfg": {"alpha": 0.8, "u_s": "bf16", "outer_tol": 1e-10, "outer_maxit": 800}},
        {"name": "floor_cdr2d64_bf16", "family": "cdr2d", "n_g": 64,
         "cfg": {"alpha": 1.0, "u_s": "bf16", "outer_tol": 0.0, "outer_maxit": 400}},
        {"name": "floor_cd3d16_fp32", "family": "cd3d", "n_g": 16,
         "cfg": {"alpha": 0.5, "u_s": "fp32", "outer_tol": 0.0, "outer_maxit": 400}},
        {"name": "nonstrict_cdr2d32_bf16", "family": "cdr2d", "n_g": 32,
         "cfg": {"alpha": 1.0, "u_s": "bf16", "outer_tol": 1e-10, "strict_model": False}},
        {"name": "innertol1e2_cd3d12_bf16", "family": "cd3d", "n_g": 12,
         "cfg": {"alpha": 0.3, "u_s": "bf16", "outer_tol": 1e-8, "inner_tol": 1e-2, "outer_maxit": 800}},
        {"name": "cfg1_cdr2d256_fp64", "family": "cdr2d", "n_g": 256,
         "cfg": {"alpha": 1.0, "u_s": "fp64", "outer_tol": 1e-10}},
    ]
    if not quick:
        cases.append({"name": "cfg1_cdr2d256_fp32", "family": "cdr2d", "n_g": 256,
                      "cfg": {"alpha": 1.0, "u_s": "fp32", "outer_tol": 1e-10}})
    return cases


def inner_cases():
    out = []
    rng = np.random.default_rng(77)
    for fam, n_g, alpha in (("cdr2d", 32, 1.0), ("cd3d", 12, 0.5), ("crd", 16, 10.0)):
        p = build(fam, n_g)
        for us in ("bf16", "fp32", "fp64"):
            sp = make_hss_splitting(p.A, alpha, us)
            r = rng.standard_normal(p.n)
            rhs = quantize(r / np.max(np.abs(r)), us)
            z, st_h = cg_spd(sp.H_low, rhs, 1e-4, None, us)
            y, st_s = cg_normal_skew(sp.S_low, rhs, 1e-4, None, us, True, sp.S_low_T)
            out.append({"family": fam, "n_g": n_g, "alpha": alpha, "u_s": us, "rhs": rhs.tolist(),
                        "h_it": st_h.iterations, "h_conv": st_h.converged, "h_true": st_h.true_relative_residual,
                        "h_x": z.tolist(), "s_it": st_s.iterations, "s_conv": st_s.converged,
                        "s_true": st_s.true_relative_residual, "s_x": y.tolist()})
    return out


def csr_cases(out):
    """General sparse systems (the reference's own graded / mixed families,
    TST/conftest.py:15-53, built by importing that conftest) for the CSR
    engine: matrices, kernel outputs and solve histories (c4, c5 settings,
    TST/test_acceptance.py:121-158)."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import graded_problem, mixed_problem  # noqa: E402

    arrays, res = {}, []
    problems = {"graded1e2": graded_problem(50, 1e2), "graded1e4": graded_problem(50, 1e4),
                "graded1e6": graded_problem(50, 1e6), "mixed1e6": mixed_problem(50, 1e6)}
    rng = np.random.default_rng(99)
    for tag, p in problems.items():
        a = p.A
        arrays[f"{tag}/rp"], arrays[f"{tag}/ci"], arrays[f"{tag}/v"] = a.row_offsets, a.col_indices, a.values
        arrays[f"{tag}/b"], arrays[f"{tag}/xs"] = p.b, p.exact_solution
        x = rng.standard_normal(a.nrows)
        b = rng.standard_normal(a.nrows)
        arrays[f"{tag}/x"], arrays[f"{tag}/bvec"] = x, b
        arrays[f"{tag}/res_fp64"] = residual(a, x, b, "fp64")
        xq32 = quantize(x, "fp32")
        arrays[f"{tag}/xq32"] = xq32
        arrays[f"{tag}/res_fp32"] = residual(a.quantized("fp32"), xq32, quantize(b, "fp32"), "fp32")
        arrays[f"{tag}/res_fp64x2"] = residual(a, x, b, "fp64x2")
        arrays[f"{tag}/Ax_fp64"] = spmv(a, x, "fp64")
        arrays[f"{tag}/norm2"] = np.array([matrix_norm_2(a)])
        for us in ("bf16", "fp32"):
            sp = make_hss_splitting(a, 1.0, us)
            xq = quantize(x, us)
            arrays[f"{tag}/{us}/xq"] = xq
            for nm, m in (("H", sp.H_low), ("S", sp.S_low), ("ST", sp.S_low_T)):
                arrays[f"{tag}/{us}/{nm}"] = spmv(m, xq, us)
    runs = []
    for tag in ("graded1e2", "graded1e4", "graded1e6"):
        for us in ("bf16", "fp32"):
            runs.append((f"c4_{tag}_{us}", tag, {"alpha": 1.0, "u_s": us, "outer_tol": 0.0, "outer_maxit": 600,
                                                 "inner_tol": 1e-4}))
    for ur in ("fp32", "fp64x2"):
        runs.append((f"c5_mixed1e6_{ur}", "mixed1e6", {"alpha": 1.0, "u": "fp32", "u_r": ur, "u_s": "fp32",
                                                       "outer_tol": 0.0, "outer_maxit": 600, "inner_tol": 1e-4}))
    runs.append(("conv_graded1e4_bf16", "graded1e4", {"alpha": 1.0, "u_s": "bf16", "outer_tol": 1e-10}))
    runs.append(("conv_mixed1e6_fp64", "mixed1e6", {"alpha": 1.0, "u_s": "fp64", "outer_tol": 1e-10}))
    for name, tag, cfg in runs:
        t0 = time.perf_counter()
        rep = gadi_solve(problems[tag], cfg=GadiConfig(**cfg))
        h = rep.history
        res.append({"name": name, "problem": tag, "cfg": cfg, "status": rep.status, "outer": rep.iterations,
                    "inner_h": [r.inner_h_iterations for r in h], "inner_s": [r.inner_s_iterations for r in h],
                    "relres": [r.relative_residual for r in h], "berr": [r.backward_error for r in h],
                    "ferr": [r.forward_error for r in h], "norm_A": rep.norm_A, "x_head": rep.x[:8].tolist(),
                    "wall_s": time.perf_counter() - t0})
        print(f"{name}: {rep.status} outer={rep.iterations} berr={h[-1].backward_error:.3e}", flush=True)
    np.savez_compressed(out / "csr.npz", **arrays)
    (out / "csr.json").write_text(json.dumps(res))


def build_crd3d_ref(n_g, s=1.0e4, seed=0, laplacian_scaling="nu_over_h2"):
    """The 3-D extension of REF/problems.py:96-120 (BASELINE config 5, SURVEY
    D1: the reference has no 3-D generator) assembled with the reference's own
    sparse operations: the 2-D recipe with the triple Kronecker sum."""
    import scipy.sparse as sp
    from gadimp.problems import Problem
    from gadimp.sparsemat import SparseMatrix, identity, kron, tridiag

    nu = 1.0e-5 * (64.0 / n_g) ** 2
    h = 1.0 / (n_g + 1)
    scale = nu / h**2 if laplacian_scaling == "nu_over_h2" else nu
    t = tridiag(n_g, -1.0, 2.0, -1.0)
    eye = identity(n_g)
    lap = scale * (kron(kron(t, eye), eye).to_scipy() + kron(kron(eye, t), eye).to_scipy()
                   + kron(kron(eye, eye), t).to_scipy())
    xi = np.random.Generator(np.random.Philox(key=seed)).uniform(size=n_g**3)
    v = sp.diags(s * xi)
    a = SparseMatrix.from_scipy(sp.bmat([[lap, -v], [v, lap]], format="csr"))
    ones = np.ones(a.nrows)
    return Problem(A=a, b=a.to_scipy() @ ones, exact_solution=ones, label="crd3d",
                   params={"n_g": n_g, "s": s, "seed": seed, "nu": nu, "laplacian_scaling": laplacian_scaling,
                           "ndim": 3})


def crd3d_cases(out):
    arrays, res = {}, []
    rng = np.random.default_rng(31)
    for n_g in (6, 8):
        p = build_crd3d_ref(n_g)
        a, tag = p.A, f"crd3d_{n_g}"
        arrays[f"{tag}/rp"], arrays[f"{tag}/ci"], arrays[f"{tag}/v"] = a.row_offsets, a.col_indices, a.values
        arrays[f"{tag}/b_ones"] = p.b
        x, b = rng.standard_normal(a.nrows), rng.standard_normal(a.nrows)
        arrays[f"{tag}/x"], arrays[f"{tag}/bvec"] = x, b
        arrays[f"{tag}/res_fp64"] = residual(a, x, b, "fp64")
        arrays[f"{tag}/norm2"] = np.array([matrix_norm_2(a)])
        for us in ("bf16", "fp32"):
            sp_ = make_hss_splitting(a, 10.0, us)
            xq = quantize(x, us)
            arrays[f"{tag}/{us}/xq"] = xq
            for nm, m in (("H", sp_.H_low), ("S", sp_.S_low), ("ST", sp_.S_low_T)):
                arrays[f"{tag}/{us}/{nm}"] = spmv(m, xq, us)
    for n_g in (6, 8):
        p = build_crd3d_ref(n_g)
        for us in ("bf16", "fp32", "fp64"):
            cfg = {"alpha": 10.0, "u_s": us, "outer_tol": 1e-6, "outer_maxit": 800}
            rep = gadi_solve(p, cfg=GadiConfig(**cfg))
            h = rep.history
            res.append({"name": f"crd3d{n_g}_{us}", "n_g": n_g, "cfg": cfg, "status": rep.status,
                        "outer": rep.iterations, "inner_h": [r.inner_h_iterations for r in h],
                        "inner_s": [r.inner_s_iterations for r in h], "relres": [r.relative_residual for r in h],
                        "berr": [r.backward_error for r in h], "norm_A": rep.norm_A,
                        "x_head": rep.x[:8].tolist()})
            print(f"crd3d{n_g}_{us}: {rep.status} outer={rep.iterations} berr={h[-1].backward_error:.3e}", flush=True)
    np.savez_compressed(out / "crd3d.npz", **arrays)
    (out / "crd3d.json").write_text(json.dumps(res))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", choices=["kernels", "solves", "inner", "csr", "crd3d", "fp16"], default=None)
    a = ap.parse_args()
    HERE.mkdir(parents=True, exist_ok=True)
    if a.only in (None, "kernels"):
        kernels(HERE)
        print("kernels done", flush=True)
    if a.only in (None, "inner"):
        (HERE / "inner.json").write_text(json.dumps(inner_cases()))
        print("inner done", flush=True)
    if a.only in (None, "fp16"):
        cases = [{"name": "fp16_cdr2d32", "family": "cdr2d", "n_g": 32,
                  "cfg": {"alpha": 1.0, "u_s": "fp16", "outer_tol": 1e-10, "outer_maxit": 800}},
                 {"name": "fp16_cd3d16", "family": "cd3d", "n_g": 16,
                  "cfg": {"alpha": 0.5, "u_s": "fp16", "outer_tol": 1e-6, "outer_maxit": 800}},
                 {"name": "fp16_crd16", "family": "crd", "n_g": 16,
                  "cfg": {"alpha": 10.0, "u_s": "fp16", "outer_tol": 1e-6, "outer_maxit": 800}}]
        res = [run_case(c) for c in cases]
        for r in res:
            print(f"{r['name']}: {r['status']} outer={r['outer']}", flush=True)
        (HERE / "solves_fp16.json").write_text(json.dumps(res))
    if a.only in (None, "crd3d"):
        crd3d_cases(HERE)
        print("crd3d done", flush=True)
    if a.only in (None, "csr"):
        csr_cases(HERE)
        print("csr done", flush=True)
    if a.only in (None, "solves"):
        res = []
        for c in solve_cases(a.quick):
            r = run_case(c)
            print(f"{c['name']}: {r['status']} outer={r['outer']} inner={r['inner']} "
                  f"relres={r['relres'][-1]:.3e} berr={r['berr'][-1]:.3e} {r['wall_s']:.1f}s", flush=True)
            res.append(r)
        (HERE / "solves.json").write_text(json.dumps(res))
    print("gadimp", gadimp.__version__)


if __name__ == "__main__":
    main()
