"""Inner Krylov solvers (drop-in for gadimp/inner.py:1-143), on the GPU.

``cg_spd`` (classical CG on H = alpha I + M) and ``cg_normal_skew`` (CGNR on
S = alpha I + N) run the same fused, device-driven kernels the outer loop
uses (csrc/passes.cuh: HcgA/HcgB, CgnrP1-3; csrc/pointwise.cuh for the crd
family).  Arithmetic follows the storage model: vectors stored in ``fmt``,
fp32 compute, fp64 accumulation of dot products; stopping quantities are
the reference's (sqrt(rs)/||rhs|| for CG, the fp64 ||r||/||rhs|| for CGNR).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .device import is_csr, make_csr_desc, make_desc, open_context
from .sparsemat import transpose
from .precision import resolve_format
from .stencil import StencilMatrix

__all__ = ["InnerSolveStats", "cg_spd", "cg_normal_skew", "default_maxit", "dot_format"]

_MAXIT_CAP = 10_000


def default_maxit(n: int) -> int:
    """min(10^4, ceil(5 sqrt(n))) (inner.py:26-27)."""
    return min(_MAXIT_CAP, max(1, math.ceil(5.0 * math.sqrt(n))))


# Inner-solver arithmetic (gadi_set_rounding, include/gadi_b200.h): the
# storage model, the reference's per-operation rounding inside the fused
# passes, or the same rounding one operation per launch (cross-check).
ROUNDING_MODES = {"storage": 0, "reference": 1, "reference_host": 2}


def rounding_mode(rounding: str) -> int:
    try:
        return ROUNDING_MODES[rounding]
    except KeyError:
        raise ValueError(f"rounding must be one of {sorted(ROUNDING_MODES)}, got {rounding!r}") from None


def dot_format(fmt, strict_model: bool):
    """Accumulation format of the reference's dot products (inner.py:39-44):
    u_s, or fp32 when ``strict_model`` is off and u_s is below fp32."""
    fmt = resolve_format(fmt)
    fp32 = resolve_format("fp32")
    if not strict_model and fmt.unit_roundoff > fp32.unit_roundoff:
        return fp32
    return fmt


@dataclass
class InnerSolveStats:
    iterations: int
    final_relative_residual: float
    converged: bool
    breakdown: bool
    true_relative_residual: float = float("nan")


def _ctx_for(op, fmt, which: str, op_t=None):
    if is_csr(op):
        # the operator sits in the H slot (CG) or the S / S^T slots (CGNR)
        st = op_t if op_t is not None else (transpose(op) if which == "S" else op)
        return open_context(make_csr_desc(op, op, op, st, fmt))
    if not isinstance(op, StencilMatrix):
        raise NotImplementedError(f"unsupported operator type {type(op).__name__}")
    spec = op.spec
    if spec.family == "crd":
        return open_context(make_desc(spec, op.alpha, fmt, coef_fmt=op.fmt))
    c = op.coefs()
    return open_context(make_desc(spec, 0.0, fmt, H=c, S=c))


def _true_relres(op, rhs, x, nrhs) -> float:
    if nrhs == 0.0:
        return 0.0
    if is_csr(op):  # fp64 true residual (inner.py:88, 142)
        with open_context(make_csr_desc(op, op, op, op, "fp64")) as ctx:
            y = ctx.spmv(0, x)
        return float(np.linalg.norm(rhs - y)) / nrhs
    spec = op.spec
    if spec.family == "crd":
        ctx = open_context(make_desc(spec, op.alpha, "fp64", coef_fmt=op.fmt))
        y = ctx.spmv({"H": 1, "S": 2, "ST": 3, "AmN": 3}[op.role], x, strict=True)
    else:
        c = op.coefs()
        ctx = open_context(make_desc(spec, 0.0, "fp64", H=c, S=c))
        y = ctx.spmv(1, x, strict=True)
    ctx.close()
    return float(np.linalg.norm(rhs - y)) / nrhs


def cg_spd(h, rhs: np.ndarray, tol: float, maxit: int | None = None, fmt="fp64",
           strict_model: bool = True, *, rounding: str = "reference"):
    """CG on H x = rhs, H SPD, x0 = 0.  ``rounding="reference"`` runs the
    reference's per-operation rounding emulation (bitwise iterates)."""
    fmt = resolve_format(fmt)
    rhs = np.asarray(rhs, dtype=np.float64)
    if maxit is None:
        maxit = default_maxit(rhs.size)
    with _ctx_for(h, fmt, "H") as ctx:
        ctx.set_rounding(rounding_mode(rounding), dot_format(fmt, strict_model).name)
        x, st = ctx.h_solve(rhs, tol, maxit)
    nrhs = float(np.linalg.norm(rhs))
    return x, InnerSolveStats(st.iterations, st.final_relative_residual, bool(st.converged),
                              bool(st.breakdown), _true_relres(h, rhs, x, nrhs))


def cg_normal_skew(s, rhs: np.ndarray, tol: float, maxit: int | None = None, fmt="fp64",
                   strict_model: bool = True, s_transpose=None, *, rounding: str = "reference"):
    """CGNR on S y = rhs (S^T S y = S^T rhs without forming S^T S), y0 = 0.
    ``s_transpose`` is implied by the stencil (S^T swaps the lo/up
    coefficients; crd flips the sign of V)."""
    fmt = resolve_format(fmt)
    rhs = np.asarray(rhs, dtype=np.float64)
    if maxit is None:
        maxit = default_maxit(rhs.size)
    with _ctx_for(s, fmt, "S", s_transpose) as ctx:
        ctx.set_rounding(rounding_mode(rounding), dot_format(fmt, strict_model).name)
        y, st = ctx.s_solve(rhs, tol, maxit)
    nrhs = float(np.linalg.norm(rhs))
    return y, InnerSolveStats(st.iterations, st.final_relative_residual, bool(st.converged),
                              bool(st.breakdown), _true_relres(s, rhs, y, nrhs))
