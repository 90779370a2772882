"""Error metrics and the ||A||_2 estimate (gadimp/analysis.py:43-96).

``matrix_norm_2`` is the power iteration on A^T A of the reference
(analysis.py:51-70: start vector N(0,1) from default_rng(12345), tol 1e-6,
<= 1000 iterations) run on the GPU (csrc/passes.cuh NormPass).  Up to
``HOST_START_MAX`` unknowns the reference's own numpy start vector is
uploaded so the estimate is comparable to the reference's to rounding; above
it a device generator avoids generating 10^8 normals on the host (both
estimates agree to the power-iteration tolerance).
"""

from __future__ import annotations

import numpy as np

from .device import is_csr, make_csr_desc, make_desc, open_context
from .errors import ZeroError, ZeroReference
from .stencil import StencilMatrix

__all__ = ["forward_error", "backward_error", "mu_k", "matrix_norm_2", "HOST_START_MAX",
           "power_start_vector"]

_POWER_TOL = 1.0e-6
_POWER_MAXIT = 1000
_POWER_SEED = 12345
HOST_START_MAX = 1 << 22


def power_start_vector(n: int):
    """The reference's normalised start vector (analysis.py:54-57), or None
    above HOST_START_MAX (device generator)."""
    if n > HOST_START_MAX:
        return None
    v = np.random.default_rng(_POWER_SEED).standard_normal(n)
    v /= np.linalg.norm(v)
    return v


def matrix_norm_2(a, tol: float = _POWER_TOL, maxit: int = _POWER_MAXIT) -> float:
    if is_csr(a):
        with open_context(make_csr_desc(a, a, a, a, "fp64")) as ctx:
            sigma, _ = ctx.norm2(power_start_vector(a.nrows), _POWER_SEED, tol, maxit)
        return sigma
    if not isinstance(a, StencilMatrix) or a.role != "A":
        raise NotImplementedError("matrix_norm_2 runs on stencil system matrices")
    with open_context(make_desc(a.spec, 1.0, "fp64")) as ctx:
        sigma, _ = ctx.norm2(power_start_vector(a.nrows), _POWER_SEED, tol, maxit)
    return sigma


def forward_error(xhat: np.ndarray, x: np.ndarray) -> float:
    nx = float(np.linalg.norm(x))
    if nx == 0.0:
        raise ZeroReference("reference solution has zero norm")
    return float(np.linalg.norm(np.asarray(xhat) - np.asarray(x))) / nx


def backward_error(a, b: np.ndarray, xhat: np.ndarray, norm_a: float | None = None) -> float:
    from .sparsemat import residual

    b = np.asarray(b, dtype=np.float64)
    xhat = np.asarray(xhat, dtype=np.float64)
    if norm_a is None:
        norm_a = matrix_norm_2(a)
    nb = float(np.linalg.norm(b))
    denom = norm_a * float(np.linalg.norm(xhat)) + nb
    if denom == 0.0:
        raise ZeroReference("both A and b have zero norm")
    return float(np.linalg.norm(residual(a, xhat, b, "fp64"))) / denom


def mu_k(a, b: np.ndarray, xhat: np.ndarray, x: np.ndarray, norm_a: float | None = None) -> float:
    from .sparsemat import spmv

    e = np.asarray(x, dtype=np.float64) - np.asarray(xhat, dtype=np.float64)
    ne = float(np.linalg.norm(e))
    if ne == 0.0:
        raise ZeroError("xhat equals x; mu is undefined")
    if norm_a is None:
        norm_a = matrix_norm_2(a)
    return float(np.linalg.norm(spmv(a, e, "fp64"))) / (norm_a * ne)
