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
from .errors import SingularMatrix, ZeroError, ZeroReference
from .stencil import StencilMatrix

__all__ = ["forward_error", "backward_error", "mu_k", "matrix_norm_2", "HOST_START_MAX",
           "power_start_vector", "condition_estimate", "DENSE_CAP"]

DENSE_CAP = 2048  # REF/analysis.py: dense SVD below this many rows

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


# ---------------------------------------------------------------- condition numbers
# The tau-gate of select_alpha (REF/alphaselect.py:245-251) multiplies the
# 2-norm condition numbers of the fp64 HSS operators H = alpha I + M and
# S = alpha I + N.  For the stencil families both are Kronecker sums of
# constant tridiagonal Toeplitz factors (REF/problems.py:42-120), so their
# spectra are known in closed form -- H symmetric:
#   lambda = alpha + d + sum_a 2 m_a cos(k_a pi / (n_a + 1)),  m_a = (lo_a + up_a) / 2;
# S normal (alpha I plus a real skew-symmetric Kronecker sum):
#   sigma = sqrt(alpha^2 + mu^2),  mu = sum_a 2 s_a cos(k_a pi / (n_a + 1)),  s_a = (up_a - lo_a) / 2;
# crd: S = alpha I + [[0, -V], [V, 0]] has sigma = sqrt(alpha^2 + v_i^2).
# These are the exact condition numbers (the reference's dense SVD to
# rounding; above its 2048-row cap the reference estimates them with power /
# inverse iteration to 1e-6).  Other operators take the reference's route:
# dense SVD below the cap, else the power iteration for ||A|| and inverse
# iteration through a sparse LU for ||A^-1|| (REF/analysis.py:106-134).
def _axis_cos(n: int) -> np.ndarray:
    return np.cos(np.arange(1, n + 1) * np.pi / (n + 1))


def _min_abs_sum(sets) -> float:
    """min |e_1 + ... + e_k| over one element of each set (k <= 3)."""
    sets = [np.sort(np.asarray(v, dtype=np.float64)) for v in sets if np.size(v)]
    if not sets:
        return 0.0
    if len(sets) == 1:
        return float(np.min(np.abs(sets[0])))
    base = sets[0]
    for extra in sets[1:-1]:
        base = np.sort((base[:, None] + extra[None, :]).ravel())
    last = sets[-1]
    pos = np.clip(np.searchsorted(base, -last), 0, base.size - 1)
    best = np.minimum(np.abs(base[pos] + last), np.abs(base[np.maximum(pos - 1, 0)] + last))
    return float(np.min(best))


def _stencil_condition(a: StencilMatrix) -> float | None:
    if a.role not in ("H", "S") or a.fmt.name != "fp64":
        return None
    sp, alpha = a.spec, float(a.alpha)
    c = sp.A
    axes = [ax for ax, n in enumerate(sp.dims) if n > 1]
    if a.role == "H":
        spread = sum(2.0 * abs(0.5 * (c.lo[ax] + c.up[ax])) * np.cos(np.pi / (sp.dims[ax] + 1)) for ax in axes)
        centre = alpha + c.d
        lo, hi = centre - spread, centre + spread
        if lo <= 0.0:
            return None  # indefinite: take the numerical route
        return float(hi / lo)
    if sp.family == "crd":
        v = np.abs(np.asarray(sp.v, dtype=np.float64))
        if np.any(0.5 * (np.asarray(c.lo) - np.asarray(c.up)) != 0.0):
            return None
        return float(np.sqrt(alpha * alpha + v.max() ** 2) / np.sqrt(alpha * alpha + v.min() ** 2))
    sets = [2.0 * 0.5 * (c.up[ax] - c.lo[ax]) * _axis_cos(sp.dims[ax]) for ax in axes
            if c.up[ax] != c.lo[ax]]
    mu_max = sum(float(np.max(np.abs(e))) for e in sets)
    mu_min = _min_abs_sum(sets)
    return float(np.sqrt(alpha * alpha + mu_max * mu_max) / np.sqrt(alpha * alpha + mu_min * mu_min))


def condition_estimate(a, dense_cap: int = DENSE_CAP) -> float:
    """2-norm condition number (REF/analysis.py:106-134)."""
    if isinstance(a, StencilMatrix):
        k = _stencil_condition(a)
        if k is not None:
            return k
    n = a.nrows
    if n <= dense_cap:
        dense = a.to_scipy().toarray() if isinstance(a, StencilMatrix) else a.to_dense()
        sv = np.linalg.svd(dense, compute_uv=False)
        if sv[-1] == 0.0:
            raise SingularMatrix("zero singular value")
        return float(sv[0] / sv[-1])
    import scipy.sparse.linalg as spla

    m = a.to_scipy().tocsc()
    norm_a = matrix_norm_2(a)
    try:
        lu = spla.splu(m)
    except RuntimeError as exc:
        raise SingularMatrix(str(exc)) from exc
    v = np.random.default_rng(_POWER_SEED).standard_normal(n)
    v /= np.linalg.norm(v)
    sigma_inv = 0.0
    for _ in range(_POWER_MAXIT):
        w = lu.solve(lu.solve(v, trans="N"), trans="T")  # (A^T A)^-1 v
        nw = float(np.linalg.norm(w))
        if not np.isfinite(nw):
            raise SingularMatrix("inverse iteration diverged")
        s_new = float(np.sqrt(nw))
        v = w / nw
        done = abs(s_new - sigma_inv) <= _POWER_TOL * s_new
        sigma_inv = s_new
        if done:
            break
    return float(norm_a * sigma_inv)
