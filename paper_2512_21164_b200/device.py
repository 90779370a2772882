"""Bridge from the reference-shaped Python objects to device contexts.

Builds ``gadi_problem_desc`` descriptors from stencil specs (the operator
coefficients of A, H = alpha I + M, S = alpha I + N and their u_s images)
and runs the public kernels (spmv, residual, inner solves, ||A||_2) through
:class:`paper_2512_21164_b200._lib.Context`.  Nothing here computes on the
CPU; a missing library or device raises ``GpuUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib
from .precision import resolve_format
from .stencil import Coefs, StencilMatrix, StencilSpec, splitting_coefs

__all__ = ["make_desc", "open_context", "spmv", "residual", "rhs_ones", "cached_context"]


def _coef(c: Coefs) -> _lib.Coef:
    return _lib.Coef.make(c.d, c.lo, c.up)


def make_desc(spec: StencilSpec, alpha: float, u_s, u="fp64", u_r="fp64", *,
              coef_fmt=None, H: Coefs | None = None, S: Coefs | None = None):
    """Descriptor for a stencil problem.  ``coef_fmt`` is the precision the
    splitting constants were rounded to (splitting.u_s; defaults to u_s)."""
    u_s = resolve_format(u_s)
    coef_fmt = resolve_format(coef_fmt) if coef_fmt is not None else u_s
    d = _lib.ProblemDesc()
    d.kind = _lib.KIND_COMPLEX if spec.family == "crd" else _lib.KIND_STENCIL
    d.ndim = spec.ndim
    dims = spec.dims
    for i in range(3):
        d.dims[i] = dims[i]
    d.n = spec.n
    sc = splitting_coefs(spec, alpha, coef_fmt) if alpha > 0 else None
    d.A = _coef(spec.A)
    d.H = _coef(H if H is not None else (sc.H_low if sc else spec.A))
    d.S = _coef(S if S is not None else (sc.S_low if sc else spec.A))
    d.alpha_s = sc.alpha_low if sc else 0.0
    keep = []
    if spec.family == "crd":
        v = np.ascontiguousarray(spec.v, dtype=np.float64)
        keep.append(v)
        d.v = v.ctypes.data_as(C.POINTER(C.c_double))
    d.u = _lib.FMT_CODES[resolve_format(u).name]
    d.u_r = _lib.FMT_CODES[resolve_format(u_r).name]
    d.u_s = _lib.FMT_CODES[u_s.name]
    d._keep = keep  # noqa: SLF001 - keep host arrays alive while the ctx is built
    return d


def _csr(m, keep):
    c = _lib.Csr()
    ro = np.ascontiguousarray(m.row_offsets, dtype=np.int64)
    ci = np.ascontiguousarray(m.col_indices, dtype=np.int64)
    va = np.ascontiguousarray(m.values, dtype=np.float64)
    keep += [ro, ci, va]
    c.nrows, c.nnz = int(m.nrows), int(va.size)
    c.row_offsets = ro.ctypes.data_as(C.POINTER(C.c_int64))
    c.col_indices = ci.ctypes.data_as(C.POINTER(C.c_int64))
    c.values = va.ctypes.data_as(C.POINTER(C.c_double))
    return c


def make_csr_desc(A, H, S, ST, u_s, u="fp64", u_r="fp64"):
    """Descriptor of a general-CSR problem (csrc/csr.cuh): A in fp64 and the
    splitting operators H_low, S_low, S_low_T with their u_s values."""
    d = _lib.ProblemDesc()
    d.kind = _lib.KIND_CSR
    d.ndim = 1
    d.dims[0], d.dims[1], d.dims[2] = int(A.nrows), 1, 1
    d.n = int(A.nrows)
    keep = []
    d.csr_A, d.csr_H, d.csr_S, d.csr_ST = (_csr(m, keep) for m in (A, H, S, ST))
    d.u = _lib.FMT_CODES[resolve_format(u).name]
    d.u_r = _lib.FMT_CODES[resolve_format(u_r).name]
    d.u_s = _lib.FMT_CODES[resolve_format(u_s).name]
    d._keep = keep  # noqa: SLF001
    return d


def is_csr(a) -> bool:
    return not isinstance(a, StencilMatrix) and hasattr(a, "row_offsets")


def open_context(desc, device: int = 0, comm=None, slab=None) -> _lib.Context:
    return _lib.Context(desc, device, comm=comm, slab=slab)


_CACHE: dict = {}
_CACHE_LOCK = threading.Lock()


def cached_context(key, make):
    """One live context per (key, thread) (reused by repeated solves of the
    same operator, e.g. warm-up + timed runs); a thread's previous context is
    released when it requests a different operator, to keep HBM free.  Per
    thread because a context is not thread-safe and slab ranks
    may run as threads of one process (dist.SlabComm.local)."""
    tid = threading.get_ident()
    with _CACHE_LOCK:
        ctx = _CACHE.get((tid, key))
        if ctx is None:
            stale = [k for k in _CACHE if k[0] == tid]
            olds = [_CACHE.pop(k) for k in stale]
        else:
            olds = []
    for o in olds:
        o.close()
    if ctx is None:
        ctx = make()
        with _CACHE_LOCK:
            _CACHE[(tid, key)] = ctx
    return ctx


def clear_cache():
    with _CACHE_LOCK:
        olds = list(_CACHE.values())
        _CACHE.clear()
    for o in olds:
        o.close()


def _require_stencil(a):
    if not isinstance(a, StencilMatrix):
        raise NotImplementedError(f"unsupported operator type {type(a).__name__}")
    return a


def _op_context(a: StencilMatrix, fmt):
    """Context whose slot H holds the coefficients of ``a`` (real families),
    or the crd family operators, with u_s = fmt for the strict apply."""
    spec = a.spec
    fmt = resolve_format(fmt)
    us = fmt if fmt.significand_bits <= 53 else resolve_format("fp64")
    if spec.family != "crd":
        c = a.coefs()
        return open_context(make_desc(spec, 0.0, us, H=c, S=c))
    return open_context(make_desc(spec, a.alpha if a.alpha > 0 else 1.0, us, coef_fmt=a.fmt))


def spmv(a, x, fmt):
    fmt = resolve_format(fmt)
    if is_csr(a):
        if fmt.compensated:
            raise NotImplementedError("fp64x2 spmv is provided through residual(..., 'fp64x2')")
        us = fmt if fmt.significand_bits < 53 else resolve_format("fp64")
        with open_context(make_csr_desc(a, a, a, a, us)) as ctx:
            return ctx.spmv(0, x) if fmt.significand_bits >= 53 else ctx.spmv(1, x, strict=True)
    a = _require_stencil(a)
    if fmt.compensated:
        raise NotImplementedError("fp64x2 spmv is provided through residual(..., 'fp64x2')")
    with _op_context(a, fmt) as ctx:
        if a.spec.family != "crd":
            return ctx.spmv(1, x, strict=True)
        if a.role == "A":
            if fmt.significand_bits < 53:
                raise NotImplementedError("crd A is applied in fp64 only")
            return ctx.spmv(0, x)
        op = {"H": 1, "S": 2, "ST": 3, "AmN": 3}.get(a.role)
        if op is None:
            raise NotImplementedError(f"crd operator {a.role}")
        return ctx.spmv(op, x, strict=True)


def residual(a, x, b, fmt):
    if is_csr(a):
        fmt = resolve_format(fmt)
        with open_context(make_csr_desc(a, a, a, a, "fp64", u="fp64", u_r=fmt)) as ctx:
            ctx.set_rhs(b)
            return ctx.residual(x)
    a = _require_stencil(a)
    if a.role != "A":
        raise NotImplementedError("residual is defined for the system matrix A")
    fmt = resolve_format(fmt)
    desc = make_desc(a.spec, 1.0, "fp64", u="fp64", u_r=fmt)
    with open_context(desc) as ctx:
        ctx.set_rhs(b)
        return ctx.residual(x)


def rhs_ones(spec: StencilSpec, device: int = 0) -> np.ndarray:
    """b = A 1 generated on the device (problems.py:42-45)."""
    desc = make_desc(spec, 0.0, "fp64")
    with open_context(desc, device) as ctx:
        ctx.gen_rhs_ones()
        return ctx.get_rhs()
