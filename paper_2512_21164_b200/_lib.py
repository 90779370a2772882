"""ctypes binding of the C ABI in ``include/gadi_b200.h``.

The shared library ``libgadi_b200.so`` is built in-tree (``make -C
paper_2512_21164_b200/csrc`` or ``__graft_entry__.build()``).  There is no
CPU fallback: every compute entry point of this package goes through this
library, and :func:`lib` raises if it is missing or no CUDA device exists.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("GADI_LIB") or Path(__file__).resolve().parent / "libgadi_b200.so")
CSRC = Path(__file__).resolve().parent / "csrc"

GADI_OK, GADI_ERR_CUDA, GADI_ERR_ARG, GADI_ERR_OOM, GADI_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
FMT_CODES = {"bf16": 0, "fp16": 1, "fp32": 2, "fp64": 3, "fp64x2": 4}
KIND_STENCIL, KIND_COMPLEX, KIND_CSR = 0, 1, 2


class Coef(C.Structure):
    _fields_ = [("d", C.c_double), ("lo", C.c_double * 3), ("up", C.c_double * 3)]

    @classmethod
    def make(cls, d, lo, up):
        c = cls()
        c.d = float(d)
        for i in range(3):
            c.lo[i] = float(lo[i])
            c.up[i] = float(up[i])
        return c


class Csr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("nnz", C.c_int64),
                ("row_offsets", C.POINTER(C.c_int64)),
                ("col_indices", C.POINTER(C.c_int64)),
                ("values", C.POINTER(C.c_double))]


class ProblemDesc(C.Structure):
    _fields_ = [("kind", C.c_int), ("ndim", C.c_int), ("dims", C.c_int64 * 3),
                ("n", C.c_int64), ("A", Coef), ("H", Coef), ("S", Coef),
                ("alpha_s", C.c_double), ("v", C.POINTER(C.c_double)),
                ("csr_A", Csr), ("csr_H", Csr), ("csr_S", Csr), ("csr_ST", Csr),
                ("u", C.c_int), ("u_r", C.c_int), ("u_s", C.c_int)]


class OuterScalars(C.Structure):
    _fields_ = [("sum_r2", C.c_double), ("max_r", C.c_double),
                ("sum_ralg2", C.c_double), ("sum_x2", C.c_double),
                ("sum_e2", C.c_double), ("sum_ae2", C.c_double)]


class InnerStats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int),
                ("breakdown", C.c_int), ("pad", C.c_int),
                ("final_relative_residual", C.c_double)]


class PhaseTimes(C.Structure):
    _fields_ = [("residual", C.c_double), ("inner_h", C.c_double),
                ("inner_s", C.c_double), ("update", C.c_double),
                ("monitor", C.c_double)]


class StepArgs(C.Structure):
    _fields_ = [("scale", C.c_double), ("coeff", C.c_double),
                ("inner_tol", C.c_double), ("maxit_h", C.c_int),
                ("maxit_s", C.c_int), ("use_graph", C.c_int)]


_DP = C.POINTER(C.c_double)
_VP = C.c_void_p

# name -> (restype, argtypes); every symbol declared in include/gadi_b200.h
SIGNATURES = {
    "gadi_last_error": (C.c_char_p, []),
    "gadi_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "gadi_build_info": (C.c_char_p, []),
    "gadi_ctx_create": (C.c_int, [C.POINTER(ProblemDesc), C.c_int, C.POINTER(_VP)]),
    "gadi_ctx_destroy": (C.c_int, [_VP]),
    "gadi_set_rhs": (C.c_int, [_VP, _DP]),
    "gadi_gen_rhs_ones": (C.c_int, [_VP]),
    "gadi_get_rhs": (C.c_int, [_VP, _DP]),
    "gadi_set_exact": (C.c_int, [_VP, _DP, C.c_int]),
    "gadi_norm2": (C.c_int, [_VP, _DP, C.c_uint64, C.c_double, C.c_int, _DP, C.POINTER(C.c_int)]),
    "gadi_outer_begin": (C.c_int, [_VP, C.POINTER(OuterScalars)]),
    "gadi_outer_step": (C.c_int, [_VP, C.POINTER(StepArgs), C.POINTER(OuterScalars),
                                  C.POINTER(InnerStats), C.POINTER(InnerStats),
                                  C.POINTER(PhaseTimes)]),
    "gadi_get_x": (C.c_int, [_VP, _DP]),
    "gadi_h_solve": (C.c_int, [_VP, _DP, C.c_double, C.c_int, _DP, C.POINTER(InnerStats)]),
    "gadi_s_solve": (C.c_int, [_VP, _DP, C.c_double, C.c_int, _DP, C.POINTER(InnerStats)]),
    "gadi_spmv": (C.c_int, [_VP, C.c_int, C.c_int, _DP, _DP]),
    "gadi_residual": (C.c_int, [_VP, _DP, _DP]),
    "gadi_set_rounding": (C.c_int, [_VP, C.c_int, C.c_int]),
    "gadi_comm_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "gadi_comm_create_nccl": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(_VP)]),
    "gadi_comm_create_local": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(_VP)]),
    "gadi_comm_create_local2": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_VP)]),
    "gadi_ctx_comm_kind": (C.c_char_p, [_VP]),
    "gadi_comm_create_host": (C.c_int, [C.c_int, C.c_int, C.POINTER(_VP)]),
    "gadi_ctx_peer_export": (C.c_int, [_VP, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "gadi_ctx_peer_attach": (C.c_int, [_VP, C.c_void_p, C.c_size_t]),
    "gadi_comm_destroy": (C.c_int, [_VP]),
    "gadi_comm_info": (C.c_int, [_VP, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "gadi_ctx_create_slab": (C.c_int, [C.POINTER(ProblemDesc), C.c_int, _VP, C.c_int64, C.c_int64,
                                       C.POINTER(_VP)]),
    "gadi_ctx_slab": (C.c_int, [_VP, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "gadi_prof_enable": (C.c_int, [_VP, C.c_int]),
    "gadi_prof_read": (C.c_int, [_VP, C.c_int, _DP, C.POINTER(C.c_int64)]),
    "gadi_timer_start": (C.c_int, [_VP]),
    "gadi_timer_stop": (C.c_int, [_VP, _DP]),
    "gadi_last_norm_ms": (C.c_double, [_VP]),
    "gadi_kernel_launches": (C.c_int64, [_VP]),
}

_LIB = None


class GpuUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing (there is no CPU path)."""


def load(path: str | os.PathLike | None = None):
    """dlopen the library and attach signatures (no device needed)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise GpuUnavailable(
            f"{p} is missing: build it with `make -C {CSRC}` or __graft_entry__.build()")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _LIB = lib
    return lib


def device_count() -> int:
    n = C.c_int(0)
    rc = load().gadi_device_count(C.byref(n))
    return int(n.value) if rc == 0 else 0


def lib():
    """The loaded library, after checking that a CUDA device is present."""
    L = load()
    if device_count() < 1:
        raise GpuUnavailable("no CUDA device: the GADI hot path runs only on the GPU")
    return L


def check(rc: int) -> None:
    if rc != GADI_OK:
        msg = load().gadi_last_error().decode(errors="replace")
        if rc == GADI_ERR_OOM:
            raise MemoryError(msg)
        if rc == GADI_ERR_UNSUPPORTED:
            raise NotImplementedError(msg)
        if rc == GADI_ERR_ARG:
            raise ValueError(msg)
        raise RuntimeError(f"gadi_b200 CUDA error: {msg}")


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_DP)


class Context:
    """Owns one ``gadi_ctx`` (device buffers + stream)."""

    def __init__(self, desc: ProblemDesc, device: int = 0, comm=None, slab=None):
        """``comm`` (dist.SlabComm) and ``slab`` = (x0, x1): a slab context of
        the decomposition owning global planes [x0, x1); vectors crossing
        this context are the slab's rows."""
        self._L = lib()
        self._desc = desc  # keep host arrays referenced during creation
        h = C.c_void_p()
        if comm is None:
            check(self._L.gadi_ctx_create(C.byref(desc), int(device), C.byref(h)))
        else:
            x0, x1 = slab
            check(self._L.gadi_ctx_create_slab(C.byref(desc), int(device), comm.h, int(x0), int(x1),
                                               C.byref(h)))
        self.h = h
        self.comm = comm
        if comm is None:
            self.n = int(desc.n)
            self.slab = None
        else:
            a, b, m = C.c_int64(), C.c_int64(), C.c_int64()
            check(self._L.gadi_ctx_slab(h, C.byref(a), C.byref(b), C.byref(m)))
            self.n = int(m.value)
            self.slab = (int(a.value), int(b.value))
            if getattr(comm, "kind", "") == "host":
                self._attach_peer(comm)

    def _attach_peer(self, comm):
        """Peer transport with the blob exchange over torch.distributed
        (dist.SlabComm.host): every rank of the group must create the same
        slab contexts in the same order."""
        import torch.distributed as dist

        n = C.c_size_t()
        check(self._L.gadi_ctx_peer_export(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(self._L.gadi_ctx_peer_export(self.h, buf, n.value, C.byref(n)))
        blobs = [None] * comm.nranks
        dist.all_gather_object(blobs, buf.raw, group=comm.group)
        allb = b"".join(blobs)
        check(self._L.gadi_ctx_peer_attach(self.h, allb, n.value))

    def close(self):
        if getattr(self, "h", None):
            self._L.gadi_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- data movement
    def set_rhs(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        check(self._L.gadi_set_rhs(self.h, dptr(b)))

    def gen_rhs_ones(self):
        check(self._L.gadi_gen_rhs_ones(self.h))

    def get_rhs(self) -> np.ndarray:
        out = np.empty(self.n)
        check(self._L.gadi_get_rhs(self.h, dptr(out)))
        return out

    def set_exact(self, xs=None, all_ones=False):
        if xs is None:
            check(self._L.gadi_set_exact(self.h, None, 1 if all_ones else 0))
        else:
            xs = np.ascontiguousarray(xs, dtype=np.float64)
            check(self._L.gadi_set_exact(self.h, dptr(xs), 0))

    def get_x(self, out=None) -> np.ndarray:
        if out is None:
            out = np.empty(self.n)
        check(self._L.gadi_get_x(self.h, dptr(out)))
        return out

    # -- compute
    def norm2(self, v0=None, seed=12345, tol=1e-6, maxit=1000):
        sig = C.c_double(0.0)
        it = C.c_int(0)
        if v0 is not None:
            v0 = np.ascontiguousarray(v0, dtype=np.float64)
            check(self._L.gadi_norm2(self.h, dptr(v0), seed, tol, maxit, C.byref(sig), C.byref(it)))
        else:
            check(self._L.gadi_norm2(self.h, None, seed, tol, maxit, C.byref(sig), C.byref(it)))
        return float(sig.value), int(it.value)

    def outer_begin(self) -> OuterScalars:
        o = OuterScalars()
        check(self._L.gadi_outer_begin(self.h, C.byref(o)))
        return o

    def outer_step(self, scale, coeff, inner_tol, maxit_h, maxit_s, use_graph=False):
        a = StepArgs(float(scale), float(coeff), float(inner_tol), int(maxit_h), int(maxit_s),
                     1 if use_graph else 0)
        o, hs, ss, t = OuterScalars(), InnerStats(), InnerStats(), PhaseTimes()
        check(self._L.gadi_outer_step(self.h, C.byref(a), C.byref(o), C.byref(hs), C.byref(ss),
                                      C.byref(t)))
        return o, hs, ss, t

    def h_solve(self, rhs, tol, maxit):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.empty(self.n)
        st = InnerStats()
        check(self._L.gadi_h_solve(self.h, dptr(rhs), float(tol), int(maxit), dptr(x), C.byref(st)))
        return x, st

    def s_solve(self, rhs, tol, maxit):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.empty(self.n)
        st = InnerStats()
        check(self._L.gadi_s_solve(self.h, dptr(rhs), float(tol), int(maxit), dptr(x), C.byref(st)))
        return x, st

    def spmv(self, op: int, x, strict=False) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.n)
        check(self._L.gadi_spmv(self.h, int(op), 1 if strict else 0, dptr(x), dptr(y)))
        return y

    def residual(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        r = np.empty(self.n)
        check(self._L.gadi_residual(self.h, dptr(x), dptr(r)))
        return r

    def set_rounding(self, mode: int, dot_fmt: str):
        check(self._L.gadi_set_rounding(self.h, int(mode), FMT_CODES[dot_fmt]))

    KERNELS = ["hcg_init", "hcg_a", "hcg_b", "cgnr_init", "cgnr_p1", "cgnr_p2", "cgnr_p3",
               "crd_init", "crd_p1", "crd_p2", "outer", "norm_a", "norm_b", "apply", "dot_tree", "hcg_z"]

    def prof_enable(self, on=True):
        check(self._L.gadi_prof_enable(self.h, 1 if on else 0))

    def prof_read(self) -> dict:
        out = {}
        for k, name in enumerate(self.KERNELS):
            ms, n = C.c_double(0.0), C.c_int64(0)
            check(self._L.gadi_prof_read(self.h, k, C.byref(ms), C.byref(n)))
            if n.value:
                out[name] = (float(ms.value), int(n.value))
        return out

    def timer_start(self):
        check(self._L.gadi_timer_start(self.h))

    def timer_stop(self) -> float:
        ms = C.c_double(0.0)
        check(self._L.gadi_timer_stop(self.h, C.byref(ms)))
        return float(ms.value)

    def comm_kind(self) -> str:
        return self._L.gadi_ctx_comm_kind(self.h).decode()

    def last_norm_ms(self) -> float:
        return float(self._L.gadi_last_norm_ms(self.h))

    def kernel_launches(self) -> int:
        return int(self._L.gadi_kernel_launches(self.h))
