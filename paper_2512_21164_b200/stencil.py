"""Matrix-free stencil operators for the three problem families.

The reference builds every operator as an explicit CSR matrix with scipy
(gadimp/problems.py:48-120, splitting.py:38-55).  On the GPU the operators
are constant-coefficient 5-point / 7-point stencils (plus the diagonal
potential V of the complex family), so only their coefficients are needed.
This module derives those coefficients with the *same fp64 operation
sequence* scipy performs when the reference assembles the matrices, so the
values are bitwise the CSR values:

* cdr2d  T = tridiag(-1,2,-1) + 2r tridiag(0.5,0,-0.5) + react I,
         A = I (x) T + T (x) I                           problems.py:48-66
* cd3d   A = T_x (x) I (x) I + I (x) T_yz (x) I + I (x) I (x) T_yz
                                                         problems.py:69-93
* crd    A = [[L, -V], [V, L]], L = scale (I (x) t + t (x) I)
                                                         problems.py:96-120
* M = (A + A^T) * 0.5, N = (A - A^T) * 0.5, H = M + alpha I, S = N + alpha I
                                                         sparsemat.py:155-172

A :class:`StencilMatrix` quacks like ``SparseMatrix`` (shape, nnz,
``to_scipy()``, ``quantized()``); its CSR form is only materialised on
request (small problems, tests).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .precision import quantize, resolve_format

__all__ = ["Coefs", "StencilSpec", "StencilMatrix", "spec_cdr_2d", "spec_cd_3d", "spec_complex_rd",
           "splitting_coefs", "recognise"]

# axis order everywhere: 0 = x (slowest), 1 = y, 2 = z (fastest)


@dataclass(frozen=True)
class Coefs:
    """d on the diagonal; lo[a] / up[a] multiply the neighbour along axis a
    with the smaller / larger linear index.  0.0 means "entry not stored"."""

    d: float
    lo: tuple
    up: tuple

    def transpose(self) -> "Coefs":
        return Coefs(self.d, tuple(self.up), tuple(self.lo))

    def quantized(self, fmt) -> "Coefs":
        q = lambda v: float(quantize(float(v), fmt))  # noqa: E731
        return Coefs(q(self.d), tuple(q(v) for v in self.lo), tuple(q(v) for v in self.up))

    def negated_offdiag(self) -> "Coefs":
        return Coefs(self.d, tuple(-v for v in self.lo), tuple(-v for v in self.up))


@dataclass(frozen=True)
class StencilSpec:
    """Operator family + grid + fp64 coefficients of A (crd: of L, plus v)."""

    family: str          # "cdr2d" | "cd3d" | "crd"
    n_g: int
    ndim: int            # 2 or 3 (grid dimension)
    A: Coefs             # real families: A ; crd: L
    params: dict = field(default_factory=dict)
    v: np.ndarray | None = None  # crd potential s * xi (n_g^2 values)

    @property
    def dims(self):
        return (self.n_g, 1, self.n_g) if self.ndim == 2 else (self.n_g,) * 3

    @property
    def n(self) -> int:
        m = self.n_g ** self.ndim
        return 2 * m if self.family == "crd" else m


def spec_cdr_2d(n_g: int, r: float = 1.0) -> StencilSpec:
    react = 100.0 / (n_g + 1) ** 2
    two_r = 2.0 * r
    t_d = 2.0 + react
    t_lo = -1.0 + two_r * 0.5
    t_up = -1.0 + two_r * -0.5
    a = Coefs(t_d + t_d, (t_lo, 0.0, t_lo), (t_up, 0.0, t_up))
    return StencilSpec("cdr2d", int(n_g), 2, a, {"n_g": n_g, "r": r})


def spec_cd_3d(n_g: int) -> StencilSpec:
    r = 1.0 / (2 * n_g + 2)
    lo, up = -1.0 - r, -1.0 + r
    a = Coefs(6.0, (lo, lo, lo), (up, up, up))
    return StencilSpec("cd3d", int(n_g), 3, a, {"n_g": n_g, "r": r})


def crd_potential(n_g: int, s: float, seed: int, ndim: int = 2) -> np.ndarray:
    xi = np.random.Generator(np.random.Philox(key=seed)).uniform(size=n_g ** ndim)
    return s * xi


def spec_complex_rd(n_g: int, s: float = 1.0e4, seed: int = 0,
                    laplacian_scaling: str = "nu_over_h2", ndim: int = 2) -> StencilSpec:
    """crd (REF/problems.py:96-120).  ``ndim=3`` is the 3-D extension of
    BASELINE config 5 (no reference generator): the same recipe
    with the 7-point Laplacian scale*(t(x)I(x)I + I(x)t(x)I + I(x)I(x)t), whose
    diagonal 2+2+2 = 6 is exact before the scaling, and V over n_g^3 points."""
    if ndim not in (2, 3):
        raise ValueError("ndim must be 2 or 3")
    nu = 1.0e-5 * (64.0 / n_g) ** 2
    h = 1.0 / (n_g + 1)
    sc = nu / h ** 2 if laplacian_scaling == "nu_over_h2" else nu
    off = sc * -1.0
    if ndim == 2:
        lap = Coefs(sc * 4.0, (off, 0.0, off), (off, 0.0, off))
    else:
        lap = Coefs(sc * 6.0, (off, off, off), (off, off, off))
    v = crd_potential(n_g, s, seed, ndim)
    params = {"n_g": n_g, "s": s, "seed": seed, "nu": nu, "laplacian_scaling": laplacian_scaling}
    if ndim == 3:
        params["ndim"] = 3
    return StencilSpec("crd", int(n_g), ndim, lap, params, v)


@dataclass(frozen=True)
class SplitCoefs:
    """fp64 coefficients of M, N, H, S and the u_s images used by the inner
    solvers (splitting.py:38-55)."""

    M: Coefs
    N: Coefs
    H: Coefs
    S: Coefs
    H_low: Coefs
    S_low: Coefs
    alpha_low: float  # crd: u_s image of the S diagonal
    v_low: np.ndarray | None


def splitting_coefs(spec: StencilSpec, alpha: float, u_s) -> SplitCoefs:
    u_s = resolve_format(u_s)
    a = spec.A
    if spec.family == "crd":
        # M = blockdiag(L, L) exactly ((x + x) * 0.5 = x); N = [[0, -V], [V, 0]]
        m = a
        n = Coefs(0.0, (0.0,) * 3, (0.0,) * 3)
        h = Coefs(a.d + alpha, a.lo, a.up)
        s = Coefs(alpha, (0.0,) * 3, (0.0,) * 3)
        return SplitCoefs(m, n, h, s, h.quantized(u_s), s.quantized(u_s),
                          float(quantize(float(alpha), u_s)), quantize(spec.v, u_s))
    m_off = tuple((lo + up) * 0.5 for lo, up in zip(a.lo, a.up))
    n_lo = tuple((lo - up) * 0.5 for lo, up in zip(a.lo, a.up))
    n_up = tuple((up - lo) * 0.5 for lo, up in zip(a.lo, a.up))
    m = Coefs((a.d + a.d) * 0.5, m_off, m_off)
    n = Coefs(0.0, n_lo, n_up)
    h = Coefs(m.d + alpha, m_off, m_off)
    s = Coefs(alpha, n_lo, n_up)
    return SplitCoefs(m, n, h, s, h.quantized(u_s), s.quantized(u_s), float(quantize(float(alpha), u_s)), None)


# ---------------------------------------------------------------- CSR view
def _stencil_csr(spec: StencilSpec, c: Coefs, v_diag_block=None):
    """Assemble the CSR of a constant stencil (rows ascending by column) --
    host-side representation only, used to hand operators to code that wants
    an explicit matrix (tests, small problems)."""
    import scipy.sparse as sp

    dims = spec.dims
    nx, ny, nz = dims
    m = nx * ny * nz
    idx = np.arange(m, dtype=np.int64)
    xi, rem = np.divmod(idx, ny * nz)
    yi, zi = np.divmod(rem, nz)
    strides = (ny * nz, nz, 1)
    coords = (xi, yi, zi)
    ext = (nx, ny, nz)
    rows, cols, vals = [], [], []
    for ax in (0, 1, 2):
        if c.lo[ax] != 0.0:
            msk = coords[ax] > 0
            rows.append(idx[msk]); cols.append(idx[msk] - strides[ax]); vals.append(np.full(msk.sum(), c.lo[ax]))
    if c.d != 0.0:
        rows.append(idx); cols.append(idx); vals.append(np.full(m, c.d))
    for ax in (2, 1, 0):
        if c.up[ax] != 0.0:
            msk = coords[ax] < ext[ax] - 1
            rows.append(idx[msk]); cols.append(idx[msk] + strides[ax]); vals.append(np.full(msk.sum(), c.up[ax]))
    r = np.concatenate(rows) if rows else np.zeros(0, np.int64)
    cc = np.concatenate(cols) if cols else np.zeros(0, np.int64)
    vv = np.concatenate(vals) if vals else np.zeros(0)
    return sp.csr_matrix((vv, (r, cc)), shape=(m, m))


class StencilMatrix:
    """A matrix-free operator described by a :class:`StencilSpec`.

    ``role`` selects which operator of the splitting it is ("A", "M", "N",
    "H", "S", "ST", "AmN" for alpha I - N); ``fmt`` is the precision its
    coefficients were rounded to (``quantized``)."""

    def __init__(self, spec: StencilSpec, role: str = "A", alpha: float = 0.0, fmt="fp64"):
        self.spec = spec
        self.role = role
        self.alpha = float(alpha)
        self.fmt = resolve_format(fmt)
        self._csr = None

    # -- SparseMatrix-compatible surface
    @property
    def nrows(self) -> int:
        return self.spec.n

    @property
    def ncols(self) -> int:
        return self.spec.n

    @property
    def shape(self):
        return (self.spec.n, self.spec.n)

    @property
    def is_square(self) -> bool:
        return True

    @property
    def nnz(self) -> int:
        return int(self.to_scipy().nnz)

    def quantized(self, fmt) -> "StencilMatrix":
        fmt = resolve_format(fmt)
        if fmt.significand_bits >= 53:
            return self
        return StencilMatrix(self.spec, self.role, self.alpha, fmt)

    def coefs(self) -> Coefs:
        """fp64 (or quantised) coefficients of this operator (real families)."""
        if self.role == "A":
            c = self.spec.A
        else:
            sc = splitting_coefs(self.spec, self.alpha, "fp64")
            c = {"M": sc.M, "N": sc.N, "H": sc.H, "S": sc.S, "ST": sc.S.transpose(),
                 "AmN": Coefs(self.alpha, tuple(-v for v in sc.N.lo), tuple(-v for v in sc.N.up))}[self.role]
        return c.quantized(self.fmt) if self.fmt.significand_bits < 53 else c

    def to_scipy(self):
        if self._csr is None:
            import scipy.sparse as sp

            spec = self.spec
            if spec.family != "crd":
                self._csr = _stencil_csr(spec, self.coefs())
            else:
                sc = splitting_coefs(spec, self.alpha, "fp64")
                zero = (0.0, 0.0, 0.0)
                lc = {"A": spec.A, "M": spec.A, "H": sc.H, "N": Coefs(0.0, zero, zero)}.get(
                    self.role, Coefs(self.alpha, zero, zero))
                low = self.fmt.significand_bits < 53
                if low:
                    lc = lc.quantized(self.fmt)
                L = _stencil_csr(spec, lc)
                sign = {"A": 1.0, "N": 1.0, "S": 1.0, "ST": -1.0, "AmN": -1.0, "M": 0.0, "H": 0.0}[self.role]
                v = quantize(spec.v, self.fmt) if low else spec.v
                V = sp.diags(sign * v, format="csr")
                self._csr = sp.bmat([[L, -V], [V, L]], format="csr")
            self._csr.sort_indices()
            self._csr.eliminate_zeros()
        return self._csr

    def to_dense(self) -> np.ndarray:
        return self.to_scipy().toarray()

    @property
    def row_offsets(self):
        return self.to_scipy().indptr.astype(np.int64)

    @property
    def col_indices(self):
        return self.to_scipy().indices.astype(np.int64)

    @property
    def values(self):
        return self.to_scipy().data

    def diagonal(self):
        return self.to_scipy().diagonal()

    def __repr__(self):
        return f"StencilMatrix({self.spec.family} n_g={self.spec.n_g}, role={self.role}, fmt={self.fmt})"


# ---------------------------------------------------------------- recognition
def recognise(problem) -> StencilSpec | None:
    """Map a problem to a stencil spec.

    Problems built by this package carry their spec.  Problems built
    elsewhere (e.g. by the reference package, or read from Matrix Market with
    the CLI sidecar, cli.py:56-68) are recognised from ``label`` + ``params``
    and then *verified*: the whole CSR (row offsets, column indices, value
    bits) must equal the stencil's, otherwise the general CSR path is used.
    """
    a = problem.A
    if isinstance(a, StencilMatrix) and a.role == "A":
        return a.spec
    label = getattr(problem, "label", None)
    params = getattr(problem, "params", None) or {}
    try:
        if label == "cdr2d":
            spec = spec_cdr_2d(int(params["n_g"]), float(params.get("r", 1.0)))
        elif label == "cd3d":
            spec = spec_cd_3d(int(params["n_g"]))
        elif label in ("crd", "crd3d"):
            spec = spec_complex_rd(int(params["n_g"]), float(params.get("s", 1.0e4)),
                                   int(params.get("seed", 0)),
                                   params.get("laplacian_scaling", "nu_over_h2"),
                                   3 if label == "crd3d" else int(params.get("ndim", 2)))
        else:
            return None
    except (KeyError, TypeError, ValueError):
        return None
    if getattr(a, "nrows", None) != spec.n or not csr_equals(a, StencilMatrix(spec)):
        return None
    return spec


def csr_equals(a, b) -> bool:
    """Bitwise equality of two CSR operators (O(nnz), vectorised): the same
    row offsets, column indices and value bit patterns."""
    def parts(m):
        if all(hasattr(m, k) for k in ("row_offsets", "col_indices", "values")):
            return (np.asarray(v) for v in (m.row_offsets, m.col_indices, m.values))
        c = m.to_scipy()
        return np.asarray(c.indptr), np.asarray(c.indices), np.asarray(c.data)

    try:
        ra, ca, va = parts(a)
        rb, cb, vb = parts(b)
    except AttributeError:
        return False
    if ra.shape != rb.shape or ca.shape != cb.shape or va.shape != vb.shape:
        return False
    return (np.array_equal(ra, rb) and np.array_equal(ca, cb)
            and np.array_equal(np.asarray(va, dtype=np.float64).view(np.uint64),
                               np.asarray(vb, dtype=np.float64).view(np.uint64)))


def same_spec(a: StencilSpec, b: StencilSpec) -> bool:
    """Two specs describe the same operator (the fp64 coefficients, grid and
    crd potential are what the kernels consume)."""
    if a is b:
        return True
    if (a.family, a.n_g, a.ndim, a.A) != (b.family, b.n_g, b.ndim, b.A):
        return False
    if (a.v is None) != (b.v is None):
        return False
    return a.v is None or a.v is b.v or np.array_equal(np.asarray(a.v).view(np.uint64),
                                                       np.asarray(b.v).view(np.uint64))


def splitting_matches(splitting, spec: StencilSpec) -> bool:
    """True when a supplied splitting is the HSS splitting of the stencil
    (its u_s operators H_low, S_low, S_low_T bitwise those the stencil path
    builds from (spec, alpha, splitting.u_s)); any other splitting must run
    on its own matrices through the CSR engine."""
    roles = (("H_low", "H"), ("S_low", "S"), ("S_low_T", "ST"))
    for attr, role in roles:
        m = getattr(splitting, attr)
        if isinstance(m, StencilMatrix) and same_spec(m.spec, spec):
            if m.role != role or float(m.alpha) != float(splitting.alpha) or m.fmt.name != splitting.u_s.name:
                return False
        elif not csr_equals(m, StencilMatrix(spec, role, splitting.alpha, splitting.u_s)):
            return False
    return True


def with_params(spec: StencilSpec, **kw) -> StencilSpec:
    return replace(spec, **kw)
