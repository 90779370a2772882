"""Benchmark problem families (drop-in for gadimp/problems.py:1-120).

``build_cdr_2d`` / ``build_cd_3d`` / ``build_complex_rd`` return problems
whose matrix is a matrix-free :class:`~.stencil.StencilMatrix` (coefficients
bitwise equal to the reference's CSR values) and whose
right-hand side b = A 1 is generated on the GPU in the reference's CSR
summation order.  Nothing of size n is built on the host until asked for:
at n = 1.3e8 the reference needs ~100 GB of CSR, this needs none.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .stencil import StencilMatrix, StencilSpec, spec_cd_3d, spec_cdr_2d, spec_complex_rd

__all__ = ["Problem", "StencilProblem", "build_cdr_2d", "build_cd_3d", "build_complex_rd"]

_SIZE_CAP = 2 ** 62


@dataclass
class Problem:
    """A linear system A x = b with provenance metadata."""

    A: object
    b: np.ndarray
    exact_solution: np.ndarray | None
    label: str
    params: dict = field(default_factory=dict)

    def __post_init__(self):
        if np.shape(self.b) != (self.A.nrows,) or not self.A.is_square:
            raise ValueError("b must match a square A")

    @property
    def n(self) -> int:
        return self.A.nrows


_ONES = object()  # sentinel: the implicit all-ones exact solution


class StencilProblem(Problem):
    """Manufactured-solution problem (x* = 1, b = A 1) on a stencil operator.

    ``b`` and ``exact_solution`` materialise lazily on first host access;
    the solver generates b directly in HBM when the host copy was never
    requested (``rhs_on_device``)."""

    def __init__(self, spec: StencilSpec):  # noqa: D107 - dataclass fields are properties here
        self.spec = spec
        self.A = StencilMatrix(spec)
        self.label = "crd3d" if (spec.family == "crd" and spec.ndim == 3) else spec.family
        self.params = dict(spec.params)
        self._b = None
        self._exact = _ONES  # implicit x* = 1 (problems.py:42-45) until set; None means "no exact solution"

    @property
    def b(self) -> np.ndarray:
        if self._b is None:
            from .device import rhs_ones

            self._b = rhs_ones(self.spec)
        return self._b

    @b.setter
    def b(self, value):
        self._b = np.asarray(value, dtype=np.float64)

    @property
    def exact_solution(self) -> np.ndarray | None:
        if self._exact is _ONES:
            self._exact = np.ones(self.spec.n)
        return self._exact

    @exact_solution.setter
    def exact_solution(self, value):
        self._exact = value

    @property
    def rhs_on_device(self) -> bool:
        """True while b has not been pulled to the host."""
        return self._b is None

    @property
    def exact_is_ones(self) -> bool:
        """x* is still the implicit all-ones vector (never materialised)."""
        return self._exact is _ONES

    def __repr__(self):
        return f"StencilProblem({self.label}, n={self.n}, params={self.params})"

    def __eq__(self, other):
        return self is other

    __hash__ = object.__hash__


def build_cdr_2d(n_g: int, r: float = 1.0) -> StencilProblem:
    """2-D convection-diffusion-reaction, n = n_g^2 (problems.py:48-66)."""
    if n_g < 2:
        raise ValueError("n_g must be >= 2")
    return StencilProblem(spec_cdr_2d(int(n_g), float(r)))


def build_cd_3d(n_g: int) -> StencilProblem:
    """3-D convection-diffusion, n = n_g^3 (problems.py:69-93)."""
    if n_g < 2:
        raise ValueError("n_g must be >= 2")
    if n_g ** 3 > _SIZE_CAP:
        raise ValueError("n_g**3 exceeds the size guard")
    return StencilProblem(spec_cd_3d(int(n_g)))


def build_complex_rd(n_g: int, s: float = 1.0e4, seed: int = 0,
                     laplacian_scaling: str = "nu_over_h2") -> StencilProblem:
    """Complex reaction-diffusion in real block form, n = 2 n_g^2
    (problems.py:96-120)."""
    if n_g < 2:
        raise ValueError("n_g must be >= 2")
    if laplacian_scaling not in ("nu_over_h2", "nu"):
        raise ValueError("laplacian_scaling must be 'nu_over_h2' or 'nu'")
    return StencilProblem(spec_complex_rd(int(n_g), float(s), int(seed), laplacian_scaling))


def build_complex_rd_3d(n_g: int, s: float = 1.0e4, seed: int = 0,
                        laplacian_scaling: str = "nu_over_h2") -> StencilProblem:
    """3-D complex reaction-diffusion, n = 2 n_g^3 (BASELINE config 5; the
    reference's 2-D recipe, REF/problems.py:96-120, with the 7-point
    Laplacian -- SURVEY D1)."""
    if n_g < 2:
        raise ValueError("n_g must be >= 2")
    if laplacian_scaling not in ("nu_over_h2", "nu"):
        raise ValueError("laplacian_scaling must be 'nu_over_h2' or 'nu'")
    if 2 * n_g ** 3 > _SIZE_CAP:
        raise ValueError("n_g**3 exceeds the size guard")
    return StencilProblem(spec_complex_rd(int(n_g), float(s), int(seed), laplacian_scaling, 3))
