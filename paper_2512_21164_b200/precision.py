"""Precision formats and the rounding contract of the solver.

The reference emulates every format on top of float64 (gadimp/precision.py).
Here the formats are native device types (bf16 / fp16 / fp32 / fp64 storage
in HBM); this module keeps the host-side vocabulary -- format table,
validation, and RNE quantisation of *scalars and coefficient sets* (the
splitting constants, (2 - omega) alpha) -- with the reference's semantics:
round-to-nearest-even, overflow to signed infinity (or RangeOverflow when
strict), subnormals kept unless flushed (precision.py:136-165).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import RangeOverflow

__all__ = ["PrecisionFormat", "FORMATS", "resolve_format", "unit_roundoff", "quantize"]


@dataclass(frozen=True)
class PrecisionFormat:
    """Binary floating-point format; ``significand_bits`` counts the hidden bit."""

    name: str
    significand_bits: int
    exponent_bits: int
    compensated: bool = field(default=False)

    def __post_init__(self):
        if self.significand_bits < 2 or self.exponent_bits < 2:
            raise ValueError("need significand_bits >= 2 and exponent_bits >= 2")

    @property
    def unit_roundoff(self) -> float:
        return 2.0 ** (-self.significand_bits)

    @property
    def max_exponent(self) -> int:
        return 2 ** (self.exponent_bits - 1) - 1

    @property
    def min_exponent(self) -> int:
        return 1 - self.max_exponent

    @property
    def max_finite(self) -> float:
        return (2.0 - 2.0 ** (1 - self.significand_bits)) * 2.0 ** self.max_exponent

    @property
    def min_normal(self) -> float:
        return 2.0 ** self.min_exponent

    def __str__(self):
        return self.name


FORMATS = {
    "bf16": PrecisionFormat("bf16", 8, 8),
    "fp16": PrecisionFormat("fp16", 11, 5),
    "fp32": PrecisionFormat("fp32", 24, 8),
    "fp64": PrecisionFormat("fp64", 53, 11),
    "fp64x2": PrecisionFormat("fp64x2", 106, 11, compensated=True),
}


def resolve_format(fmt) -> PrecisionFormat:
    if isinstance(fmt, PrecisionFormat):
        return fmt
    key = str(fmt).lower()
    if key not in FORMATS:
        raise ValueError(f"unknown precision format {fmt!r}; expected one of {sorted(FORMATS)}")
    return FORMATS[key]


def unit_roundoff(fmt) -> float:
    return resolve_format(fmt).unit_roundoff


def _bf16_rne(a: np.ndarray) -> np.ndarray:
    # f64 -> f32 (RNE) then RNE to the top 16 bits; the double rounding is
    # innocuous because 24 >= 2*8 + 2.
    f = a.astype(np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    keep = (u >> np.uint64(16)) & np.uint64(1)
    u = ((u + np.uint64(0x7FFF) + keep) >> np.uint64(16)) << np.uint64(16)
    out = (u & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32).astype(np.float64)
    return np.where(np.isnan(a), a, out)


def _generic_rne(a: np.ndarray, fmt: PrecisionFormat) -> np.ndarray:
    _, e = np.frexp(a)
    step = np.maximum(e - 1, fmt.min_exponent) - (fmt.significand_bits - 1)
    q = np.ldexp(np.rint(np.ldexp(a, -step)), step)
    return np.where(np.abs(q) > fmt.max_finite, np.copysign(np.inf, a), q)


def quantize(x, fmt, flush_subnormals: bool = False, strict: bool = False):
    """RNE image of ``x`` in ``fmt`` (scalars and arrays)."""
    fmt = resolve_format(fmt)
    is_scalar = np.isscalar(x) or (isinstance(x, np.ndarray) and x.ndim == 0)
    a = np.asarray(x, dtype=np.float64)
    with np.errstate(over="ignore"):
        if fmt.significand_bits >= 53:
            out = a
        elif fmt.name == "fp32":
            out = a.astype(np.float32).astype(np.float64)
        elif fmt.name == "fp16":
            out = a.astype(np.float16).astype(np.float64)
        elif fmt.name == "bf16":
            out = _bf16_rne(a)
        else:
            out = _generic_rne(a, fmt)
    if strict and np.any(np.isinf(out) & np.isfinite(a)):
        raise RangeOverflow(f"value overflows {fmt.name} range")
    if flush_subnormals and fmt.significand_bits < 53:
        tiny = (np.abs(out) < fmt.min_normal) & (out != 0.0)
        if np.any(tiny):
            out = np.where(tiny, np.copysign(0.0, out), out)
    return float(out) if is_scalar else out
