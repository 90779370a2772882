"""GPU-backed alpha search.

``grid_search_alpha`` is the reference's selection rule
(REF/alphaselect.py:126-145): one solve per candidate alpha, keep the
converged candidate with the fewest outer iterations (ties: fewer total inner
iterations, then the smaller alpha).  Every candidate solve is this package's
``gadi_solve`` on the GPU; the device context is reused across candidates of
the same operator only when alpha repeats (the splitting constants depend on
alpha), so each candidate costs one context build plus one solve.

The GPR model / tau-gate of ``select_alpha`` (REF/alphaselect.py:174-266) is
host-side numerical work outside the hot path (SURVEY §2 marks it out of
scope); its probe solves would go through ``gadi_solve`` the same way.
"""

from __future__ import annotations

import dataclasses

from .errors import AllDiverged
from .gadi import GadiConfig, gadi_solve

__all__ = ["grid_search_alpha", "log_grid"]


def log_grid(lo: float, hi: float, points: int = 13) -> list[float]:
    """The CLI's default 13-point log grid (REF/cli.py:239-249)."""
    import numpy as np

    return [float(a) for a in np.logspace(np.log10(lo), np.log10(hi), points)]


def grid_search_alpha(problem, candidates, cfg: GadiConfig, **solve_kw):
    """Return (best_alpha, counts) with counts = [(alpha, status, outer, inner)]
    in ascending alpha, as REF/alphaselect.py:126-145."""
    candidates = [float(c) for c in candidates]
    if not candidates or any(c <= 0 for c in candidates):
        raise ValueError("candidates must be a nonempty list of positive reals")
    results, counts = [], []
    for alpha in sorted(candidates):
        report = gadi_solve(problem, cfg=dataclasses.replace(cfg, alpha=alpha), return_x=False, **solve_kw)
        counts.append((alpha, report.status, report.iterations, report.total_inner_iterations))
        if report.status == "Converged":
            results.append((report.iterations, report.total_inner_iterations, alpha))
    if not results:
        raise AllDiverged("no candidate alpha converged")
    return min(results)[2], counts
