"""Alpha selection on top of the GPU solve.

The reference's pipeline (REF/alphaselect.py, REF/cli.py:233-261):

1. ``grid_search_alpha`` (REF/alphaselect.py:126-145): one solve per candidate
   alpha; the converged candidate with the fewest outer iterations wins (ties:
   fewer total inner iterations, then the smaller alpha).  Every candidate is
   this package's ``gadi_solve`` on the GPU.
2. ``train_alpha`` (the CLI's ``train-alpha``): grid search on small training
   sizes, then ``gpr_fit`` of log(alpha_opt) on the features
   (log n_g, log2(1/u_s) [, family one-hot]) -- a Gaussian process with an RBF
   kernel whose (signal variance, per-feature length scales, noise variance)
   maximise the log marginal likelihood over a fixed grid.
3. ``select_alpha`` (REF/alphaselect.py:233-266): alpha = exp(posterior mean),
   escalated by a factor until the safety gate passes -- either
   kappa(H) kappa(S) u_s < tau (``condition_estimate``: closed-form spectra for
   the stencil families, analysis.py), or a GPU probe solve that neither
   stagnates nor diverges.

The GP algebra is small dense host work; the JSON model format is the
reference's (``GprModel.save`` / ``load`` interoperate with ``gadi-mp``).
"""

from __future__ import annotations

import dataclasses
import json
import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

from .analysis import DENSE_CAP, condition_estimate
from .errors import AllDiverged, EscalationExhausted, IllConditionedGram
from .gadi import GadiConfig, gadi_solve
from .precision import resolve_format
from .splitting import make_hss_splitting

__all__ = ["grid_search_alpha", "log_grid", "make_features", "GprModel", "gpr_fit", "gpr_predict",
           "predict_alpha", "AlphaSelectConfig", "select_alpha", "train_alpha"]

_NOISE_FLOOR = 1.0e-6


def log_grid(lo: float, hi: float, points: int = 13) -> list[float]:
    """The CLI's default 13-point log grid (REF/cli.py:239-249)."""
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


# ---------------------------------------------------------------- Gaussian process
def make_features(n_g: int, u_s, family: str | None = None, families: tuple = ()) -> np.ndarray:
    """(log n_g, log2(1/u_s)) plus a one-hot of ``family`` over ``families``."""
    u = resolve_format(u_s).unit_roundoff
    onehot = [1.0 if f == family else 0.0 for f in families]
    return np.array([math.log(n_g), math.log2(1.0 / u)] + onehot)


def _rbf(xa, xb, sf2, ls):
    z = (np.asarray(xa)[:, None, :] - np.asarray(xb)[None, :, :]) / ls
    return sf2 * np.exp(-0.5 * np.einsum("ijk,ijk->ij", z, z))


@dataclass
class GprModel:
    """GP posterior on log(alpha); the reference's JSON layout."""

    training_inputs: np.ndarray
    training_targets: np.ndarray
    signal_variance: float
    length_scales: np.ndarray
    noise_variance: float
    families: tuple = ()
    _L: np.ndarray | None = field(default=None, repr=False, compare=False)
    _w: np.ndarray | None = field(default=None, repr=False, compare=False)

    def _kernel(self, xa, xb):
        return _rbf(xa, xb, self.signal_variance, self.length_scales)

    def _factor(self):
        """Cholesky factor L of K + sn2 I and the weights K^-1 y."""
        if self._L is None:
            k = self._kernel(self.training_inputs, self.training_inputs)
            k[np.diag_indices_from(k)] += self.noise_variance
            self._L = np.linalg.cholesky(k)
            z = scipy.linalg.solve_triangular(self._L, self.training_targets, lower=True)
            self._w = scipy.linalg.solve_triangular(self._L.T, z, lower=False)
        return self._L

    def to_dict(self) -> dict:
        return {"training_inputs": np.asarray(self.training_inputs).tolist(),
                "training_targets": np.asarray(self.training_targets).tolist(),
                "signal_variance": self.signal_variance,
                "length_scales": np.asarray(self.length_scales).tolist(),
                "noise_variance": self.noise_variance, "families": list(self.families)}

    @classmethod
    def from_dict(cls, d: dict) -> "GprModel":
        return cls(np.asarray(d["training_inputs"], dtype=float), np.asarray(d["training_targets"], dtype=float),
                   float(d["signal_variance"]), np.asarray(d["length_scales"], dtype=float),
                   float(d["noise_variance"]), tuple(d.get("families", ())))

    def save(self, path) -> None:
        with open(path, "w") as f:
            json.dump(self.to_dict(), f, indent=2)

    @classmethod
    def load(cls, path) -> "GprModel":
        with open(path) as f:
            return cls.from_dict(json.load(f))


def _lml(x, y, sf2, ls, sn2) -> float:
    """log p(y | x) = -y^T K^-1 y / 2 - sum log diag L - m/2 log 2 pi."""
    k = _rbf(x, x, sf2, ls)
    k[np.diag_indices_from(k)] += sn2
    try:
        L = np.linalg.cholesky(k)
    except np.linalg.LinAlgError:
        return -np.inf
    z = scipy.linalg.solve_triangular(L, y, lower=True)
    return float(-0.5 * z @ z - np.sum(np.log(np.diag(L))) - 0.5 * y.size * math.log(2.0 * math.pi))


def _hyper_grid(x):
    """Signal variance x length-scale multiple (of each feature's span) x noise
    (REF/alphaselect.py:163-171)."""
    span = np.ptp(x, axis=0)
    span = np.where(span > 0, span, 1.0)
    return [(sf2, mult * span, sn2) for sf2 in (0.25, 1.0, 4.0, 16.0) for mult in (0.25, 0.5, 1.0, 2.0, 4.0)
            for sn2 in (_NOISE_FLOOR, 1.0e-4, 1.0e-2)]


def gpr_fit(x, y, hyper_grid=None, families: tuple = ()) -> GprModel:
    """Maximum-likelihood hyperparameters over the grid (first maximum wins);
    if no candidate's Gram matrix factorises, retry with noise >= 1e-2."""
    x = np.atleast_2d(np.asarray(x, dtype=float))
    y = np.asarray(y, dtype=float)
    if x.shape[0] < 2:
        raise ValueError("gpr_fit needs at least two training points")
    if hyper_grid is None:
        grid = _hyper_grid(x)
    else:
        grid = [(h["signal_variance"], h["length_scales"], h["noise_variance"]) for h in hyper_grid]
    grid = [(float(a), np.broadcast_to(np.asarray(b, dtype=float), (x.shape[1],)).copy(), float(c))
            for a, b, c in grid]
    for attempt in (grid, [(a, b, max(c, 1.0e-2)) for a, b, c in grid]):
        scores = [_lml(x, y, *h) for h in attempt]
        best = int(np.argmax(scores))
        if np.isfinite(scores[best]):
            sf2, ls, sn2 = attempt[best]
            model = GprModel(x, y, sf2, ls, max(sn2, _NOISE_FLOOR), tuple(families))
            model._factor()
            return model
    raise IllConditionedGram("no hyperparameter candidate gives a positive definite Gram matrix")


def gpr_predict(model: GprModel, x) -> tuple[float, float]:
    """Posterior mean and variance at one feature vector."""
    x = np.atleast_2d(np.asarray(x, dtype=float))
    L = model._factor()
    ks = model._kernel(model.training_inputs, x)[:, 0]
    mean = float(ks @ model._w)
    v = scipy.linalg.solve_triangular(L, ks, lower=True)
    return mean, max(float(model.signal_variance - v @ v), 0.0)


def predict_alpha(model: GprModel, features) -> float:
    return math.exp(gpr_predict(model, features)[0])


# ---------------------------------------------------------------- selection
@dataclass
class AlphaSelectConfig:
    tau: float = 0.01
    escalation_factor: float = 2.0
    max_escalations: int = 20
    candidate_grid: np.ndarray = field(default_factory=lambda: np.logspace(-2, 2, 13))
    check_condition: bool = True
    dense_cap: int = DENSE_CAP

    def __post_init__(self):
        if not 0.0 < self.tau < 1.0:
            raise ValueError(f"tau must lie in (0, 1), got {self.tau}")
        if not self.escalation_factor > 1.0:
            raise ValueError(f"escalation_factor must exceed 1, got {self.escalation_factor}")


def select_alpha(problem, model: GprModel, sel_cfg: AlphaSelectConfig, cfg: GadiConfig, features=None, **solve_kw):
    """GP-predicted alpha, multiplied by ``escalation_factor`` until the gate
    passes (REF/alphaselect.py:233-266).  Returns (alpha, trace)."""
    if features is None:
        features = make_features(problem.params.get("n_g", problem.A.nrows), cfg.u_s, problem.label,
                                 model.families)
    alpha = predict_alpha(model, features)
    u_s = resolve_format(cfg.u_s).unit_roundoff
    trace = []
    for step in range(sel_cfg.max_escalations + 1):
        if sel_cfg.check_condition:
            sp = make_hss_splitting(problem.A, alpha, cfg.u_s)
            gate = condition_estimate(sp.H, sel_cfg.dense_cap) * condition_estimate(sp.S, sel_cfg.dense_cap) * u_s
            ok = gate < sel_cfg.tau
            trace.append({"step": step, "alpha": alpha, "gate": gate, "passed": ok})
        else:
            probe = gadi_solve(problem, cfg=dataclasses.replace(cfg, alpha=alpha), return_x=False, **solve_kw)
            ok = probe.status not in ("Stagnated", "Diverged")
            trace.append({"step": step, "alpha": alpha, "probe_status": probe.status, "passed": ok})
        if ok:
            return alpha, trace
        alpha *= sel_cfg.escalation_factor
    raise EscalationExhausted(f"the gate still fails after {sel_cfg.max_escalations} escalations")


def train_alpha(build, sizes, u_s="fp64", candidates=None, outer_tol: float = 1e-8, inner_tol: float = 1e-4,
                outer_maxit: int = 500, **solve_kw):
    """The CLI's train-alpha (REF/cli.py:233-261) on the GPU: grid-search the
    best alpha per training size, fit the GP.  Returns (model, per-size
    results)."""
    candidates = np.logspace(-2, 2, 13) if candidates is None else np.asarray(candidates, dtype=float)
    feats, targets, per = [], [], []
    for n_g in sizes:
        cfg = GadiConfig(alpha=1.0, u_s=u_s, outer_tol=outer_tol, inner_tol=inner_tol, outer_maxit=outer_maxit)
        best, counts = grid_search_alpha(build(n_g), candidates, cfg, **solve_kw)
        feats.append(make_features(n_g, u_s))
        targets.append(math.log(best))
        per.append({"n_g": n_g, "best": best, "counts": counts})
    return gpr_fit(np.array(feats), np.array(targets)), per
