"""GPR alpha-selection fixtures from the UNMODIFIED reference
(REF/alphaselect.py:126-266, REF/analysis.py:106-134, REF/cli.py:233-261):

  * condition_estimate of the HSS H and S (the tau-gate factors) on small
    cdr2d / cd3d / crd instances (dense SVD below the 2048 cap);
  * gpr_fit / gpr_predict on the reference tests' line data set;
  * the train-alpha flow (grid_search_alpha per training size, gpr_fit on
    (log n_g, log2 1/u_s) -> log alpha) for cd3d at u_s = fp32, n_g in
    {4, 6, 8}, and select_alpha at n_g = 10 (gate and probe modes).

    PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_gpr_golden.py   ->  tests/golden/gpr.json
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from gadimp import (AlphaSelectConfig, GadiConfig, build_cd_3d, build_cdr_2d, build_complex_rd,  # noqa: E402
                    condition_estimate, gpr_fit, gpr_predict, grid_search_alpha, make_features,
                    make_hss_splitting, predict_alpha, select_alpha)

out = {"cond": []}
for fam, ng, kw in (("cdr2d", 6, {}), ("cdr2d", 12, {"r": 0.3}), ("cdr2d", 9, {"r": 0.0}), ("cd3d", 5, {}),
                    ("cd3d", 8, {}), ("cd3d", 12, {}), ("crd", 8, {}), ("crd", 12, {"s": 300.0})):
    p = {"cdr2d": build_cdr_2d, "cd3d": build_cd_3d, "crd": build_complex_rd}[fam](ng, **kw)
    for alpha in (0.1, 1.0, 10.0):
        s = make_hss_splitting(p.A, alpha, "fp64")
        out["cond"].append({"family": fam, "n_g": ng, "kw": kw, "alpha": alpha,
                            "kappa_H": condition_estimate(s.H), "kappa_S": condition_estimate(s.S)})

x = np.linspace(0.0, 3.0, 8).reshape(-1, 1)
y = 0.5 * x[:, 0] + 1.0
m = gpr_fit(x, y)
q = [0.0, 0.37, 1.234, 2.9, 3.5, 10.0]
out["line"] = {"x": x.tolist(), "y": y.tolist(), "model": m.to_dict(),
               "queries": q, "pred": [list(gpr_predict(m, np.array([v]))) for v in q]}

cands = np.logspace(-2, 2, 13)
feats, targets, per_size = [], [], []
for ng in (4, 6, 8):
    p = build_cd_3d(ng)
    cfg = GadiConfig(alpha=1.0, u_s="fp32", outer_tol=1e-8, inner_tol=1e-4, outer_maxit=500)
    best, counts = grid_search_alpha(p, cands, cfg)
    feats.append(make_features(ng, "fp32"))
    targets.append(np.log(best))
    per_size.append({"n_g": ng, "best": best, "counts": counts})
    print("n_g", ng, "best", best, flush=True)
model = gpr_fit(np.array(feats), np.array(targets))
p10 = build_cd_3d(10)
cfg10 = GadiConfig(alpha=1.0, u_s="fp32", outer_tol=1e-8, inner_tol=1e-4, outer_maxit=500)
a_gate, tr_gate = select_alpha(p10, model, AlphaSelectConfig(), cfg10)
a_probe, tr_probe = select_alpha(p10, model, AlphaSelectConfig(check_condition=False), cfg10)
# a tight gate that forces escalation (bf16; tau below u_s = 2^-8 can never pass)
a_esc, tr_esc = select_alpha(p10, model, AlphaSelectConfig(tau=0.02), GadiConfig(alpha=1.0, u_s="bf16"),
                             features=make_features(10, "fp32"))
out["train"] = {"family": "cd3d", "u_s": "fp32", "candidates": cands.tolist(), "sizes": per_size,
                "model": model.to_dict(), "predict_10": predict_alpha(model, make_features(10, "fp32")),
                "predict_64": predict_alpha(model, make_features(64, "fp32")),
                "select_gate": {"alpha": a_gate, "trace": tr_gate},
                "select_probe": {"alpha": a_probe, "trace": tr_probe},
                "select_escalate": {"alpha": a_esc, "trace": tr_esc}}
(Path(__file__).resolve().parent / "gpr.json").write_text(json.dumps(out, default=float))
print("gate", a_gate, len(tr_gate), "probe", a_probe, "escalate", a_esc, len(tr_esc))
