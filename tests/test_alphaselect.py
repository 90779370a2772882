"""GPR alpha selection (paper_2512_21164_b200.alphaselect) against the
unmodified reference's outputs (tests/golden/gpr.json, make_gpr_golden.py).

CPU tests: the closed-form condition numbers of the HSS operators, the GP fit
/ posterior, the gate-mode selection (host-only work).  GPU tests: the
train-alpha flow and probe-mode selection, whose solves run on the GPU."""

import json
import math
from pathlib import Path

import numpy as np
import pytest

import paper_2512_21164_b200 as g
from paper_2512_21164_b200 import alphaselect as A
from paper_2512_21164_b200.analysis import condition_estimate

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "gpr.json").read_text())
BUILD = {"cdr2d": g.build_cdr_2d, "cd3d": g.build_cd_3d, "crd": g.build_complex_rd}


def test_condition_numbers_match_reference():
    for c in GOLD["cond"]:
        p = BUILD[c["family"]](c["n_g"], **c["kw"])
        s = g.make_hss_splitting(p.A, c["alpha"], "fp64")
        assert condition_estimate(s.H) == pytest.approx(c["kappa_H"], rel=1e-12), c
        assert condition_estimate(s.S) == pytest.approx(c["kappa_S"], rel=1e-12), c


def test_condition_numbers_numeric_route():
    """Operators without a closed form (A itself, a CSR) take the dense SVD
    route below the cap: the closed form agrees with it on H and S."""
    p = g.build_cd_3d(6)
    s = g.make_hss_splitting(p.A, 0.3, "fp64")
    for op in (s.H, s.S):
        dense = np.linalg.svd(op.to_scipy().toarray(), compute_uv=False)
        assert condition_estimate(op) == pytest.approx(dense[0] / dense[-1], rel=1e-12)
    a = np.linalg.svd(p.A.to_scipy().toarray(), compute_uv=False)
    assert condition_estimate(p.A) == pytest.approx(a[0] / a[-1], rel=1e-12)


def test_gp_fit_and_posterior_match_reference():
    d = GOLD["line"]
    m = A.gpr_fit(np.array(d["x"]), np.array(d["y"]))
    ref = d["model"]
    assert m.signal_variance == ref["signal_variance"] and m.noise_variance == ref["noise_variance"]
    assert np.allclose(m.length_scales, ref["length_scales"], rtol=0, atol=0)
    for q, (mean, var) in zip(d["queries"], d["pred"]):
        mm, vv = A.gpr_predict(m, np.array([q]))
        assert mm == pytest.approx(mean, rel=1e-10, abs=1e-12)
        assert vv == pytest.approx(var, rel=1e-8, abs=1e-12)
    # JSON round trip in the reference's layout
    back = A.GprModel.from_dict(json.loads(json.dumps(m.to_dict())))
    assert A.gpr_predict(back, np.array([0.7])) == A.gpr_predict(m, np.array([0.7]))
    with pytest.raises(ValueError):
        A.gpr_fit(np.array([[1.0]]), np.array([0.0]))


def _trained_model():
    t = GOLD["train"]
    feats = [A.make_features(s["n_g"], t["u_s"]) for s in t["sizes"]]
    return A.gpr_fit(np.array(feats), np.log([s["best"] for s in t["sizes"]]))


def test_trained_model_and_gate_selection_match_reference():
    t = GOLD["train"]
    m = _trained_model()
    assert m.signal_variance == t["model"]["signal_variance"]
    assert np.array_equal(m.length_scales, np.array(t["model"]["length_scales"]))
    assert A.predict_alpha(m, A.make_features(10, "fp32")) == pytest.approx(t["predict_10"], rel=1e-10)
    assert A.predict_alpha(m, A.make_features(64, "fp32")) == pytest.approx(t["predict_64"], rel=1e-10)
    p = g.build_cd_3d(10)
    for key, sel, cfg, feats in (
            ("select_gate", A.AlphaSelectConfig(), g.GadiConfig(alpha=1.0, u_s="fp32"), None),
            ("select_escalate", A.AlphaSelectConfig(tau=0.02), g.GadiConfig(alpha=1.0, u_s="bf16"),
             A.make_features(10, "fp32"))):
        alpha, trace = A.select_alpha(p, m, sel, cfg, features=feats)
        ref = t[key]
        assert alpha == pytest.approx(ref["alpha"], rel=1e-10)
        assert [s["passed"] for s in trace] == [s["passed"] for s in ref["trace"]]
        for s, r in zip(trace, ref["trace"]):
            assert s["gate"] == pytest.approx(r["gate"], rel=1e-10)
    with pytest.raises(g.errors.EscalationExhausted):  # tau below u_s can never pass
        A.select_alpha(p, m, A.AlphaSelectConfig(tau=1e-3, max_escalations=3), g.GadiConfig(alpha=1.0, u_s="bf16"),
                       features=A.make_features(10, "fp32"))


@pytest.mark.gpu
def test_train_alpha_on_gpu_matches_reference(gpu):
    t = GOLD["train"]
    model, per = A.train_alpha(g.build_cd_3d, [s["n_g"] for s in t["sizes"]], t["u_s"], t["candidates"])
    for mine, ref in zip(per, t["sizes"]):
        assert mine["best"] == ref["best"]
        assert [tuple(c) for c in mine["counts"]] == [tuple(c) for c in ref["counts"]]
    assert A.predict_alpha(model, A.make_features(10, "fp32")) == pytest.approx(t["predict_10"], rel=1e-10)


@pytest.mark.gpu
def test_probe_selection_on_gpu_matches_reference(gpu):
    t = GOLD["train"]
    m = _trained_model()
    cfg = g.GadiConfig(alpha=1.0, u_s="fp32", outer_tol=1e-8, inner_tol=1e-4, outer_maxit=500)
    alpha, trace = A.select_alpha(g.build_cd_3d(10), m, A.AlphaSelectConfig(check_condition=False), cfg)
    ref = t["select_probe"]
    assert alpha == pytest.approx(ref["alpha"], rel=1e-10)
    assert [s["probe_status"] for s in trace] == [s["probe_status"] for s in ref["trace"]]
    assert math.isfinite(alpha)
