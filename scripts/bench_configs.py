"""BASELINE.json configs 1, 2, 3, 5 on one B200 (the bench line is config 4):
device-timed solves, one JSON line per solve, plus the reference CLI's bench
outputs (summary.csv, per-run trace JSONL; REF/cli.py:320-342 via report.py)
under gpurun_out/configs_report/.

    python scripts/bench_configs.py [1] [2] [3] [5] [5sweep]

Config 3 takes its alpha from the GPR pipeline as the reference's CLI does
(train-alpha on n_g in {8, 16, 32, 64} at u_s = fp32, then select_alpha with
the kappa(H) kappa(S) u_s < tau gate; REF/cli.py:233-261,
REF/alphaselect.py:233-266), the training grid searches running on the GPU.
"""
import json
import sys
import time
from pathlib import Path

import paper_2512_21164_b200 as g
from paper_2512_21164_b200 import alphaselect as A
from paper_2512_21164_b200 import report

OUT = Path(__file__).resolve().parent.parent / "gpurun_out" / "configs_report"


class T:
    def on_start(self, ctx):
        ctx.timer_start()

    def on_end(self, ctx):
        self.ms = ctx.timer_stop()


def run(tag, build, ng, us, alpha, outer_tol, inner_tol=1e-4, maxit=2000, rounding="storage", extra=None):
    cfg = g.GadiConfig(alpha=alpha, u_s=us, outer_tol=outer_tol, inner_tol=inner_tol, outer_maxit=maxit,
                       strict_model=False)
    build(ng)  # spec construction outside the timer
    g.gadi_solve(build(min(ng, 64)), cfg=cfg, return_x=False, rounding=rounding)  # kernels loaded
    t = T()
    w0 = time.perf_counter()
    p = build(ng)
    rep = g.gadi_solve(p, cfg=cfg, return_x=False, hooks=t, rounding=rounding)
    wall = time.perf_counter() - w0
    out = {"config": tag, "n_g": ng, "u_s": us, "alpha": alpha, "outer_tol": outer_tol, "inner_tol": inner_tol,
           "rounding": rounding, "device_s": round(t.ms / 1e3, 4), "wall_s": round(wall, 3), "status": rep.status,
           "outer": rep.iterations, "inner_h": sum(h.inner_h_iterations for h in rep.history),
           "inner_s": sum(h.inner_s_iterations for h in rep.history),
           "relres": rep.history[-1].relative_residual, "berr": rep.history[-1].backward_error, **(extra or {})}
    print(json.dumps(out), flush=True)
    OUT.mkdir(parents=True, exist_ok=True)
    report.append_summary(OUT / "summary.csv", p, cfg, rep, t.ms / 1e3, 0,
                          gpu={"n_gpus": 1, "device_time_s": t.ms / 1e3, "achieved_gbs": None, "roofline_frac": None})
    report.write_trace(OUT / f"{tag}_{p.label}_ng{ng}_{us}_a{alpha:.4g}_trace.jsonl", rep)
    return out


which = sys.argv[1:] or ["1", "2", "3", "5"]
if "1" in which:  # cdr2d 256^2, fp32 inner, alpha = 1 (the reference's own test problem, 209 outer)
    for us in ("fp32", "fp64", "bf16"):
        run("cfg1", g.build_cdr_2d, 256, us, 1.0, 1e-10)
if "2" in which:  # cdr2d 4096^2, bf16 vs fp64 inner, relres 1e-10
    for a in (0.5, 1.0, 2.0):
        for us in ("bf16", "fp64"):
            run("cfg2", g.build_cdr_2d, 4096, us, a, 1e-10, 1e-4, 4000)
if "3" in which:  # cd3d 256^3, fp32 inner, relres 1e-6, GPR-initialised alpha
    t0 = time.perf_counter()
    model, per = A.train_alpha(g.build_cd_3d, [8, 16, 32, 64], "fp32")
    p = g.build_cd_3d(256)
    cfg = g.GadiConfig(alpha=1.0, u_s="fp32", outer_tol=1e-6, inner_tol=1e-3, outer_maxit=2000)
    alpha, trace = A.select_alpha(p, model, A.AlphaSelectConfig(), cfg)
    OUT.mkdir(parents=True, exist_ok=True)
    model.save(OUT / "cfg3_gpr_model.json")
    gpr = {"training": [{"n_g": s["n_g"], "best": s["best"]} for s in per],
           "predicted": A.predict_alpha(model, A.make_features(256, "fp32")), "gate_trace": trace,
           "train_select_s": round(time.perf_counter() - t0, 2)}
    run("cfg3_gpr", g.build_cd_3d, 256, "fp32", alpha, 1e-6, 1e-3, 2000, extra={"gpr": gpr})
    for a in (0.025, 0.05):
        run("cfg3", g.build_cd_3d, 256, "fp32", a, 1e-6, 1e-3, 2000)
if "5" in which:  # crd 2-D n_g = 8192 (n = 1.34e8), precision sweep, relres 1e-6;
    # alpha = 1, inner_tol 1e-2 from the GPU sweeps (profiles/crd_sweep_r2_*.jsonl: alpha = 10 -- the
    # reference tests' value at n_g <= 32 -- leaves the CGNR at maxit every step and stalls near 2e-6)
    for us in ("bf16", "fp32", "fp64"):
        run("cfg5", g.build_complex_rd, 8192, us, 1.0, 1e-6, 1e-2, 400)
