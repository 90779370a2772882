"""Secondary BASELINE.json configs on one B200 (the bench line is config 4):
device-timed solves with a small alpha grid per config, reporting time,
counts, final relres / berr.  Prints one JSON line per solve."""
import json
import sys
import time

import paper_2512_21164_b200 as g


class T:
    def on_start(self, ctx):
        ctx.timer_start()

    def on_end(self, ctx):
        self.ms = ctx.timer_stop()


def run(tag, build, ng, us, alpha, outer_tol, inner_tol=1e-4, maxit=2000):
    cfg = g.GadiConfig(alpha=alpha, u_s=us, outer_tol=outer_tol, inner_tol=inner_tol, outer_maxit=maxit,
                       strict_model=False)
    build(ng)  # spec construction outside the timer
    g.gadi_solve(build(ng), cfg=cfg, return_x=False, reuse_context=True, rounding="storage")  # warm-up
    t = T()
    w0 = time.perf_counter()
    rep = g.gadi_solve(build(ng), cfg=cfg, return_x=False, hooks=t, rounding="storage")
    out = {"config": tag, "n_g": ng, "u_s": us, "alpha": alpha, "outer_tol": outer_tol, "inner_tol": inner_tol,
           "device_s": round(t.ms / 1e3, 4), "wall_s": round(time.perf_counter() - w0, 3), "status": rep.status,
           "outer": rep.iterations, "inner_h": sum(h.inner_h_iterations for h in rep.history),
           "inner_s": sum(h.inner_s_iterations for h in rep.history),
           "relres": rep.history[-1].relative_residual, "berr": rep.history[-1].backward_error}
    print(json.dumps(out), flush=True)
    return out


which = sys.argv[1:] or ["1", "2", "3", "5"]
if "1" in which:  # cdr2d 256^2, fp32 inner, alpha = 1 (the reference's own test problem, 209 outer)
    for us in ("fp32", "fp64", "bf16"):
        run("cfg1", g.build_cdr_2d, 256, us, 1.0, 1e-10)
if "2" in which:  # cdr2d 4096^2, bf16 vs fp64 inner, relres 1e-10
    for a in (0.5, 1.0, 2.0):
        for us in ("bf16", "fp64"):
            run("cfg2", g.build_cdr_2d, 4096, us, a, 1e-10, 1e-4, 4000)
if "3" in which:  # cd3d 256^3, fp32 inner, relres 1e-6
    for a in (0.025, 0.05, 0.1):
        run("cfg3", g.build_cd_3d, 256, "fp32", a, 1e-6, 1e-3, 2000)
if "5" in which:  # crd 2-D n_g = 8192 (n = 1.34e8), precision sweep, relres 1e-6;
    # every S-solve runs up to 10^4 CGNR iterations here, so only 3 outer
    # steps are timed (per-step cost; the full solve is the 8-GPU config)
    for us in ("bf16", "fp32", "fp64"):
        run("cfg5_3steps", g.build_complex_rd, 8192, us, 10.0, 1e-6, 1e-4, 3)
