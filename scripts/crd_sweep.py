"""Config 5 exploration: crd 2-D (complex reaction-diffusion, s = 1e4) outer
traces over (alpha, inner_tol) at one precision.
python scripts/crd_sweep.py NG US MAXIT alpha,tol ..."""
import json
import sys

import paper_2512_21164_b200 as g


class T:
    def on_start(self, ctx):
        ctx.timer_start()

    def on_end(self, ctx):
        self.ms = ctx.timer_stop()


ng, us, maxit = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
for a in sys.argv[4:]:
    alpha, tol = (float(v) for v in a.split(","))
    cfg = g.GadiConfig(alpha=alpha, u_s=us, outer_tol=1e-6, inner_tol=tol, outer_maxit=maxit, strict_model=False)
    t = T()
    rep = g.gadi_solve(g.build_complex_rd(ng), cfg=cfg, rounding="storage", return_x=False, hooks=t)
    print(json.dumps({"n_g": ng, "u_s": us, "alpha": alpha, "inner_tol": tol, "status": rep.status,
                      "outer": rep.iterations, "s": round(t.ms / 1e3, 3),
                      "relres": [h.relative_residual for h in rep.history],
                      "inner_h": [h.inner_h_iterations for h in rep.history],
                      "inner_s": [h.inner_s_iterations for h in rep.history]}), flush=True)
