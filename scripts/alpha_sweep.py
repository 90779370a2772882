"""Grid search of (alpha, inner_tol) for the benchmark workload on the GPU
(the paper hand-picks alpha for 3-D bf16; SURVEY §8d
config 4: "GPU grid search").  Prints one JSON line per setting: device
solve time, outer / inner counts, final relres and berr."""
import json
import sys
import time

import paper_2512_21164_b200 as g

ng = int(sys.argv[1]) if len(sys.argv) > 1 else 512
us = sys.argv[2] if len(sys.argv) > 2 else "bf16"
alphas = [float(a) for a in (sys.argv[3] if len(sys.argv) > 3 else "0.00625,0.0125,0.025,0.05").split(",")]
tols = [float(t) for t in (sys.argv[4] if len(sys.argv) > 4 else "1e-3").split(",")]
outer_tol = float(sys.argv[5]) if len(sys.argv) > 5 else 1e-12
omegas = [float(w) for w in (sys.argv[6] if len(sys.argv) > 6 else "1.0").split(",")]
maxit = int(sys.argv[7]) if len(sys.argv) > 7 else 2000


class T:
    def on_start(self, ctx):
        ctx.timer_start()

    def on_end(self, ctx):
        self.ms = ctx.timer_stop()


for a, it, om in [(a, it, om) for a in alphas for it in tols for om in omegas]:
        cfg = g.GadiConfig(alpha=a, u_s=us, outer_tol=outer_tol, inner_tol=it, outer_maxit=maxit,
                           strict_model=False, omega=om)
        t = T()
        w0 = time.perf_counter()
        rep = g.gadi_solve(g.build_cd_3d(ng), cfg=cfg, return_x=False, hooks=t, rounding="storage")
        print(json.dumps({"ng": ng, "us": us, "alpha": a, "inner_tol": it, "omega": om, "s": round(t.ms / 1e3, 3),
                          "wall": round(time.perf_counter() - w0, 2), "status": rep.status,
                          "outer": rep.iterations,
                          "inner_h": sum(h.inner_h_iterations for h in rep.history),
                          "inner_s": sum(h.inner_s_iterations for h in rep.history),
                          "relres": rep.history[-1].relative_residual,
                          "berr": rep.history[-1].backward_error}), flush=True)
