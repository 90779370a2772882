"""Config 5's 3-D extension at the largest grid one B200 holds: crd 3-D
(n = 2 n_g^3), a few outer steps (per-step cost and memory), and the 2-D
precision sweep's alpha.  python scripts/crd3d_large.py NG US STEPS"""
import json
import sys
import time

import paper_2512_21164_b200 as g


class T:
    def on_start(self, ctx):
        ctx.timer_start()

    def on_end(self, ctx):
        self.ms = ctx.timer_stop()


ng, us, steps = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
t0 = time.perf_counter()
p = g.build_complex_rd_3d(ng)
t_build = time.perf_counter() - t0
cfg = g.GadiConfig(alpha=1.0, u_s=us, outer_tol=1e-6, inner_tol=1e-2, outer_maxit=steps, strict_model=False)
t = T()
t1 = time.perf_counter()
rep = g.gadi_solve(p, cfg=cfg, rounding="storage", return_x=False, hooks=t)
wall = time.perf_counter() - t1
try:
    import torch

    free, total = torch.cuda.mem_get_info()
except Exception:  # noqa: BLE001
    free = total = None
print(json.dumps({"family": "crd3d", "n_g": ng, "n": p.n, "u_s": us, "alpha": 1.0, "steps": rep.iterations,
                  "status": rep.status, "device_s": round(t.ms / 1e3, 3), "wall_s": round(wall, 2),
                  "spec_build_s": round(t_build, 2), "relres": [h.relative_residual for h in rep.history],
                  "inner_h": [h.inner_h_iterations for h in rep.history],
                  "inner_s": [h.inner_s_iterations for h in rep.history],
                  "norm_iters": rep.norm_iterations, "norm_s": round(rep.norm_seconds, 3),
                  "gpu_free_gb_after": None if free is None else round(free / 2**30, 1),
                  "gpu_total_gb": None if total is None else round(total / 2**30, 1)}), flush=True)
