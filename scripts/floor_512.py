"""The survey's berr-floor run: the benchmark workload with
outer_tol = 0, so the solve ends by the stagnation test at the attainable
floor; reports the per-step relres / berr and the final backward error."""
import json

import paper_2512_21164_b200 as g

for rounding in ("storage",):
    cfg = g.GadiConfig(alpha=0.0125, u_s="bf16", strict_model=False, inner_tol=1e-2, outer_tol=0.0, outer_maxit=400)
    rep = g.gadi_solve(g.build_cd_3d(512), cfg=cfg, rounding=rounding, return_x=False)
    print(json.dumps({"n_g": 512, "rounding": rounding, "outer_tol": 0.0, "status": rep.status,
                      "outer": rep.iterations, "final_berr": rep.history[-1].backward_error,
                      "min_berr": min(h.backward_error for h in rep.history),
                      "final_relres": rep.history[-1].relative_residual,
                      "final_ferr": rep.history[-1].forward_error,
                      "berr": [h.backward_error for h in rep.history],
                      "relres": [h.relative_residual for h in rep.history]}), flush=True)
