"""Per-step outer trace (H its, S its, relres) of the storage-model solve,
several sizes, to compare with the CPU oracle."""
import json
import sys

import paper_2512_21164_b200 as g

us = sys.argv[1] if len(sys.argv) > 1 else "fp64"
alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0125
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 8
for ng in [int(v) for v in (sys.argv[4] if len(sys.argv) > 4 else "32,64,128,256,512").split(",")]:
    cfg = g.GadiConfig(alpha=alpha, u_s=us, outer_tol=0.0, outer_maxit=steps, inner_tol=1e-3, strict_model=False)
    rep = g.gadi_solve(g.build_cd_3d(ng), cfg=cfg, return_x=False, rounding="storage")
    print(json.dumps({"ng": ng, "us": us, "alpha": alpha,
                      "trace": [(h.inner_h_iterations, h.inner_s_iterations, h.relative_residual) for h in rep.history]}),
          flush=True)
