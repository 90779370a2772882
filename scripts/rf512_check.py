"""Tiling-independence check at 512^3: the first outer steps in the
reference's per-operation rounding (fl_dot trees aligned to global index
blocks, so bitwise independent of the tile shape) -- compare the printed
histories across GADI_* tiling knobs."""
import json
import sys

import paper_2512_21164_b200 as g

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = g.GadiConfig(alpha=0.0125, u_s="bf16", outer_tol=1e-12, outer_maxit=steps, inner_tol=1e-2, strict_model=False)
rep = g.gadi_solve(g.build_cd_3d(512), cfg=cfg, return_x=False, rounding="reference")
print(json.dumps({"relres": [h.relative_residual for h in rep.history],
                  "inner_h": [h.inner_h_iterations for h in rep.history],
                  "inner_s": [h.inner_s_iterations for h in rep.history]}))
