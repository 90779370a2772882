"""Per-step outer traces of the benchmark workload in both inner-solver
arithmetics (gadi_solve rounding="reference" | "storage"): relres, berr,
inner counts, time.  python scripts/rounding_trace.py NG [MAXIT] > jsonl"""
import json
import sys
import time

import paper_2512_21164_b200 as g

ng = int(sys.argv[1])
maxit = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for rounding in ("reference", "storage"):
    cfg = g.GadiConfig(alpha=0.0125, u_s="bf16", strict_model=False, inner_tol=1e-2, outer_tol=1e-12,
                       outer_maxit=maxit)
    t0 = time.perf_counter()
    rep = g.gadi_solve(g.build_cd_3d(ng), cfg=cfg, rounding=rounding, return_x=False)
    print(json.dumps({"n_g": ng, "rounding": rounding, "status": rep.status, "outer": rep.iterations,
                      "wall_s": round(time.perf_counter() - t0, 3),
                      "relres": [h.relative_residual for h in rep.history],
                      "berr": [h.backward_error for h in rep.history],
                      "inner_h": [h.inner_h_iterations for h in rep.history],
                      "inner_s": [h.inner_s_iterations for h in rep.history]}), flush=True)
