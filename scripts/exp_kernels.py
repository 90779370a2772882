"""Per-kernel live timings of a few outer steps (cd3d, bf16 inner) -- for
scheduling / tiling experiments driven by GADI_* environment knobs."""
import json
import os
import sys

import paper_2512_21164_b200 as g

ng = int(sys.argv[1]) if len(sys.argv) > 1 else 512
us = sys.argv[2] if len(sys.argv) > 2 else "bf16"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
fam = sys.argv[4] if len(sys.argv) > 4 else "cd3d"
build = {"cd3d": g.build_cd_3d, "cdr2d": g.build_cdr_2d, "crd": g.build_complex_rd}[fam]
cfg = g.GadiConfig(alpha=0.0125 if fam == "cd3d" else 1.0, u_s=us, outer_tol=1e-12, outer_maxit=steps,
                   inner_tol=1e-3, strict_model=False)
g.gadi_solve(build(ng), cfg=cfg, return_x=False, rounding="storage")  # warm-up
ctx = next(iter(g.device._CACHE.values()))
ctx.prof_enable(True)
rep = g.gadi_solve(build(ng), cfg=cfg, return_x=False, rounding="storage")
prof = ctx.prof_read()
ctx.prof_enable(False)
knobs = {k: v for k, v in os.environ.items() if k.startswith("GADI_")}
ih = sum(h.inner_h_iterations for h in rep.history)
is_ = sum(h.inner_s_iterations for h in rep.history)
real = {"hcg_a": ih, "hcg_b": ih, "cgnr_p1": is_, "cgnr_p2": is_, "cgnr_p3": max(1, is_ - rep.iterations), "norm_b": rep.norm_iterations,
        "norm_a": rep.norm_iterations, "outer": rep.iterations + 1, "hcg_init": rep.iterations,
        "cgnr_init": rep.iterations}
# per launch that did work (no-op launches past convergence included in the time)
print(json.dumps({"knobs": knobs, "ng": ng, "us": us, "norm_A": rep.norm_A, "norm_iterations": rep.norm_iterations,
                  "relres": [h.relative_residual for h in rep.history],
                  "kernels": {k: round(ms / max(1, min(n, real.get(k, n))) * 1e3, 2) for k, (ms, n) in prof.items()},
                  "launches": {k: n for k, (ms, n) in prof.items()}, "real": real,
                  "total_ms": {k: round(ms, 2) for k, (ms, n) in prof.items()}}))
