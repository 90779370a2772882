"""A few outer steps of cd3d (bf16 inner) for ncu captures."""
import sys
import paper_2512_21164_b200 as g

ng = int(sys.argv[1]) if len(sys.argv) > 1 else 256
us = sys.argv[2] if len(sys.argv) > 2 else "bf16"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
p = g.build_cd_3d(ng)
cfg = g.GadiConfig(alpha=0.025, u_s=us, outer_tol=1e-12, outer_maxit=steps, strict_model=False)
rep = g.gadi_solve(p, cfg=cfg, rounding="storage")
print(rep.iterations, [(h.inner_h_iterations, h.inner_s_iterations) for h in rep.history], rep.wallclock)
