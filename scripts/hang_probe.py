import sys, time
import paper_2512_21164_b200 as g
from paper_2512_21164_b200 import device
ng = int(sys.argv[1]); what = sys.argv[2]
p = g.build_cd_3d(ng)
t0 = time.time()
if what == "rhs":
    b = p.b; print("rhs ok", time.time() - t0, flush=True)
elif what == "norm":
    print("norm", g.matrix_norm_2(p.A), time.time() - t0, flush=True)
elif what == "solve":
    cfg = g.GadiConfig(alpha=0.0125, u_s="bf16", outer_tol=1e-12, inner_tol=1e-3, outer_maxit=int(sys.argv[3]), strict_model=False)
    r = g.gadi_solve(p, cfg=cfg); print("solve", r.status, r.iterations, time.time() - t0, flush=True)
