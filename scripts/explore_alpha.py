"""Sweep alpha / precision for cd3d to pick the benchmark configuration."""
import sys, time, json
import paper_2512_21164_b200 as g

out = []
for spec in sys.argv[1:]:
    ng, alpha, us, tol, maxit = spec.split(":")
    p = g.build_cd_3d(int(ng))
    cfg = g.GadiConfig(alpha=float(alpha), u_s=us, outer_tol=float(tol), outer_maxit=int(maxit), strict_model=False)
    t0 = time.perf_counter()
    rep = g.gadi_solve(p, cfg=cfg)
    dt = time.perf_counter() - t0
    h = rep.history[-1]
    r = dict(ng=int(ng), alpha=float(alpha), us=us, tol=float(tol), status=rep.status, outer=rep.iterations,
             inner_h=sum(x.inner_h_iterations for x in rep.history), inner_s=sum(x.inner_s_iterations for x in rep.history),
             relres=h.relative_residual, berr=h.backward_error, ferr=h.forward_error, wall=dt,
             wc={k: round(v, 3) for k, v in rep.wallclock.items()}, normA=rep.norm_A)
    print(json.dumps(r), flush=True)
