"""alpha / inner_tol / outer_tol exploration for the cd3d benchmark config."""
import json, sys, time
import paper_2512_21164_b200 as g
for spec in sys.argv[1:]:
    ng, alpha, us, tol, itol, maxit = spec.split(":")
    p = g.build_cd_3d(int(ng))
    cfg = g.GadiConfig(alpha=float(alpha), u_s=us, outer_tol=float(tol), inner_tol=float(itol),
                       outer_maxit=int(maxit), strict_model=False)
    t0 = time.perf_counter(); rep = g.gadi_solve(p, cfg=cfg); dt = time.perf_counter() - t0
    h = rep.history[-1]
    print(json.dumps(dict(ng=int(ng), alpha=float(alpha), us=us, tol=float(tol), itol=float(itol), status=rep.status,
        outer=rep.iterations, inner_h=sum(x.inner_h_iterations for x in rep.history),
        inner_s=sum(x.inner_s_iterations for x in rep.history), relres=h.relative_residual, berr=h.backward_error,
        wall=round(dt, 2), wc={k: round(v, 2) for k, v in rep.wallclock.items()})), flush=True)
