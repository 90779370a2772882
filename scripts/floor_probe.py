"""Run the outer loop to stagnation and print, per outer step, the cumulative
device time, relres and berr (to choose a benchmark tolerance both u_s reach).
Usage: floor_probe.py ng us alpha inner_tol maxit"""
import json
import math
import sys

import numpy as np

import paper_2512_21164_b200 as g
from paper_2512_21164_b200.analysis import power_start_vector
from paper_2512_21164_b200.device import make_desc, open_context
from paper_2512_21164_b200.precision import quantize

ng, us, alpha, itol, maxit = int(sys.argv[1]), sys.argv[2], float(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
target = float(sys.argv[6]) if len(sys.argv) > 6 else 0.0
p = g.build_cd_3d(ng)
spec = p.A.spec
ctx = open_context(make_desc(spec, alpha, us))
ctx.gen_rhs_ones()
ctx.set_exact(all_ones=True)
ctx.timer_start()
na, _ = ctx.norm2(power_start_vector(spec.n), 12345, 1e-6, 1000)
t_norm = ctx.timer_stop()
s0 = ctx.outer_begin()
r0 = math.sqrt(s0.sum_r2)
coeff = float(quantize((2.0 - 1.0) * alpha, us))
inner_max = min(10000, math.ceil(5 * math.sqrt(spec.n)))
rmax = s0.max_r
t = t_norm
hist = []
best = []
for k in range(maxit):
    scale = float(2.0 ** -np.ceil(np.log2(rmax))) if rmax > 0 else 1.0
    o, hs, ss, tm = ctx.outer_step(scale, coeff, itol, inner_max, inner_max)
    t += tm.inner_h + tm.inner_s + tm.residual
    relres = math.sqrt(o.sum_r2) / r0
    berr = math.sqrt(o.sum_r2) / (na * math.sqrt(o.sum_x2) + r0)
    hist.append((k, round(t / 1e3, 3), relres, berr, hs.iterations, ss.iterations))
    rmax = o.max_r
    best.append(relres)
    if relres <= target:
        break
    if len(best) > 10 and min(best[-10:]) > 0.99 * min(best[:-10]):
        break
print(json.dumps({"ng": ng, "us": us, "alpha": alpha, "inner_tol": itol, "norm_s": round(t_norm / 1e3, 3),
                  "hist": hist}))
