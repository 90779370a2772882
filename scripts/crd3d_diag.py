import json, sys
import numpy as np
import paper_2512_21164_b200 as g
d = {c["name"]: c for c in json.load(open("tests/golden/crd3d.json"))}
for n in ("crd3d6_fp64", "crd3d6_bf16", "crd3d8_fp64"):
    c = d[n]
    for rnd in ("storage", "reference"):
        rep = g.gadi_solve(g.build_complex_rd_3d(c["n_g"]), cfg=g.GadiConfig(**c["cfg"]), rounding=rnd)
        print(n, rnd, rep.iterations, c["outer"])
        print("  ours", ["%.4e" % h.relative_residual for h in rep.history[:6]], [h.inner_h_iterations for h in rep.history[:6]], [h.inner_s_iterations for h in rep.history[:6]])
        print("  ref ", ["%.4e" % r for r in c["relres"][:6]], c["inner_h"][:6], c["inner_s"][:6])
