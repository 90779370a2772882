"""Storage-model outer counts of every golden solve vs the reference's (no asserts)."""
import json
import sys
sys.path.insert(0, ".")
import paper_2512_21164_b200 as g

B = {"cdr2d": g.build_cdr_2d, "cd3d": g.build_cd_3d, "crd": g.build_complex_rd}
out = []
for c in json.load(open("tests/golden/solves.json")):
    p = B[c["family"]](c["n_g"], **c.get("kw", {}) or {})
    rep = g.gadi_solve(p, cfg=g.GadiConfig(**c["cfg"]))
    d = rep.iterations - c["outer"]
    out.append((c["name"], rep.status, c["status"], rep.iterations, c["outer"], d,
                rep.history[-1].backward_error / c["berr"][-1]))
    print(f"{c['name']:28s} {rep.status:10s} {c['status']:10s} {rep.iterations:5d} {c['outer']:5d} {d:+3d} berr x{out[-1][-1]:.2f}")
