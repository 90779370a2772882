"""Golden grid search from the UNMODIFIED reference (REF/alphaselect.py:126-145):
PYTHONDONTWRITEBYTECODE=1 PYTHONPATH=/root/reference/pkg/src python tests/golden/make_alpha_golden.py"""
import json
from pathlib import Path

from gadimp import GadiConfig, build_cd_3d, build_cdr_2d
from gadimp.alphaselect import grid_search_alpha

out = []
for fam, ng, us, cands in (("cdr2d", 16, "fp32", [0.25, 0.5, 1.0, 2.0, 4.0]),
                           ("cd3d", 8, "bf16", [0.125, 0.25, 0.5, 1.0, 2.0])):
    p = (build_cdr_2d if fam == "cdr2d" else build_cd_3d)(ng)
    cfg = GadiConfig(alpha=1.0, u_s=us, outer_tol=1e-8, outer_maxit=400)
    best, counts = grid_search_alpha(p, cands, cfg)
    out.append({"family": fam, "n_g": ng, "u_s": us, "candidates": cands, "best": best, "counts": counts})
    print(fam, ng, us, best, counts)
(Path(__file__).resolve().parent / "alpha.json").write_text(json.dumps(out))
