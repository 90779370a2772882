import json
import numpy as np
import paper_2512_21164_b200 as g
arr = np.load("tests/golden/csr.npz")
runs = {c["name"]: c for c in json.load(open("tests/golden/csr.json"))}
for name in ("c4_graded1e2_bf16", "c4_graded1e4_bf16", "c4_graded1e4_fp32"):
    c = runs[name]
    tag = c["problem"]
    n = arr[f"{tag}/rp"].size - 1
    a = g.SparseMatrix(arr[f"{tag}/rp"], arr[f"{tag}/ci"], arr[f"{tag}/v"], (n, n))
    p = g.Problem(A=a, b=arr[f"{tag}/b"], exact_solution=arr[f"{tag}/xs"], label=tag)
    for reuse in (True, False):
        rep = g.gadi_solve(p, cfg=g.GadiConfig(**c["cfg"]), reuse_context=reuse)
        xs = arr[f"{tag}/xs"]
        print(name, reuse, rep.status, rep.iterations, c["outer"], "ferr", [f"{h.forward_error:.3e}" for h in rep.history[:3]],
              [f"{h.forward_error:.3e}" for h in rep.history[-2:]], "true ferr", np.linalg.norm(rep.x - xs) / np.linalg.norm(xs),
              "berr", rep.history[-1].backward_error, c["berr"][-1])
