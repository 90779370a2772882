"""Row-copy vs tensor-map producer at 16-row tiles: z after k H-CG iterations
(storage model) and where the two first differ."""
import json
import os

import numpy as np

import paper_2512_21164_b200 as g
from paper_2512_21164_b200 import device
from paper_2512_21164_b200.inner import rounding_mode
from paper_2512_21164_b200.stencil import spec_cd_3d

import sys
for ng, k in [(int(a.split(":")[0]), int(a.split(":")[1])) for a in sys.argv[1:]] or [(32, 1), (32, 2), (32, 3)]:
  spec = spec_cd_3d(ng)
  rng = np.random.default_rng(5)
  rhs = g.quantize(rng.uniform(-1.0, 1.0, spec.n), "bf16")
  if True:
    out = {}
    for tm in ("1", "0"):
        os.environ["GADI_TMAP"] = tm
        with device.open_context(device.make_desc(spec, 0.05, "bf16")) as ctx:
            ctx.set_rounding(rounding_mode("storage"), "fp32")
            z, st = ctx.h_solve(rhs, 1e-12, k)
        out[tm] = np.asarray(z, dtype=np.float64).reshape(ng, ng, ng)
    d = np.abs(out["1"] - out["0"])
    idx = np.argwhere(d > 0)
    print(json.dumps({"ng": ng, "k": k, "ndiff": int(len(idx)), "max": float(d.max()),
                      "first": idx[:12].tolist(),
                      "x_hist": np.bincount(idx[:, 0], minlength=ng).tolist() if len(idx) else [],
                      "y_hist": np.bincount(idx[:, 1], minlength=ng).tolist() if len(idx) else [],
                      "z_hist": np.bincount(idx[:, 2], minlength=ng).tolist() if len(idx) else []}), flush=True)
