"""TY=16 diagnosis: H/S-solves at several sizes in both rounding models with
the tensor-map and row-copy producers; prints iterations and a hash of z."""
import hashlib
import json
import os
import sys

import numpy as np

import paper_2512_21164_b200 as g
from paper_2512_21164_b200 import device
from paper_2512_21164_b200.inner import rounding_mode
from paper_2512_21164_b200.stencil import spec_cd_3d

for ng in (16, 40, 64):
    spec = spec_cd_3d(ng)
    rng = np.random.default_rng(ng)
    rhs = g.quantize(rng.uniform(-1.0, 1.0, spec.n), "bf16")
    for rnd in ("reference", "storage"):
        for tm in ("1", "0"):
            os.environ["GADI_TMAP"] = tm
            with device.open_context(device.make_desc(spec, 0.05, "bf16")) as ctx:
                ctx.set_rounding(rounding_mode(rnd), "fp32")
                zh, sh = ctx.h_solve(rhs, 1e-6, 400)
                zs, ss = ctx.s_solve(rhs, 1e-6, 400)
            h = hashlib.sha1(np.asarray(zh).tobytes()).hexdigest()[:10]
            print(json.dumps({"lib": os.environ.get("GADI_LIB", "default")[-20:], "ng": ng, "rnd": rnd, "tmap": tm,
                              "h_it": sh.iterations, "s_it": ss.iterations, "zh": h}), flush=True)
