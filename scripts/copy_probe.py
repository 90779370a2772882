"""Time the host<->device legs of the e2e path at cd3d 512^3 (1 GiB fp64):
set_rhs from a resident pageable array, get_x into a fresh / pre-faulted
array, and the pinned-memory bandwidth for comparison."""
import json
import time

import numpy as np
import torch

import paper_2512_21164_b200 as g
from paper_2512_21164_b200 import device

spec = g.build_cd_3d(512).A.spec
n = spec.n
out = {}
b = np.ones(n)
with device.open_context(device.make_desc(spec, 0.0125, "bf16")) as ctx:
    ctx.set_rhs(b)
    for i in range(3):
        t = time.perf_counter(); ctx.set_rhs(b); out[f"set_rhs_{i}"] = time.perf_counter() - t
    for i in range(2):
        t = time.perf_counter(); x = ctx.get_x(); out[f"get_x_fresh_{i}"] = time.perf_counter() - t
    buf = np.empty(n); buf[:] = 0.0
    for i in range(2):
        t = time.perf_counter(); ctx.get_x(buf); out[f"get_x_prefaulted_{i}"] = time.perf_counter() - t
    t = time.perf_counter(); z = np.empty(n); z[:] = 0.0; out["np_empty_fault_1GiB"] = time.perf_counter() - t
    t = time.perf_counter(); np.copyto(z, b); out["host_memcpy_1GiB"] = time.perf_counter() - t
pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for i in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(pin); torch.cuda.synchronize()
    out[f"pinned_h2d_{i}"] = time.perf_counter() - t
    t = time.perf_counter(); pin.copy_(d); torch.cuda.synchronize(); out[f"pinned_d2h_{i}"] = time.perf_counter() - t
import os
out["cpus"] = os.cpu_count()
print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in out.items()}))
