"""Peer-transport diagnostics: P slabs on one GPU (threads), timing per case.
python scripts/peer_diag.py P NG [graphs 0|1] [peer 0|1]"""
import json
import os

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import random
import sys
import threading
import time

import paper_2512_21164_b200 as g
from paper_2512_21164_b200.dist import SlabComm

P, ng = int(sys.argv[1]), int(sys.argv[2])
if len(sys.argv) > 3:
    os.environ["GADI_GRAPHS"] = sys.argv[3]
peer = len(sys.argv) <= 4 or sys.argv[4] == "1"
cfg = g.GadiConfig(alpha=0.0125, u_s="bf16", strict_model=False, inner_tol=1e-2, outer_tol=1e-3, outer_maxit=60)
t0 = time.perf_counter()
ref = g.gadi_solve(g.build_cd_3d(ng), cfg=cfg, reuse_context=False, rounding="storage", return_x=False)
t_ref = time.perf_counter() - t0
key = random.randrange(1 << 30)
out, errs, kinds = [None] * P, [], [None] * P


def work(r):
    comm = SlabComm.local(key, P, r, peer=peer)
    try:
        out[r] = g.gadi_solve(g.build_cd_3d(ng), cfg=cfg, comm=comm, reuse_context=False, rounding="storage",
                              return_x=False)
    except BaseException as e:  # noqa: BLE001
        errs.append(repr(e))
    finally:
        comm.close()


t0 = time.perf_counter()
ts = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(P)]
for t in ts:
    t.start()
for t in ts:
    t.join(120)
alive = sum(t.is_alive() for t in ts)
print(json.dumps({"P": P, "ng": ng, "graphs": os.environ.get("GADI_GRAPHS", "1"), "peer": peer, "alive": alive,
                  "errs": errs, "t_slabs": round(time.perf_counter() - t0, 2), "t_ref": round(t_ref, 2),
                  "ref_outer": ref.iterations,
                  "outer": [o.iterations if o else None for o in out]}), flush=True)
os._exit(0)
