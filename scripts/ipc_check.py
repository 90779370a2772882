"""Cross-process check of the peer transport's CUDA IPC path on ONE GPU:
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        --master-port 29611 scripts/ipc_check.py [NG]
Two processes (gloo for the blob exchange) share device 0; the slab solve must
match the single-domain solve (outer +-1, same status).  Kernels of the two
processes time-slice on one GPU, so every handshake costs a time slice: small
grids only."""
import json
import os
import sys
import time

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import torch.distributed as dist  # noqa: E402

import paper_2512_21164_b200 as g  # noqa: E402

ng = int(sys.argv[1]) if len(sys.argv) > 1 else 16
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
comm = g.SlabComm.host()
cfg = g.GadiConfig(alpha=0.5, u_s="bf16", outer_tol=1e-6, outer_maxit=300)
t0 = time.perf_counter()
rep = g.gadi_solve(g.build_cd_3d(ng), cfg=cfg, comm=comm, rounding="storage", reuse_context=False)
t = time.perf_counter() - t0
out = {"rank": rank, "world": world, "status": rep.status, "outer": rep.iterations, "slab": rep.slab, "s": round(t, 2)}
if rank == 0:
    ref = g.gadi_solve(g.build_cd_3d(ng), cfg=cfg, rounding="storage", reuse_context=False)
    out["ref_outer"] = ref.iterations
    out["ok"] = ref.status == rep.status and abs(ref.iterations - rep.iterations) <= 1
print(json.dumps(out), flush=True)
dist.barrier()
dist.destroy_process_group()
