"""CPU restatement of the slab decomposition -- TEST INFRASTRUCTURE ONLY.

The reference is single-process; the multi-GPU path of
this build (csrc/comm.cu, dist.py) splits the slowest grid axis
into contiguous slabs.  This module restates that algorithm with numpy on
top of the oracle's stencils (gadi_oracle.py) so that CPU tests can run it
over ``torch.distributed`` (gloo, world_size >= 2) and check it against the
single-domain oracle:

* ``slab_range`` -- the balanced contiguous split (first nx % P ranks take
  one extra plane);
* ``exchange_halos`` -- plane 0 to rank-1, plane nx-1 to rank+1 (the
  ncclSend/ncclRecv pair of comm.cu);
* ``slab_apply`` -- the stencil on [halo_lo; slab; halo_hi] restricted to the
  slab rows, bitwise the global stencil's rows;
* ``rank_order_sum`` -- all-gather of per-rank partials reduced in rank order
  (finalize_kernel), identical on every rank.

Only tests import it; the product never does.
"""

from __future__ import annotations

import numpy as np

from . import gadi_oracle as O


def slab_range(nx: int, nranks: int, rank: int):
    q, r = divmod(nx, nranks)
    x0 = rank * q + min(rank, r)
    return x0, x0 + q + (1 if rank < r else 0)


def _planes(op: O.Stencil, v, block=0):
    """View of one block of v as (planes, plane_size)."""
    nx = op.dims[0]
    m = int(np.prod(op.dims))
    vb = v[block * m:(block + 1) * m] if len(v) > m else v
    return vb.reshape(nx, -1)


def exchange_halos(local, rank, nranks, send, recv):
    """local: (planes, plane) array of this rank.  Returns (lo, hi) halo
    planes (None at the domain boundary).  send(t, dst) / recv(shape, src)
    are the transport (torch.distributed send/recv on CPU tensors)."""
    lo = hi = None
    # even ranks send first, odd ranks receive first: no deadlock with
    # blocking point-to-point calls
    ops = []
    if rank > 0:
        ops.append(("lo", rank - 1))
    if rank < nranks - 1:
        ops.append(("hi", rank + 1))
    for side, peer in ops:
        plane = local[0] if side == "lo" else local[-1]
        if rank % 2 == 0:
            send(plane, peer)
            got = recv(plane.shape, peer)
        else:
            got = recv(plane.shape, peer)
            send(plane, peer)
        if side == "lo":
            lo = got
        else:
            hi = got
    return lo, hi


def slab_apply(op: O.Stencil, x_local, x0, x1, halos, f="fp64"):
    """Rows [x0, x1) of op @ x from this slab's rows and its halo planes.

    ``x_local`` is the slab's part of x in the reference layout (crd: block
    form, both halves); ``halos`` holds (lo, hi) per block."""
    nx, ny, nz = op.dims
    nb = 2 if (op.v is not None or op.blocks == 2) else 1
    nloc = x1 - x0
    per = ny * nz
    has_lo, has_hi = x0 > 0, x1 < nx
    ext = nloc + has_lo + has_hi
    parts = []
    for b in range(nb):
        xb = np.asarray(x_local[b * nloc * per:(b + 1) * nloc * per]).reshape(nloc, per)
        lo, hi = halos[b]
        stack = ([lo[None]] if has_lo else []) + [xb] + ([hi[None]] if has_hi else [])
        parts.append(np.concatenate(stack).ravel())
    e0 = x0 - has_lo
    v = None if op.v is None else op.v.reshape(nx, per)[e0:e0 + ext].ravel()
    sub = O.Stencil((ext, ny, nz), op.d, op.lo, op.up, v, op.vsign, op.blocks)
    y = O.stencil_apply(sub, np.concatenate(parts), f)
    out = []
    for b in range(nb):
        yb = y[b * ext * per:(b + 1) * ext * per].reshape(ext, per)
        out.append(yb[has_lo:has_lo + nloc].ravel())
    return np.concatenate(out)


def rank_order_sum(partial: float, all_gather) -> float:
    """all_gather(value) -> list of every rank's value; summed in rank order."""
    vals = all_gather(partial)
    s = vals[0]
    for v in vals[1:]:
        s = s + v
    return s
