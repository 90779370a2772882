"""Host-side tests of the slab decomposition (no GPU): the split, the
layout slicing, the NCCL-id plumbing over torch.distributed, and the
decomposition algorithm itself -- halo exchange + slab stencil + rank-order
reductions restated on the CPU (oracle/slab_oracle.py) and run over gloo
with world_size 2 and 3 against the single-domain oracle."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import gadi_oracle as O
from oracle import slab_oracle as SO
from paper_2512_21164_b200.dist import SlabComm, slab_range, slab_rows
from paper_2512_21164_b200.stencil import spec_cd_3d, spec_cdr_2d, spec_complex_rd


def test_slab_range_partitions():
    for nx in (1, 7, 16, 512, 1000):
        for P in (1, 2, 3, 4, 8):
            if nx < P:
                with pytest.raises(ValueError):
                    slab_range(nx, P, 0)
                continue
            r = [slab_range(nx, P, k) for k in range(P)]
            assert r[0][0] == 0 and r[-1][1] == nx
            assert all(r[k][1] == r[k + 1][0] for k in range(P - 1))
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1
            assert r == [SO.slab_range(nx, P, k) for k in range(P)]


@pytest.mark.parametrize("spec", [spec_cdr_2d(10), spec_cd_3d(6), spec_complex_rd(8)])
def test_slab_rows_cover_the_vector(spec):
    v = np.arange(spec.n, dtype=np.float64)
    P = 3
    parts = [slab_rows(v, spec, *slab_range(spec.dims[0], P, k)) for k in range(P)]
    if spec.family == "crd":
        re = np.concatenate([p[:p.size // 2] for p in parts])
        im = np.concatenate([p[p.size // 2:] for p in parts])
        assert np.array_equal(np.concatenate([re, im]), v)
    else:
        assert np.array_equal(np.concatenate(parts), v)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, fn, *args):
    port = _free_port()
    mp.start_processes(_entry, args=(world, port, fn, args), nprocs=world, start_method="fork", join=True)


def _entry(rank, world, port, fn, args):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def _send(t, dst):
    import torch

    dist.send(torch.from_numpy(np.ascontiguousarray(t)), dst)


def _recv(shape, src):
    import torch

    buf = torch.empty(shape, dtype=torch.float64)
    dist.recv(buf, src)
    return buf.numpy()


def _gather(v):
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, v)
    return out


def _stencil_worker(rank, world, family, ng, f):
    op = O.build(family, ng)
    rng = np.random.default_rng(3)
    x = rng.standard_normal(op.n)
    if f != "fp64":
        x = O.q(x, f)
    want = O.stencil_apply(op, x, f)
    x0, x1 = SO.slab_range(op.dims[0], world, rank)
    spec = {"cdr2d": spec_cdr_2d, "cd3d": spec_cd_3d, "crd": spec_complex_rd}[family](ng)
    xl = slab_rows(x, spec, x0, x1)
    nb = 2 if op.v is not None else 1
    nloc = x1 - x0
    halos = []
    for b in range(nb):
        planes = xl[b * xl.size // nb:(b + 1) * xl.size // nb].reshape(nloc, -1)
        halos.append(SO.exchange_halos(planes, rank, world, _send, _recv))
    got = SO.slab_apply(op, xl, x0, x1, halos, f)
    assert np.array_equal(got, slab_rows(want, spec, x0, x1)), (rank, family)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("family,ng,f", [("cdr2d", 12, "fp64"), ("cd3d", 9, "fp64"), ("cd3d", 8, "bf16"),
                                         ("crd", 10, "fp64")])
def test_gloo_slab_stencil_equals_single_domain(world, family, ng, f):
    _run(world, _stencil_worker, family, ng, f)


def _cg_worker(rank, world, ng, alpha):
    """fp64 CG on H = alpha I + M, distributed: slab stencils with halos,
    dot products as all-gathered partials summed in rank order."""
    op = O.cd3d(ng)
    H, _, _ = O.splitting(op, alpha, "fp64")
    rhs = np.random.default_rng(5).standard_normal(op.n)
    z_ref, st_ref = O.cg_spd(H, rhs, 1e-10, 200, "fp64")
    x0, x1 = SO.slab_range(op.dims[0], world, rank)
    sl = slice(x0 * ng * ng, x1 * ng * ng)

    def apply(v):
        lo, hi = SO.exchange_halos(v.reshape(x1 - x0, -1), rank, world, _send, _recv)
        return SO.slab_apply(H, v, x0, x1, [(lo, hi)])

    def dot(a, b):
        return SO.rank_order_sum(float(np.dot(a, b)), _gather)

    r = rhs[sl].copy()
    p = r.copy()
    z = np.zeros_like(r)
    rs = dot(r, r)
    nrhs = np.sqrt(dot(rhs[sl], rhs[sl]))
    it = 0
    while it < 200:
        hp = apply(p)
        a = rs / dot(p, hp)
        z += a * p
        r -= a * hp
        rs_new = dot(r, r)
        it += 1
        if np.sqrt(rs_new) / nrhs <= 1e-10:
            break
        p = r + (rs_new / rs) * p
        rs = rs_new
    assert abs(it - st_ref.iterations) <= 1, (it, st_ref.iterations)
    np.testing.assert_allclose(z, z_ref[sl], rtol=0, atol=1e-9 * np.abs(z_ref).max())


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_distributed_cg_matches_oracle(world):
    _run(world, _cg_worker, 9, 0.5)


def _id_worker(rank, world):
    uid = bytes(range(128)) if rank == 0 else None
    got = SlabComm.broadcast_id(uid)
    assert got == bytes(range(128))


def test_nccl_unique_id_broadcast_over_gloo():
    _run(2, _id_worker)
