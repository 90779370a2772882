"""Slab decomposition across GPUs -- host side.

The grid's slowest axis (x planes of cd3d, rows of cdr2d / crd) is split into
contiguous slabs, one per rank (one process per GPU).  Every stencil pass
exchanges one halo plane with each neighbour (ncclSend/ncclRecv) and every
Krylov / monitor reduction all-gathers the per-rank sums, which each rank
then reduces in rank order on the device -- so all ranks take identical
decisions and the outer loop runs redundantly on every rank with no extra
broadcast.  The collectives live in the C library (csrc/comm.cu);
``torch.distributed`` is only the plumbing that broadcasts the NCCL unique id.

On one node the slab contexts switch from NCCL to the peer transport
(csrc/peer.cu): the neighbours' buffers are mapped with CUDA IPC and every
halo exchange / scalar all-gather is a few kernels writing peer memory and
synchronising on device flags, so the inner loops run as CUDA graphs with no
host involvement (``GADI_COMM=nccl`` keeps NCCL).

``SlabComm.local`` builds the same decomposition inside one process: P slabs
on one device, one host thread per rank, collectives by device copies behind
host barriers -- or, with ``peer=True``, by the peer-transport kernels (the
multi-GPU code path, plain pointers instead of IPC mappings).  It is the
single-GPU test harness of the multi-GPU path.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib

__all__ = ["SlabComm", "slab_range", "slab_rows", "nccl_library_path"]


def slab_range(nx: int, nranks: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of nx planes: the first nx % nranks ranks
    get one extra plane."""
    if not 0 <= rank < nranks or nx < nranks:
        raise ValueError(f"cannot split {nx} planes over {nranks} ranks (rank {rank})")
    q, r = divmod(nx, nranks)
    x0 = rank * q + min(rank, r)
    return x0, x0 + q + (1 if rank < r else 0)


def slab_rows(v: np.ndarray, spec, x0: int, x1: int) -> np.ndarray:
    """The slab's part of a global vector in the reference layout (the crd
    family is in block form [re; im], REF/problems.py:116: both halves are
    sliced)."""
    v = np.asarray(v)
    nx = spec.dims[0]
    if spec.family == "crd":
        m = v.size // 2
        per = m // nx
        return np.concatenate([v[x0 * per:x1 * per], v[m + x0 * per:m + x1 * per]])
    per = v.size // nx
    return v[x0 * per:x1 * per]


def nccl_library_path() -> str | None:
    """torch's bundled libnccl.so.2 (the C library also reuses an already
    loaded copy)."""
    try:
        import nvidia.nccl  # type: ignore

        for d in nvidia.nccl.__path__:
            p = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(p):
                return p
    except ImportError:
        pass
    return None


class SlabComm:
    """Handle of a ``gadi_comm`` (include/gadi_b200.h)."""

    def __init__(self, handle, kind: str):
        self.h = handle
        self.kind = kind
        r, n = C.c_int(), C.c_int()
        _lib.check(_lib.load().gadi_comm_info(handle, C.byref(r), C.byref(n)))
        self.rank, self.nranks = int(r.value), int(n.value)

    @classmethod
    def local(cls, key: int, nranks: int, rank: int, peer: bool = False) -> "SlabComm":
        """P slabs as P threads on one device.  peer=True: the contexts use the
        device-signalled peer transport (csrc/peer.cu) -- the kernels of the
        multi-GPU path -- instead of host barriers and copies.  The P ranks'
        streams then spin on each other's flags on one GPU, so each needs its
        own hardware queue: set CUDA_DEVICE_MAX_CONNECTIONS >= P + 2 before
        CUDA initialises (tests/conftest.py sets 32).  One process per GPU
        has one stream per device and no such constraint."""
        h = C.c_void_p()
        _lib.check(_lib.load().gadi_comm_create_local2(int(key), int(nranks), int(rank), 1 if peer else 0,
                                                       C.byref(h)))
        return cls(h, "local-peer" if peer else "local")

    @classmethod
    def host(cls, group=None) -> "SlabComm":
        """No transport of its own: each slab context built on it exchanges
        its CUDA IPC blob over ``torch.distributed`` (``group``, any backend)
        and attaches the device-signalled peer transport (csrc/peer.cu)."""
        import torch.distributed as dist

        h = C.c_void_p()
        _lib.check(_lib.load().gadi_comm_create_host(dist.get_world_size(group), dist.get_rank(group), C.byref(h)))
        c = cls(h, "host")
        c.group = group
        return c

    @staticmethod
    def unique_id() -> bytes:
        if nccl_library_path() and "GADI_NCCL_LIB" not in os.environ:
            os.environ["GADI_NCCL_LIB"] = nccl_library_path()
        buf = C.create_string_buffer(128)
        _lib.check(_lib.load().gadi_comm_nccl_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, uid: bytes, nranks: int, rank: int, device: int) -> "SlabComm":
        if len(uid) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        if nccl_library_path() and "GADI_NCCL_LIB" not in os.environ:
            os.environ["GADI_NCCL_LIB"] = nccl_library_path()
        h = C.c_void_p()
        _lib.check(_lib.lib().gadi_comm_create_nccl(uid, int(nranks), int(rank), int(device), C.byref(h)))
        return cls(h, "nccl")

    @staticmethod
    def broadcast_id(uid: bytes | None, group=None) -> bytes:
        """Rank 0's id to every rank through torch.distributed (any backend)."""
        import torch.distributed as dist

        obj = [uid]
        dist.broadcast_object_list(obj, src=0, group=group)
        return obj[0]

    @classmethod
    def from_torch(cls, device: int | None = None, group=None) -> "SlabComm":
        """NCCL communicator over the ranks of an initialised torch process group."""
        import torch.distributed as dist

        rank, nranks = dist.get_rank(group), dist.get_world_size(group)
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0"))
        uid = cls.unique_id() if rank == 0 else None
        uid = cls.broadcast_id(uid, group)
        return cls.nccl(uid, nranks, rank, device)

    def close(self):
        if getattr(self, "h", None):
            _lib.load().gadi_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
