// Slab-decomposition communicator.  The grid's slowest axis is
// split into contiguous slabs, one per rank; a stencil pass needs one halo
// plane from each neighbour, and every Krylov / monitor reduction needs the
// per-rank partial sums of all ranks.  Two collectives cover the hot path:
//
//   gather(buf, nr): rank r deposits nr doubles at buf[r*GROW ...]; after the
//                    call every rank holds every row (ncclAllGather).  Each
//                    rank then reduces the rows in rank order on the device
//                    (finalize_kernel), so all ranks take bitwise-identical
//                    decisions without a broadcast.
//   halo(base, plane_bytes, nx): send plane 0 to rank-1 (its plane nx) and
//                    plane nx-1 to rank+1 (its plane -1); receive likewise
//                    (ncclSend/ncclRecv in one group).
//
// NcclComm binds NCCL at run time (dlopen, so the library loads on hosts
// without it and reuses the copy torch already loaded).  LocalComm runs P
// slabs as P host threads on ONE device (the single-GPU test harness): the
// same engine code, collectives by device-to-device copies behind host
// barriers.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace gadi {

constexpr int GROW = 8;  // doubles per rank row of the gather buffer

struct Comm {
  int rank = 0, nranks = 1;
  int want_peer = 0;  // contexts built on this communicator switch to the peer transport (peer.cu)
  virtual ~Comm() {}
  virtual int gather(double* buf, int nr, cudaStream_t s) = 0;
  virtual int halo(void* base, size_t plane_bytes, long long nx, cudaStream_t s) = 0;
  // host bytes: every rank's `len` bytes, in rank order, into `all` (setup only)
  virtual int exchange(const void* mine, size_t len, void* all, cudaStream_t s) = 0;
  // collectives are kernels only (graph-capturable, no host in the loop)
  virtual bool device_only() const { return false; }
  // Split-phase halo of a vector whose producing pass writes its own boundary
  // planes straight into the neighbours' halo planes (peer transport):
  // halo_begin before the pass (the neighbours' slots are free; returns the
  // peer plane pointers for the pass, or false: use halo() after the pass),
  // halo_end after it (the data has landed on both sides).
  virtual bool halo_begin(void* /*base*/, size_t /*plane_bytes*/, long long /*nx*/, void** /*lo_plane*/,
                          void** /*hi_plane*/, cudaStream_t) { return false; }
  virtual int halo_end(void* /*base*/, cudaStream_t) { return 0; }
  virtual const char* kind() const = 0;
};

}  // namespace gadi

struct gadi_comm {
  gadi::Comm* c = nullptr;
};
