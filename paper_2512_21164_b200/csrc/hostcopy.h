// Host <-> device transfers of the fp64 vectors that cross the C ABI
// (right-hand side, exact solution, solution x: 1 GiB each at cd3d 512^3).
//
// A plain cudaMemcpy from pageable memory runs at ~11 GB/s on the B200 box
// (the driver stages through its own pinned buffers with one thread), and a
// D2H into a freshly allocated numpy array is dominated by the page faults of
// the destination (~180 ms per GiB, single-threaded).  The stager moves large
// vectors through two pinned chunk buffers: a small pool of host threads
// fills (H2D) or drains (D2H) one chunk -- faulting fresh destination pages
// in parallel -- while the copy engine moves the other.  Transfers below
// 2 chunks take the direct path.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace gadi {

struct HostStager;

// chunk_bytes per pinned buffer (two are allocated); threads = host copy
// threads (0: min(8, hardware threads / 2)).  Returns nullptr if the pinned
// allocation fails (callers then use the direct path).
HostStager* stager_create(size_t chunk_bytes, int threads);
void stager_destroy(HostStager* s);
size_t stager_chunk(const HostStager* s);

// dev <- host.  On return the host buffer has been read completely; the last
// chunks may still be in flight on `stream` (stream-ordered before later work).
cudaError_t stager_h2d(HostStager* s, void* dev, const void* host, size_t bytes, cudaStream_t stream);
// host <- dev, after all prior work on `stream`; synchronous.
cudaError_t stager_d2h(HostStager* s, void* host, const void* dev, size_t bytes, cudaStream_t stream);

}  // namespace gadi
