// Device-signalled slab collectives over peer memory (one process per GPU on
// an NVLink / NVSwitch node, or P threads on one GPU for the tests).
//
// The NCCL transport (comm.cu) issues ncclSend/Recv groups and
// ncclAllGather between the passes and keeps the inner loops host-batched.
// Here every collective is a few small kernels on the context stream that
// read and write the neighbours' buffers directly (CUDA IPC mappings; plain
// pointers inside one process) and synchronise through epoch flags in the
// peers' memory (st.release.sys / ld.acquire.sys), so:
//   * a halo exchange is three launches -- "my halo slot is free" / wait for
//     the neighbours' slots, push my two boundary planes into the neighbours'
//     halo planes (grid-stride 16-byte stores over NVLink), "your data is
//     there" / wait for mine;
//   * the scalar all-gather is one single-thread kernel (the same two-phase
//     handshake around GROW doubles per rank);
// and, with no host in the loop, a slab context's inner solves run as the
// same CUDA-graph WHILE loops as a single domain.
//
// The epoch of each collective is a device counter advanced by the kernels
// themselves, so graph replays and WHILE-loop iterations stay in step on
// every rank (all ranks issue the same sequence of collectives).  The
// two-phase handshake makes every write into a peer's buffer wait until that
// peer has passed the same collective, i.e. has finished the passes that
// read the old halo / gather rows (no write-after-read hazard even when a
// rank runs one collective ahead).
#include <unistd.h>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <vector>
#include "ctx.h"

namespace gadi {

namespace {

constexpr int FSTRIDE = 16;  // u64 per flag slot (128 B: one writer per line)
enum : int { F_HREADY_LO = 0, F_HREADY_HI = 1, F_HDATA_LO = 2, F_HDATA_HI = 3, F_GREADY = 4 };
__host__ __device__ inline int f_gdata(int nranks) { return F_GREADY + nranks; }
inline int nflags(int nranks) { return F_GREADY + 2 * nranks; }

__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Bounded wait: a peer that never arrives (a crashed rank, a mismatched
// collective sequence) must not hang the GPU forever.  After ~10 s the wait
// records the fault in the context's error word (checked by the host at its
// next synchronisation: gadi_last_error) and gives up.
__device__ __forceinline__ void wait_ge(const unsigned long long* p, unsigned long long e, unsigned* err, int what,
                                        int rank) {
  const long long t0 = clock64();
  while (ld_acq(p) < e) {
    __nanosleep(128);
    if (clock64() - t0 > 20000000000LL) {
      if (err) atomicCAS(err, 0u, (unsigned)what);
      printf("gadi peer: rank %d wait %d timed out (epoch %llu, flag %llu)\n", rank, what, e, ld_acq(p));
      return;
    }
  }
}

struct HaloArgs {
  int rank;
  unsigned* err;               // the context's peer error word
  unsigned long long* cnt;     // this rank's epoch counters [0] halo, [1] gather
  unsigned long long* own;     // this rank's flags
  unsigned long long* lo_f;    // lower neighbour's flags (nullptr: none)
  unsigned long long* hi_f;    // upper neighbour's flags
  const uint4* src_lo;         // my plane 0
  uint4* dst_lo;               // lower neighbour's plane nx_lo (its upper halo)
  const uint4* src_hi;         // my plane nx-1
  uint4* dst_hi;               // upper neighbour's plane -1
  long long n16;               // 16-byte words per plane (0: byte path)
  long long nbytes;            // bytes per plane
};

__global__ void peer_halo_ready(HaloArgs a) {
  const unsigned long long e = ++a.cnt[0];
  if (a.lo_f) st_rel(a.lo_f + F_HREADY_HI * FSTRIDE, e);  // lower may write my plane -1
  if (a.hi_f) st_rel(a.hi_f + F_HREADY_LO * FSTRIDE, e);  // upper may write my plane nx
  if (a.lo_f) wait_ge(a.own + F_HREADY_LO * FSTRIDE, e, a.err, 1, a.rank);
  if (a.hi_f) wait_ge(a.own + F_HREADY_HI * FSTRIDE, e, a.err, 2, a.rank);
}

__global__ void peer_halo_push(HaloArgs a) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (a.n16) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.n16; i += stride) {
      if (a.dst_lo) a.dst_lo[i] = a.src_lo[i];
      if (a.dst_hi) a.dst_hi[i] = a.src_hi[i];
    }
  } else {  // planes that are not whole 16-byte words (small odd grids)
    const unsigned char* sl = reinterpret_cast<const unsigned char*>(a.src_lo);
    const unsigned char* sh = reinterpret_cast<const unsigned char*>(a.src_hi);
    unsigned char* dl = reinterpret_cast<unsigned char*>(a.dst_lo);
    unsigned char* dh = reinterpret_cast<unsigned char*>(a.dst_hi);
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.nbytes; i += stride) {
      if (dl) dl[i] = sl[i];
      if (dh) dh[i] = sh[i];
    }
  }
  __threadfence_system();
}

__global__ void peer_halo_done(HaloArgs a) {
  const unsigned long long e = a.cnt[0];
  __threadfence_system();
  if (a.lo_f) st_rel(a.lo_f + F_HDATA_HI * FSTRIDE, e);  // your upper halo is written
  if (a.hi_f) st_rel(a.hi_f + F_HDATA_LO * FSTRIDE, e);  // your lower halo is written
  if (a.lo_f) wait_ge(a.own + F_HDATA_LO * FSTRIDE, e, a.err, 3, a.rank);
  if (a.hi_f) wait_ge(a.own + F_HDATA_HI * FSTRIDE, e, a.err, 4, a.rank);
}

constexpr int MAXR = 64;
struct GatherArgs {
  unsigned* err;
  unsigned long long* cnt;
  unsigned long long* own;
  unsigned long long* pf[MAXR];  // peers' flags
  double* pg[MAXR];              // peers' gather buffers
  double* buf;                   // mine
  int rank, nranks, nr;
};

__global__ void peer_gather(GatherArgs a) {
  const unsigned long long g = ++a.cnt[1];
  const int gd = f_gdata(a.nranks);
  for (int j = 0; j < a.nranks; ++j)
    if (j != a.rank) st_rel(a.pf[j] + (F_GREADY + a.rank) * FSTRIDE, g);
  for (int j = 0; j < a.nranks; ++j)
    if (j != a.rank) wait_ge(a.own + (F_GREADY + j) * FSTRIDE, g, a.err, 5, a.rank);
  const double* mine = a.buf + (size_t)a.rank * GROW;
  for (int j = 0; j < a.nranks; ++j)
    if (j != a.rank)
      for (int s = 0; s < a.nr; ++s) a.pg[j][(size_t)a.rank * GROW + s] = mine[s];
  __threadfence_system();
  for (int j = 0; j < a.nranks; ++j)
    if (j != a.rank) st_rel(a.pf[j] + (gd + a.rank) * FSTRIDE, g);
  for (int j = 0; j < a.nranks; ++j)
    if (j != a.rank) wait_ge(a.own + (gd + j) * FSTRIDE, g, a.err, 6, a.rank);
}

// ------------------------------------------------------------------ export / import
constexpr int PB_MAGIC = 0x47504552;  // "GPER"
constexpr int MAXV = 16;
struct PeerBlob {
  int magic, pid, device, rank, nranks, nx, nvec, pad;
  struct Mem {
    cudaIpcMemHandle_t h;
    unsigned long long raw;  // raw allocation pointer in the exporter's address space
    long long off;           // vector base - raw
  } flags, gbuf, vec[MAXV];
};

struct Mapping {
  std::vector<void*> opened;  // IPC mappings to close
  ~Mapping() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
  }
};

struct PeerComm : Comm {
  Ctx* c = nullptr;
  unsigned long long* flags = nullptr;  // own (allocated by the context)
  unsigned long long* cnt = nullptr;
  std::vector<unsigned long long*> pflags;
  std::vector<double*> pgbuf;
  struct VecPeer {
    unsigned char* lo = nullptr;  // lower neighbour's vector base
    unsigned char* hi = nullptr;  // upper neighbour's vector base
  };
  std::map<const void*, VecPeer> vmap;
  long long nx_lo = 0, nx_hi = 0;
  Mapping maps;
  int gather(double* buf, int nr, cudaStream_t s) override {
    GatherArgs a;
    std::memset(&a, 0, sizeof(a));
    a.err = reinterpret_cast<unsigned*>(cnt + 2);
    a.cnt = cnt;
    a.own = flags;
    for (int j = 0; j < nranks; ++j) {
      a.pf[j] = pflags[j];
      a.pg[j] = pgbuf[j];
    }
    a.buf = buf;
    a.rank = rank;
    a.nranks = nranks;
    a.nr = nr;
    peer_gather<<<1, 1, 0, s>>>(a);
    GADI_CUDA(cudaGetLastError());
    return 0;
  }
  int halo(void* base, size_t pb, long long nx, cudaStream_t s) override {
    auto it = vmap.find(base);
    if (it == vmap.end()) return set_error("peer halo: buffer not registered", GADI_ERR_ARG);
    HaloArgs a;
    std::memset(&a, 0, sizeof(a));
    unsigned char* b = static_cast<unsigned char*>(base);
    a.rank = rank;
    a.err = reinterpret_cast<unsigned*>(cnt + 2);
    a.cnt = cnt;
    a.own = flags;
    a.nbytes = (long long)pb;
    a.n16 = pb % 16 ? 0 : (long long)(pb / 16);  // vector bases are 256-byte aligned
    if (rank > 0) {
      a.lo_f = pflags[rank - 1];
      a.src_lo = reinterpret_cast<const uint4*>(b);
      a.dst_lo = reinterpret_cast<uint4*>(it->second.lo + (size_t)nx_lo * pb);
    }
    if (rank < nranks - 1) {
      a.hi_f = pflags[rank + 1];
      a.src_hi = reinterpret_cast<const uint4*>(b + (size_t)(nx - 1) * pb);
      a.dst_hi = reinterpret_cast<uint4*>(it->second.hi - pb);
    }
    peer_halo_ready<<<1, 1, 0, s>>>(a);
    const long long units = a.n16 ? a.n16 : a.nbytes;
    const int nb = (int)std::min<long long>(std::max<long long>(1, (units + 255) / 256), 2LL * c->sms);
    peer_halo_push<<<nb, 256, 0, s>>>(a);
    peer_halo_done<<<1, 1, 0, s>>>(a);
    GADI_CUDA(cudaGetLastError());
    c->launches += 3;
    return 0;
  }
  bool halo_begin(void* base, size_t pb, long long nx, void** lo_plane, void** hi_plane, cudaStream_t s) override {
    auto it = vmap.find(base);
    if (it == vmap.end() || getenv_flag_off()) return false;
    HaloArgs a;
    std::memset(&a, 0, sizeof(a));
    a.rank = rank;
    a.err = reinterpret_cast<unsigned*>(cnt + 2);
    a.cnt = cnt;
    a.own = flags;
    *lo_plane = *hi_plane = nullptr;
    if (rank > 0) {
      a.lo_f = pflags[rank - 1];
      *lo_plane = it->second.lo + (size_t)nx_lo * pb;  // the lower neighbour's plane nx_lo
    }
    if (rank < nranks - 1) {
      a.hi_f = pflags[rank + 1];
      *hi_plane = it->second.hi - pb;  // the upper neighbour's plane -1
    }
    (void)nx;
    peer_halo_ready<<<1, 1, 0, s>>>(a);
    c->launches += 1;
    return cudaGetLastError() == cudaSuccess;
  }
  int halo_end(void* base, cudaStream_t s) override {
    HaloArgs a;
    std::memset(&a, 0, sizeof(a));
    a.rank = rank;
    a.err = reinterpret_cast<unsigned*>(cnt + 2);
    a.cnt = cnt;
    a.own = flags;
    if (rank > 0) a.lo_f = pflags[rank - 1];
    if (rank < nranks - 1) a.hi_f = pflags[rank + 1];
    (void)base;
    peer_halo_done<<<1, 1, 0, s>>>(a);
    c->launches += 1;
    GADI_CUDA(cudaGetLastError());
    return 0;
  }
  static bool getenv_flag_off() {
    static const bool off = getenv("GADI_FUSED_HALO") && atoi(getenv("GADI_FUSED_HALO")) == 0;
    return off;
  }
  int exchange(const void*, size_t, void*, cudaStream_t) override {
    return set_error("peer transport: exchange is a setup collective of the base communicator", GADI_ERR_UNSUPPORTED);
  }
  bool device_only() const override { return true; }
  const char* kind() const override { return "peer"; }
};

// the context's halo'd vectors, in allocation order (identical on every rank)
int export_blob(Ctx* c, PeerBlob* b) {
  std::memset(b, 0, sizeof(*b));
  b->magic = PB_MAGIC;
  b->pid = (int)getpid();
  b->device = c->device;
  b->rank = c->comm->rank;
  b->nranks = c->comm->nranks;
  b->nx = c->nx;
  if ((int)c->gvec.size() > MAXV) return set_error("too many halo'd vectors", GADI_ERR_UNSUPPORTED);
  b->nvec = (int)c->gvec.size();
  auto mem = [&](PeerBlob::Mem& m, void* raw, const void* base) -> int {
    GADI_CUDA(cudaIpcGetMemHandle(&m.h, raw));
    m.raw = (unsigned long long)(uintptr_t)raw;
    m.off = (long long)(static_cast<const unsigned char*>(base) - static_cast<unsigned char*>(raw));
    return 0;
  };
  GADI_TRY(mem(b->flags, c->pflags, c->pflags));
  GADI_TRY(mem(b->gbuf, c->gbuf, c->gbuf));
  for (int i = 0; i < b->nvec; ++i) GADI_TRY(mem(b->vec[i], c->gvec[i].raw, c->gvec[i].base));
  return 0;
}

}  // namespace

int peer_export(Ctx* c, void* out, size_t cap, size_t* len);

int peer_import(Ctx* c, const void* blobs, size_t blob_len) {
  if (!c->comm) return set_error("peer transport needs a slab context", GADI_ERR_ARG);
  if (blob_len != sizeof(PeerBlob)) return set_error("peer blob size mismatch", GADI_ERR_ARG);
  const int P = c->comm->nranks, me = c->comm->rank;
  if (P > MAXR) return set_error("too many ranks for the peer transport", GADI_ERR_UNSUPPORTED);
  const PeerBlob* all = static_cast<const PeerBlob*>(blobs);
  auto pc = std::make_unique<PeerComm>();
  pc->c = c;
  pc->rank = me;
  pc->nranks = P;
  pc->flags = c->pflags;
  pc->cnt = c->pcnt;
  const int mypid = (int)getpid();
  auto open = [&](const PeerBlob& b, const PeerBlob::Mem& m, unsigned char** out) -> int {
    if (b.pid == mypid) {  // same process: the raw pointer is valid here
      *out = reinterpret_cast<unsigned char*>((uintptr_t)m.raw) + m.off;
      return 0;
    }
    void* p = nullptr;
    GADI_CUDA(cudaIpcOpenMemHandle(&p, m.h, cudaIpcMemLazyEnablePeerAccess));
    pc->maps.opened.push_back(p);
    *out = static_cast<unsigned char*>(p) + m.off;
    return 0;
  };
  pc->pflags.assign(P, nullptr);
  pc->pgbuf.assign(P, nullptr);
  for (int j = 0; j < P; ++j) {
    const PeerBlob& b = all[j];
    if (b.magic != PB_MAGIC || b.rank != j || b.nranks != P || b.nvec != (int)c->gvec.size())
      return set_error("peer blobs do not describe the same decomposition", GADI_ERR_ARG);
    if (j == me) {
      pc->pflags[j] = c->pflags;
      pc->pgbuf[j] = c->gbuf;
      continue;
    }
    unsigned char* p = nullptr;
    GADI_TRY(open(b, b.flags, &p));
    pc->pflags[j] = reinterpret_cast<unsigned long long*>(p);
    GADI_TRY(open(b, b.gbuf, &p));
    pc->pgbuf[j] = reinterpret_cast<double*>(p);
  }
  for (int i = 0; i < (int)c->gvec.size(); ++i) {
    PeerComm::VecPeer vp;
    if (me > 0) GADI_TRY(open(all[me - 1], all[me - 1].vec[i], &vp.lo));
    if (me < P - 1) GADI_TRY(open(all[me + 1], all[me + 1].vec[i], &vp.hi));
    pc->vmap[c->gvec[i].base] = vp;
  }
  pc->nx_lo = me > 0 ? all[me - 1].nx : 0;
  pc->nx_hi = me < P - 1 ? all[me + 1].nx : 0;
  c->peer.reset(pc.release());
  return 0;
}

// Switch a slab context to the peer transport (collective over the base
// communicator): export, exchange, import, then agree -- every rank keeps the
// base transport unless all ranks imported successfully.
int peer_enable(Ctx* c) {
  Comm* base = c->comm;
  const int P = base->nranks;
  PeerBlob mine;
  int rc = peer_export(c, &mine, sizeof(mine), nullptr);
  std::vector<PeerBlob> all(P);
  struct Ok { int ok, pad[3]; };
  Ok me{rc == 0 ? 1 : 0, {0, 0, 0}};
  std::vector<Ok> oks(P);
  GADI_TRY(base->exchange(&me, sizeof(me), oks.data(), c->stream));
  for (const Ok& o : oks)
    if (!o.ok) return set_error("peer transport unavailable on some rank", GADI_ERR_UNSUPPORTED);
  GADI_TRY(base->exchange(&mine, sizeof(mine), all.data(), c->stream));
  rc = peer_import(c, all.data(), sizeof(PeerBlob));
  me.ok = rc == 0 ? 1 : 0;
  GADI_TRY(base->exchange(&me, sizeof(me), oks.data(), c->stream));
  bool every = true;
  for (const Ok& o : oks) every = every && o.ok;
  if (!every) {
    c->peer.reset();
    return set_error("peer transport: import failed on some rank", GADI_ERR_UNSUPPORTED);
  }
  c->base_comm = base;
  c->comm = c->peer.get();
  return 0;
}

int peer_export(Ctx* c, void* out, size_t cap, size_t* len) {
  if (!c->comm) return set_error("peer transport needs a slab context", GADI_ERR_ARG);
  if (len) *len = sizeof(PeerBlob);
  if (!out) return 0;
  if (cap < sizeof(PeerBlob)) return set_error("peer blob buffer too small", GADI_ERR_ARG);
  if (!c->pflags) {
    const size_t fb = sizeof(unsigned long long) * FSTRIDE * (size_t)nflags(c->comm->nranks);
    GADI_CUDA(cudaMalloc((void**)&c->pflags, fb));
    // pcnt: [0] halo epoch, [1] gather epoch, [2] error word (peer_check)
    GADI_CUDA(cudaMalloc((void**)&c->pcnt, 3 * sizeof(unsigned long long)));
    GADI_CUDA(cudaMemset(c->pflags, 0, fb));
    GADI_CUDA(cudaMemset(c->pcnt, 0, 3 * sizeof(unsigned long long)));
  }
  return export_blob(c, static_cast<PeerBlob*>(out));
}

}  // namespace gadi

namespace gadi {
// Host side of the bounded waits: after a synchronisation, report a peer
// that never arrived as an error instead of returning wrong results.
int peer_check(Ctx* c) {
  if (!c->peer || !c->pcnt) return 0;
  unsigned e = 0;
  GADI_CUDA(cudaMemcpy(&e, c->pcnt + 2, sizeof(unsigned), cudaMemcpyDeviceToHost));
  if (e) return set_error("peer transport: a neighbour did not arrive within 10 s (wait " + std::to_string(e) + ")",
                          GADI_ERR_CUDA);
  return 0;
}
}  // namespace gadi

using namespace gadi;

namespace {
// A communicator with no transport of its own: its slab contexts exchange
// their peer blobs through the caller (e.g. torch.distributed over gloo) and
// attach the peer transport with gadi_ctx_peer_attach.
struct HostComm : Comm {
  int gather(double*, int, cudaStream_t) override {
    return set_error("host communicator: attach the peer transport first", GADI_ERR_UNSUPPORTED);
  }
  int halo(void*, size_t, long long, cudaStream_t) override {
    return set_error("host communicator: attach the peer transport first", GADI_ERR_UNSUPPORTED);
  }
  int exchange(const void*, size_t, void*, cudaStream_t) override {
    return set_error("host communicator: the caller exchanges the blobs", GADI_ERR_UNSUPPORTED);
  }
  const char* kind() const override { return "host"; }
};
}  // namespace

extern "C" {

int gadi_comm_create_host(int nranks, int rank, gadi_comm** out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) return set_error("bad communicator arguments", GADI_ERR_ARG);
  auto* c = new HostComm();
  c->rank = rank;
  c->nranks = nranks;
  *out = new gadi_comm{c};
  return 0;
}

int gadi_ctx_peer_export(gadi_ctx* h, void* out, size_t cap, size_t* len) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  return peer_export(c, out, cap, len);
}

int gadi_ctx_peer_attach(gadi_ctx* h, const void* blobs, size_t blob_len) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  if (c->peer) return 0;
  GADI_TRY(peer_import(c, blobs, blob_len));
  c->base_comm = c->comm;
  c->comm = c->peer.get();
  return 0;
}

}  // extern "C"
