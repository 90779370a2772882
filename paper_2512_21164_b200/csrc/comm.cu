// Communicators of the slab decomposition (comm.h) and their C ABI.
#include <dlfcn.h>
#include <nccl.h>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>
#include "ctx.h"

namespace gadi {

// ------------------------------------------------------------------ NCCL
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

// Bind NCCL: the copy already in the process (torch's) first, then
// $GADI_NCCL_LIB, then the loader's search path.
int load_nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.h) return 0;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h && getenv("GADI_NCCL_LIB")) h = dlopen(getenv("GADI_NCCL_LIB"), RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return set_error(std::string("cannot load NCCL: ") + dlerror(), GADI_ERR_UNSUPPORTED);
#define SYM(f, name)                                                                      \
  g_nccl.f = reinterpret_cast<decltype(g_nccl.f)>(dlsym(h, name));                        \
  if (!g_nccl.f) return set_error(std::string("NCCL symbol missing: ") + name, GADI_ERR_UNSUPPORTED);
  SYM(GetUniqueId, "ncclGetUniqueId");
  SYM(CommInitRank, "ncclCommInitRank");
  SYM(CommDestroy, "ncclCommDestroy");
  SYM(AllGather, "ncclAllGather");
  SYM(Send, "ncclSend");
  SYM(Recv, "ncclRecv");
  SYM(GroupStart, "ncclGroupStart");
  SYM(GroupEnd, "ncclGroupEnd");
  SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
  g_nccl.h = h;
  return 0;
}

#define GADI_NCCL(call)                                                                              \
  do {                                                                                               \
    ncclResult_t r_ = (call);                                                                        \
    if (r_ != ncclSuccess)                                                                           \
      return set_error(std::string(#call) + ": " + g_nccl.GetErrorString(r_), GADI_ERR_CUDA);        \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) g_nccl.CommDestroy(comm);
  }
  int gather(double* buf, int, cudaStream_t s) override {
    GADI_NCCL(g_nccl.AllGather(buf + (size_t)rank * GROW, buf, GROW, ncclDouble, comm, s));
    return 0;
  }
  int halo(void* base, size_t pb, long long nx, cudaStream_t s) override {
    unsigned char* b = static_cast<unsigned char*>(base);
    GADI_NCCL(g_nccl.GroupStart());
    if (rank > 0) {
      GADI_NCCL(g_nccl.Send(b, pb, ncclUint8, rank - 1, comm, s));
      GADI_NCCL(g_nccl.Recv(b - pb, pb, ncclUint8, rank - 1, comm, s));
    }
    if (rank < nranks - 1) {
      GADI_NCCL(g_nccl.Send(b + (size_t)(nx - 1) * pb, pb, ncclUint8, rank + 1, comm, s));
      GADI_NCCL(g_nccl.Recv(b + (size_t)nx * pb, pb, ncclUint8, rank + 1, comm, s));
    }
    GADI_NCCL(g_nccl.GroupEnd());
    return 0;
  }
  int exchange(const void* mine, size_t len, void* all, cudaStream_t s) override {
    unsigned char* d = nullptr;
    GADI_CUDA(cudaMalloc((void**)&d, len * (size_t)nranks));
    GADI_CUDA(cudaMemcpyAsync(d + len * (size_t)rank, mine, len, cudaMemcpyHostToDevice, s));
    const ncclResult_t r = g_nccl.AllGather(d + len * (size_t)rank, d, len, ncclUint8, comm, s);
    cudaError_t e = cudaMemcpyAsync(all, d, len * (size_t)nranks, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(d);
    if (r != ncclSuccess) return set_error(std::string("ncclAllGather: ") + g_nccl.GetErrorString(r), GADI_ERR_CUDA);
    GADI_CUDA(e);
    return 0;
  }
  const char* kind() const override { return "nccl"; }
};

// ------------------------------------------------------------------ local
// P slabs on one device, one host thread each.  Collectives synchronise the
// caller's stream, meet the other ranks at a host barrier, copy what they
// need from the peers' buffers, and meet again so no rank overwrites a
// buffer another is still reading.
struct Group {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  std::vector<void*> ptr;
  std::vector<const void*> cptr;
  std::vector<long long> nx;
  int members = 0;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const unsigned long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

std::mutex g_groups_mu;
std::map<int, std::shared_ptr<Group>> g_groups;

struct LocalComm : Comm {
  std::shared_ptr<Group> g;
  int key = 0;
  ~LocalComm() override {
    std::lock_guard<std::mutex> lk(g_groups_mu);
    if (--g->members == 0) g_groups.erase(key);
  }
  int gather(double* buf, int nr, cudaStream_t s) override {
    GADI_CUDA(cudaStreamSynchronize(s));
    g->ptr[rank] = buf;
    g->barrier();
    for (int j = 0; j < nranks; ++j)
      if (j != rank)
        GADI_CUDA(cudaMemcpyAsync(buf + (size_t)j * GROW, static_cast<double*>(g->ptr[j]) + (size_t)j * GROW,
                                  sizeof(double) * nr, cudaMemcpyDeviceToDevice, s));
    GADI_CUDA(cudaStreamSynchronize(s));
    g->barrier();
    return 0;
  }
  int halo(void* base, size_t pb, long long nx, cudaStream_t s) override {
    GADI_CUDA(cudaStreamSynchronize(s));
    g->ptr[rank] = base;
    g->nx[rank] = nx;
    g->barrier();
    unsigned char* b = static_cast<unsigned char*>(base);
    if (rank > 0) {
      const unsigned char* nb = static_cast<const unsigned char*>(g->ptr[rank - 1]);
      GADI_CUDA(cudaMemcpyAsync(b - pb, nb + (size_t)(g->nx[rank - 1] - 1) * pb, pb, cudaMemcpyDeviceToDevice, s));
    }
    if (rank < nranks - 1) {
      const unsigned char* nb = static_cast<const unsigned char*>(g->ptr[rank + 1]);
      GADI_CUDA(cudaMemcpyAsync(b + (size_t)nx * pb, nb, pb, cudaMemcpyDeviceToDevice, s));
    }
    GADI_CUDA(cudaStreamSynchronize(s));
    g->barrier();
    return 0;
  }
  int exchange(const void* mine, size_t len, void* all, cudaStream_t) override {
    g->cptr[rank] = mine;
    g->barrier();
    for (int j = 0; j < nranks; ++j) std::memcpy(static_cast<unsigned char*>(all) + len * (size_t)j, g->cptr[j], len);
    g->barrier();
    return 0;
  }
  const char* kind() const override { return "local"; }
};

}  // namespace
}  // namespace gadi

using namespace gadi;

extern "C" {

int gadi_comm_nccl_unique_id(unsigned char* out) {
  if (!out) return set_error("null argument", GADI_ERR_ARG);
  GADI_TRY(load_nccl());
  ncclUniqueId id;
  GADI_NCCL(g_nccl.GetUniqueId(&id));
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return 0;
}

int gadi_comm_create_nccl(const unsigned char* id, int nranks, int rank, int device, gadi_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return set_error("bad communicator arguments", GADI_ERR_ARG);
  *out = nullptr;
  GADI_TRY(load_nccl());
  GADI_CUDA(cudaSetDevice(device));
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
  auto* c = new NcclComm();
  c->rank = rank;
  c->nranks = nranks;
  c->want_peer = !(getenv("GADI_COMM") && std::string(getenv("GADI_COMM")) == "nccl");
  ncclResult_t r = g_nccl.CommInitRank(&c->comm, nranks, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return set_error(std::string("ncclCommInitRank: ") + g_nccl.GetErrorString(r), GADI_ERR_CUDA);
  }
  *out = new gadi_comm{c};
  return 0;
}

int gadi_comm_create_local(int key, int nranks, int rank, gadi_comm** out) {
  return gadi_comm_create_local2(key, nranks, rank, 0, out);
}

int gadi_comm_create_local2(int key, int nranks, int rank, int peer, gadi_comm** out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) return set_error("bad communicator arguments", GADI_ERR_ARG);
  std::shared_ptr<Group> g;
  {
    std::lock_guard<std::mutex> lk(g_groups_mu);
    auto& slot = g_groups[key];
    if (!slot) {
      slot = std::make_shared<Group>();
      slot->n = nranks;
      slot->ptr.assign(nranks, nullptr);
      slot->cptr.assign(nranks, nullptr);
      slot->nx.assign(nranks, 0);
    }
    if (slot->n != nranks) return set_error("local group size mismatch", GADI_ERR_ARG);
    slot->members++;
    g = slot;
  }
  auto* c = new LocalComm();
  c->g = g;
  c->key = key;
  c->rank = rank;
  c->nranks = nranks;
  c->want_peer = peer ? 1 : 0;
  *out = new gadi_comm{c};
  return 0;
}

int gadi_comm_destroy(gadi_comm* c) {
  if (!c) return 0;
  delete c->c;
  delete c;
  return 0;
}

int gadi_comm_info(gadi_comm* c, int* rank, int* nranks) {
  if (!c) return set_error("null communicator", GADI_ERR_ARG);
  if (rank) *rank = c->c->rank;
  if (nranks) *nranks = c->c->nranks;
  return 0;
}

}  // extern "C"
