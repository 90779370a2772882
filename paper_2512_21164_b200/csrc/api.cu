// C ABI of the B200 GADI hot path (include/gadi_b200.h): context lifetime,
// host <-> device transfers in the reference's layout, the ||A||_2 power
// iteration, and the outer step that chains H-solve, S-solve and the fused
// update/residual/monitor pass.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include "engine.cuh"
#include "norm_fused.cuh"
#include "hostcopy.h"

namespace gadi {

static thread_local std::string g_err;
int set_error(const std::string& msg, int code) {
  g_err = msg;
  return code;
}

int kernel_occupancy(const void* fn, int device, int nthreads, size_t smem, bool carveout, int* occ) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({fn, device});
  if (it != cache.end()) {
    *occ = it->second;
    return 0;
  }
  if (smem > 48 * 1024) GADI_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (carveout) GADI_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int o = 0;
  GADI_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, nthreads, smem));
  if (o < 1) o = 1;
  cache[{fn, device}] = o;
  *occ = o;
  return 0;
}

static int getenv_int(const char* k) { return getenv(k) ? atoi(getenv(k)) : 0; }

static size_t fmt_bytes(int f) {
  switch (f) {
    case GADI_BF16:
    case GADI_FP16: return 2;
    case GADI_FP32: return 4;
    default: return 8;
  }
}

static EngineVT* engine_for(int us) {
  switch (us) {
    case GADI_BF16: return &engine_bf16;
    case GADI_FP16: return &engine_fp16;
    case GADI_FP32: return &engine_fp32;
    case GADI_FP64: return &engine_fp64;
    default: return nullptr;
  }
}

static int grid_blocks_pw(const Ctx* c) { return std::max(1, c->sms * 16); }

static int launch_1d(const Ctx* c, long long n) {
  return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, (long long)c->sms * 16));
}

// large vectors cross through the pinned double-buffered stager (hostcopy.h)
static cudaError_t h2d(Ctx* c, double* dev, const double* host, size_t bytes) {
  if (c->stager && bytes >= 2 * stager_chunk(c->stager)) return stager_h2d(c->stager, dev, host, bytes, c->stream);
  return cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, c->stream);
}
static cudaError_t d2h(Ctx* c, double* host, const double* dev, size_t bytes) {
  if (c->stager && bytes >= 2 * stager_chunk(c->stager)) return stager_d2h(c->stager, host, dev, bytes, c->stream);
  return cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, c->stream);
}

// host block layout -> device internal layout (crd: interleaved)
static int upload(Ctx* c, const double* host, double* dev) {
  if (c->kind == GADI_COMPLEX) {
    GADI_CUDA(h2d(c, c->tmp, host, sizeof(double) * c->n));
    interleave_kernel<<<launch_1d(c, c->n / 2), 256, 0, c->stream>>>(c->tmp, dev, c->n / 2);
    c->launches++;
  } else {
    GADI_CUDA(h2d(c, dev, host, sizeof(double) * c->n));
  }
  GADI_CUDA(cudaGetLastError());
  return 0;
}

static int download(Ctx* c, const double* dev, double* host) {
  if (c->kind == GADI_COMPLEX) {
    deinterleave_kernel<<<launch_1d(c, c->n / 2), 256, 0, c->stream>>>(dev, c->tmp, c->n / 2);
    c->launches++;
    GADI_CUDA(d2h(c, host, c->tmp, sizeof(double) * c->n));
  } else {
    GADI_CUDA(d2h(c, host, dev, sizeof(double) * c->n));
  }
  GADI_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

template <int DIM, int ZS, bool CPLX, bool TRANS>
static int norm_pass(Ctx* c, const double* in, double* out) {
  typedef GeoT<double, DIM, ZS> G;
  NormPass<G, CPLX, TRANS> p;
  p.ns = c->nst;
  p.in = in;
  p.outv = out;
  p.v = c->v64;
  p.A = TRANS ? c->AT : c->A;
  return launch_sweep(c, p);
}
// the same pass followed by the halo exchange of its output (fused push on
// the peer transport)
template <int DIM, int ZS, bool CPLX, bool TRANS>
static int norm_pass_halo(Ctx* c, const double* in, double* out) {
  typedef GeoT<double, DIM, ZS> G;
  NormPass<G, CPLX, TRANS> p;
  p.ns = c->nst;
  p.in = in;
  p.outv = out;
  p.v = c->v64;
  p.A = TRANS ? c->AT : c->A;
  HaloOut ho;
  const bool hf = halo_begin(c, out, 8, ho);
  GADI_TRY(launch_sweep(c, p, &ho));
  return halo_end(c, out, 8, hf);
}
template <bool TRANS>
static int norm_pass_h(Ctx* c, const double* in, double* out) {
  if (c->kind == GADI_COMPLEX)
    return c->ndim == 3 ? norm_pass_halo<3, 2, true, TRANS>(c, in, out)
                        : norm_pass_halo<2, 2, true, TRANS>(c, in, out);
  if (c->ndim == 3) return norm_pass_halo<3, 1, false, TRANS>(c, in, out);
  return norm_pass_halo<2, 1, false, TRANS>(c, in, out);
}

template <bool TRANS>
static int norm_pass_d(Ctx* c, const double* in, double* out) {
  if (c->kind == GADI_CSR) {
    const CsrDev& m = c->csr[TRANS ? CS_AT : CS_A];
    CsrNorm<TRANS> p;
    p.ns = c->nst;
    p.M = CsrT<double>{m.rp, m.ci, m.v64};
    p.in = in;
    p.outv = out;
    return launch_pw(c, p);
  }
  if (c->kind == GADI_COMPLEX)
    return c->ndim == 3 ? norm_pass<3, 2, true, TRANS>(c, in, out) : norm_pass<2, 2, true, TRANS>(c, in, out);
  if (c->ndim == 3) return norm_pass<3, 1, false, TRANS>(c, in, out);
  return norm_pass<2, 1, false, TRANS>(c, in, out);
}

// One power-iteration step in a single sweep (norm_fused.cuh): single-domain
// real stencils whose rows are TMA-aligned; other contexts use the two passes.
static bool norm_fused_ok(const Ctx* c) {
  if (c->kind != GADI_STENCIL || c->comm || c->no_tma) return false;
  if (getenv("GADI_NORM_2PASS") && atoi(getenv("GADI_NORM_2PASS"))) return false;
  return ((long long)c->nz * 8) % 16 == 0 && c->nz % GADI_VZNORM == 0;
}

template <int DIM, bool DENSE>
static int norm_fused_step(Ctx* c, const double* in, double* out) {
  using S = NFShape<DIM>;
  NormFused<DIM, DENSE> p;
  p.defer = nullptr;
  p.partials = c->partials;
  p.ticket = c->ticket;
  p.ns = c->nst;
  p.in = in;
  p.outv = out;
  p.A = c->A;
  p.AT = c->AT;
  // the v tile of a stage as one tensor-map box ((TZ + 2 HZ) x (TY + 2 HV)
  // fp64, zero-filled outside the grid) instead of TY + 2 HV row copies
  CUtensorMap tmw;
  std::memset(&tmw, 0, sizeof(tmw));
  p.use_tm = (DIM == 3 && c->tmap && !getenv_int("GADI_NORM_TM0") &&
              tm_map(c, in, 8, S::TZ + 2 * S::HZ, S::VROWS, &tmw)) ? 1 : 0;
  int occ = 1;
  GADI_TRY(occupancy_of(c, norm_fused_kernel<DIM, DENSE>, S::NTOT, S::SMEM, &occ, true));
  p.g = make_geom(c, S::TZ, S::TY, S::VZ, (long long)occ * c->sms);
  const long long units = (long long)p.g.nzt * p.g.nyt * p.g.nx;
  const int nb = (int)std::min<long long>(units, (long long)occ * c->sms * c->waves);
  if (nb > c->pstride) return set_error("fused norm grid exceeds partials buffer", GADI_ERR_ARG);
  prof_begin(c, K_NORM_B);
  norm_fused_kernel<DIM, DENSE><<<nb, S::NTOT, S::SMEM, c->stream>>>(p, tmw);
  prof_end(c);
  c->launches++;
  GADI_CUDA(cudaGetLastError());
  return 0;
}

// Vectors carry guard bands so the TMA sweep may copy whole padded rows
// (16 bytes before the first and up to a tile past the last element) and,
// in a slab decomposition, one halo plane on each side of the slab.  The
// whole allocation starts zeroed; the raw pointer is kept for freeing.
static constexpr size_t GUARD = 256 * 1024;
static size_t margin_bytes(const Ctx* c, size_t esz) { return c->comm ? esz * (size_t)c->ny * c->nz : 0; }
static cudaError_t guarded_malloc(Ctx* c, void** p, size_t bytes, size_t esz) {
  const size_t mb = margin_bytes(c, esz);
  unsigned char* raw = nullptr;
  cudaError_t e = cudaMalloc((void**)&raw, bytes + 2 * (GUARD + mb));
  if (e != cudaSuccess) return e;
  c->raws.push_back(raw);
  *p = raw + GUARD + mb;
  c->gvec.push_back({*p, raw});
  // on the context stream: a legacy-stream cudaMemset is not ordered with the
  // (non-blocking) context stream and could land after the first upload
  return cudaMemsetAsync(raw, 0, bytes + 2 * (GUARD + mb), c->stream);
}
// zero a vector including its halo planes
static int zero_vec(Ctx* c, void* p, size_t esz) {
  const size_t mb = margin_bytes(c, esz);
  GADI_CUDA(cudaMemsetAsync(static_cast<unsigned char*>(p) - mb, 0, esz * (size_t)c->n + 2 * mb, c->stream));
  return 0;
}

static void free_ctx(Ctx* c) {
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->peer) {
    c->comm = c->base_comm;
    c->peer.reset();
  }
  for (void* p : c->raws) cudaFree(p);
  c->raws.clear();
  for (CsrDev& m : c->csr) {
    void* cp[] = {m.rp, m.ci, m.v64, m.vs};
    for (void* p : cp)
      if (p) cudaFree(p);
    m = CsrDev();
  }
  void* sp[] = {c->v64, c->partials, c->VS, c->ticket, c->hst, c->sst, c->osum, c->nst, c->gbuf, c->wavecnt,
                c->tree, c->tlvl, c->tticket, c->taux, c->pflags, c->pcnt};
  for (void* p : sp)
    if (p) cudaFree(p);
  void* hp[] = {c->h_hst, c->h_sst, c->h_osum, c->h_nst};
  for (void* p : hp)
    if (p) cudaFreeHost(p);
  exact_free(c);
  stager_destroy(c->stager);
  c->stager = nullptr;
  if (c->gexec_h) cudaGraphExecDestroy(c->gexec_h);
  if (c->gexec_s) cudaGraphExecDestroy(c->gexec_s);
  if (c->graph_h) cudaGraphDestroy(c->graph_h);
  if (c->graph_s) cudaGraphDestroy(c->graph_s);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->evpool) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
}

}  // namespace gadi

using namespace gadi;

#define ALLOCG(ptr, bytes, esz)                                                                \
  do {                                                                                         \
    cudaError_t e_ = guarded_malloc(c, (void**)&(ptr), (bytes), (esz));                        \
    if (e_ != cudaSuccess) {                                                                   \
      free_ctx(c);                                                                             \
      delete h;                                                                                \
      return set_error(std::string("cudaMalloc ") + #ptr + ": " + cudaGetErrorString(e_),   \
                       e_ == cudaErrorMemoryAllocation ? GADI_ERR_OOM : GADI_ERR_CUDA);        \
    }                                                                                          \
  } while (0)

#define ALLOC(ptr, bytes)                                                                      \
  do {                                                                                         \
    cudaError_t e_ = cudaMalloc((void**)&(ptr), (bytes));                                      \
    if (e_ != cudaSuccess) {                                                                   \
      free_ctx(c);                                                                             \
      delete h;                                                                                \
      return set_error(std::string("cudaMalloc ") + #ptr + ": " + cudaGetErrorString(e_),   \
                       e_ == cudaErrorMemoryAllocation ? GADI_ERR_OOM : GADI_ERR_CUDA);        \
    }                                                                                          \
  } while (0)

extern "C" {

const char* gadi_last_error(void) { return g_err.c_str(); }

const char* gadi_build_info(void) {
  return "gadi_b200: sm_100a matrix-free GADI kernels (2.5-D stencil sweeps, device-side Krylov scalars)";
}

int gadi_device_count(int* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    return set_error(std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e), GADI_ERR_CUDA);
  }
  *count = n;
  return 0;
}

// Upload one CSR operator (int64 offsets, int32 columns, fp64 values; the
// u_s copy is made by the engine's quantize kernel).  `transpose` uploads
// the transpose instead (ascending columns by construction).
static int upload_csr(Ctx* c, const gadi_csr& h, CsrDev& d, bool transpose, bool typed) {
  if (!h.row_offsets || !h.col_indices || !h.values || h.nrows != c->n)
    return set_error("CSR operator missing or of the wrong size", GADI_ERR_ARG);
  const long long n = h.nrows, nnz = h.nnz;
  if (n >= (1LL << 31)) return set_error("CSR operators need fewer than 2^31 rows", GADI_ERR_UNSUPPORTED);
  // validate the structure before indexing with it (a malformed matrix must
  // not corrupt host memory: the reference raises IndexError)
  if (h.row_offsets[0] != 0 || h.row_offsets[n] != nnz || nnz < 0)
    return set_error("CSR row offsets must start at 0 and end at nnz", GADI_ERR_ARG);
  for (long long i = 0; i < n; ++i)
    if (h.row_offsets[i + 1] < h.row_offsets[i]) return set_error("CSR row offsets must be nondecreasing", GADI_ERR_ARG);
  for (long long k = 0; k < nnz; ++k)
    if (h.col_indices[k] < 0 || h.col_indices[k] >= n) return set_error("CSR column index out of range", GADI_ERR_ARG);
  std::vector<long long> rp(n + 1);
  std::vector<int> ci((size_t)nnz);
  std::vector<double> v((size_t)nnz);
  if (!transpose) {
    for (long long i = 0; i <= n; ++i) rp[i] = h.row_offsets[i];
    for (long long k = 0; k < nnz; ++k) {
      ci[k] = (int)h.col_indices[k];
      v[k] = h.values[k];
    }
  } else {
    std::fill(rp.begin(), rp.end(), 0LL);
    for (long long k = 0; k < nnz; ++k) rp[h.col_indices[k] + 1]++;
    for (long long i = 0; i < n; ++i) rp[i + 1] += rp[i];
    std::vector<long long> pos(rp.begin(), rp.end() - 1);
    for (long long i = 0; i < n; ++i)
      for (long long k = h.row_offsets[i]; k < h.row_offsets[i + 1]; ++k) {
        const long long dst = pos[h.col_indices[k]]++;
        ci[dst] = (int)i;
        v[dst] = h.values[k];
      }
  }
  d.nnz = nnz;
  GADI_CUDA(cudaMalloc((void**)&d.rp, sizeof(long long) * (size_t)(n + 1)));
  GADI_CUDA(cudaMalloc((void**)&d.ci, sizeof(int) * (size_t)std::max(1LL, nnz)));
  GADI_CUDA(cudaMalloc((void**)&d.v64, sizeof(double) * (size_t)std::max(1LL, nnz)));
  GADI_CUDA(cudaMemcpy(d.rp, rp.data(), sizeof(long long) * (size_t)(n + 1), cudaMemcpyHostToDevice));
  if (nnz) {
    GADI_CUDA(cudaMemcpy(d.ci, ci.data(), sizeof(int) * (size_t)nnz, cudaMemcpyHostToDevice));
    GADI_CUDA(cudaMemcpy(d.v64, v.data(), sizeof(double) * (size_t)nnz, cudaMemcpyHostToDevice));
  }
  if (typed) {
    GADI_CUDA(cudaMalloc(&d.vs, c->ssz * (size_t)std::max(1LL, nnz)));
    if (nnz) GADI_TRY(c->vt->quantize(c, d.v64, d.vs, nnz));
  }
  return 0;
}

// Optional L2 residency for one u_s vector of the inner solves
// (GADI_L2_PERSIST_MB = persisting bytes, GADI_L2_VEC = R | Z | RB | P0):
// an access-policy window on the context stream marks that share of the
// vector's lines persisting, so the pass that writes it and the next pass
// that reads it meet in L2 (kernel nodes captured from the stream inherit it).
static void l2_persist_setup(Ctx* c) {
  const char* e = getenv("GADI_L2_PERSIST_MB");
  if (!e || atof(e) <= 0.0 || c->kind == GADI_CSR) return;
  const char* which = getenv("GADI_L2_VEC") ? getenv("GADI_L2_VEC") : "R";
  void* base = c->R;
  if (!strcmp(which, "Z")) base = c->Z;
  else if (!strcmp(which, "RB")) base = c->RB;
  else if (!strcmp(which, "P0")) base = c->P[0];
  int maxwin = 0, maxpers = 0;
  cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, c->device);
  cudaDeviceGetAttribute(&maxpers, cudaDevAttrMaxPersistingL2CacheSize, c->device);
  const size_t want = (size_t)(atof(e) * 1048576.0);
  const size_t limit = std::min(want, (size_t)maxpers);
  const size_t bytes = c->ssz * (size_t)c->n;
  const size_t win = std::min(bytes, (size_t)maxwin);
  if (!limit || !win) return;
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, limit);
  cudaStreamAttrValue a = {};
  a.accessPolicyWindow.base_ptr = base;
  a.accessPolicyWindow.num_bytes = win;
  a.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)limit / (double)win);
  a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &a);
  if (getenv("GADI_L2_VERBOSE"))
    fprintf(stderr, "gadi: L2 persist %s: window %zu B of %zu, persisting limit %zu B (max window %d, max persisting %d)\n",
            which, win, bytes, limit, maxwin, maxpers);
  cudaGetLastError();
}

static int ctx_create(const gadi_problem_desc* desc, int device, gadi_comm* comm, int64_t x0, int64_t x1,
                      gadi_ctx** out) {
  if (!desc || !out) return set_error("null argument", GADI_ERR_ARG);
  *out = nullptr;
  if (desc->kind != GADI_STENCIL && desc->kind != GADI_COMPLEX && desc->kind != GADI_CSR)
    return set_error("unknown kind", GADI_ERR_ARG);
  if (desc->kind == GADI_CSR && comm) return set_error("CSR operators run on a single domain", GADI_ERR_UNSUPPORTED);
  EngineVT* vt = engine_for(desc->u_s);
  if (!vt) return set_error("u_s must be bf16, fp16, fp32 or fp64", GADI_ERR_ARG);
  gadi_ctx* h = new gadi_ctx();
  Ctx* c = &h->c;
  c->d = *desc;
  c->d.v = nullptr;
  c->device = device;
  c->kind = desc->kind;
  c->ndim = desc->ndim;
  c->us = desc->u_s;
  c->u = desc->u;
  c->ur = desc->u_r;
  c->ssz = fmt_bytes(desc->u_s);
  c->vt = vt;
  c->no_tma = getenv("GADI_NO_TMA") ? atoi(getenv("GADI_NO_TMA")) : 0;
  if (getenv("GADI_WAVES")) c->waves = std::max(1, atoi(getenv("GADI_WAVES")));
  if (getenv("GADI_MIN_CHUNK")) c->min_chunk = std::max(1, atoi(getenv("GADI_MIN_CHUNK")));
  if (getenv("GADI_LOCKSTEP")) c->lockstep = atoi(getenv("GADI_LOCKSTEP"));
  if (getenv("GADI_WAVEFRONT")) c->wavefront = atoi(getenv("GADI_WAVEFRONT"));
  if (getenv("GADI_BATCH_CAP")) c->batch_cap = std::max(0, atoi(getenv("GADI_BATCH_CAP")));
  if (getenv("GADI_TMA2")) c->tma2 = atoi(getenv("GADI_TMA2"));
  if (getenv("GADI_TALL")) c->tall = atoi(getenv("GADI_TALL"));
  if (getenv("GADI_ZLAG")) c->zlag_on = atoi(getenv("GADI_ZLAG")) != 0;
  if (getenv("GADI_TMAP")) c->tmap = atoi(getenv("GADI_TMAP"));
  if (getenv("GADI_TM_PROMO")) c->tm_promo = atoi(getenv("GADI_TM_PROMO"));
  if (getenv("GADI_GRAPHS")) c->graphs = atoi(getenv("GADI_GRAPHS"));
  if (c->kind == GADI_CSR) {
    // rows as a 1-D "grid" (no stencil geometry is used)
    c->nx = (int)desc->csr_A.nrows;
    c->ny = 1;
    c->nz = 1;
    c->ndim = 1;
  } else if (c->kind == GADI_STENCIL) {
    c->nx = (int)desc->dims[0];
    c->ny = (int)desc->dims[1];
    c->nz = (int)desc->dims[2];
    if (c->ndim == 2 && c->ny != 1) {
      delete h;
      return set_error("2-D stencils use dims (n_g, 1, n_g)", GADI_ERR_ARG);
    }
  } else {
    // crd: interleaved (re, im) pairs, z-stride 2; 2-D (n_g, 1, n_g) or the
    // 3-D extension (n_g, n_g, n_g)
    c->nx = (int)desc->dims[0];
    c->ny = (int)desc->dims[1];
    c->nz = 2 * (int)desc->dims[2];
    c->ndim = desc->ndim == 3 ? 3 : 2;
    if (c->ndim == 2 && c->ny != 1) {
      delete h;
      return set_error("2-D crd uses dims (n_g, 1, n_g)", GADI_ERR_ARG);
    }
    if (c->ur != GADI_FP64) {
      delete h;
      return set_error("complex family supports u_r = fp64 only", GADI_ERR_UNSUPPORTED);
    }
  }
  c->gn = (long long)c->nx * c->ny * c->nz;
  if (c->gn != desc->n || c->gn <= 0) {
    delete h;
    return set_error("dims do not match n", GADI_ERR_ARG);
  }
  c->gnx = c->nx;
  if (comm) {
    if (x0 < 0 || x1 <= x0 || x1 > c->gnx) {
      delete h;
      return set_error("slab range outside the grid", GADI_ERR_ARG);
    }
    c->comm = comm->c;
    c->x0 = (int)x0;
    c->nx = (int)(x1 - x0);
    c->hlo = x0 > 0 ? 1 : 0;
    c->hhi = x1 < c->gnx ? 1 : 0;
  }
  c->n = (long long)c->nx * c->ny * c->nz;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    delete h;
    return set_error(std::string("cudaSetDevice: ") + cudaGetErrorString(e), GADI_ERR_CUDA);
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) c->sms = prop.multiProcessorCount;
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete h;
    return set_error(std::string("cudaStreamCreate: ") + cudaGetErrorString(e), GADI_ERR_CUDA);
  }
  // coefficients
  c->A = coef_of(desc->A);
  c->AT = transpose_coef(c->A);
  c->H = coef_of(desc->H);
  c->S = coef_of(desc->S);
  c->ST = transpose_coef(c->S);
  c->A32 = cast_coef<float>(c->A);
  // partials stride: the largest grid any pass of this context launches
  {
    int mx = grid_blocks_pw(c) + 64;
    const int vzs = std::max(2, (int)(16 / c->ssz));
    const int bz = c->ndim == 3 ? 32 : 64, by = c->ndim == 3 ? 8 : 1;
    const int tzs[2] = {bz * vzs, bz * 2};
    for (int t : tzs) {
      c->pstride = 0;
      SweepGeom g = make_geom(c, t, by, 1);
      mx = std::max(mx, geom_blocks(g));
    }
    mx = std::max(mx, c->sms * 16 * c->waves + 64);
    c->pstride = mx;
  }
  const size_t n8 = sizeof(double) * (size_t)c->n, ns = c->ssz * (size_t)c->n;
  ALLOCG(c->b, n8, 8);
  ALLOCG(c->x[0], n8, 8);
  ALLOCG(c->x[1], n8, 8);
  ALLOCG(c->r, n8, 8);
  ALLOCG(c->tmp, n8, 8);
  ALLOCG(c->R, ns, c->ssz);
  ALLOCG(c->P[0], ns, c->ssz);
  ALLOCG(c->P[1], ns, c->ssz);
  ALLOCG(c->Z, ns, c->ssz);
  ALLOCG(c->RB, ns, c->ssz);
  ALLOCG(c->Y, ns, c->ssz);
  ALLOC(c->gbuf, sizeof(double) * GROW * (size_t)(c->comm ? c->comm->nranks : 1));
  ALLOC(c->wavecnt, sizeof(unsigned) * 2 * (size_t)c->nx);
  ALLOC(c->partials, sizeof(double) * 8 * (size_t)c->pstride);
  ALLOC(c->ticket, sizeof(unsigned int));
  ALLOC(c->hst, sizeof(InnerState));
  ALLOC(c->sst, sizeof(InnerState));
  ALLOC(c->osum, sizeof(OuterSums));
  ALLOC(c->nst, sizeof(NormState));
  if (c->kind == GADI_COMPLEX) {
    if (!desc->v) {
      free_ctx(c);
      delete h;
      return set_error("complex family needs v", GADI_ERR_ARG);
    }
    ALLOC(c->v64, sizeof(double) * (size_t)(c->n / 2));
    ALLOC(c->VS, c->ssz * (size_t)(c->n / 2));
  }
#define CHK(call)                                                                    \
  do {                                                                               \
    cudaError_t e2_ = (call);                                                        \
    if (e2_ != cudaSuccess) {                                                        \
      free_ctx(c);                                                                   \
      delete h;                                                                      \
      return set_error(std::string(#call) + ": " + cudaGetErrorString(e2_), GADI_ERR_CUDA); \
    }                                                                                \
  } while (0)
  CHK(cudaMallocHost((void**)&c->h_hst, sizeof(InnerState)));
  CHK(cudaMallocHost((void**)&c->h_sst, sizeof(InnerState)));
  CHK(cudaMallocHost((void**)&c->h_osum, sizeof(OuterSums)));
  CHK(cudaMallocHost((void**)&c->h_nst, sizeof(NormState)));
  // vectors of >= 128 MiB cross the ABI through pinned 32 MiB chunks (falls
  // back to direct copies if the pinned allocation fails)
  if ((size_t)c->n * sizeof(double) >= ((size_t)128 << 20) && !std::getenv("GADI_NO_STAGER"))
    c->stager = stager_create((size_t)32 << 20, 0);
  for (auto& ev : c->ev) CHK(cudaEventCreate(&ev));
  CHK(cudaMemsetAsync(c->ticket, 0, sizeof(unsigned int), c->stream));
  CHK(cudaMemsetAsync(c->wavecnt, 0, sizeof(unsigned) * 2 * (size_t)c->nx, c->stream));
  CHK(cudaMemsetAsync(c->hst, 0, sizeof(InnerState), c->stream));
  CHK(cudaMemsetAsync(c->sst, 0, sizeof(InnerState), c->stream));
  if (c->kind == GADI_COMPLEX) {
    // desc->v is the whole grid's potential; this slab owns rows [x0, x0+nx)
    const double* vs = desc->v + (size_t)c->x0 * (size_t)c->ny * (size_t)(c->nz / 2);
    CHK(cudaMemcpyAsync(c->v64, vs, sizeof(double) * (size_t)(c->n / 2), cudaMemcpyHostToDevice, c->stream));
    int rc = c->vt->quantize(c, c->v64, c->VS, c->n / 2);
    if (rc) {
      free_ctx(c);
      delete h;
      return rc;
    }
  }
  if (c->kind == GADI_CSR) {
    const gadi_csr* ops[CS_N] = {&desc->csr_A, &desc->csr_A, &desc->csr_H, &desc->csr_S, &desc->csr_ST};
    for (int s = 0; s < CS_N; ++s) {
      int rc = upload_csr(c, *ops[s], c->csr[s], s == CS_AT, s >= CS_H);
      if (rc) {
        free_ctx(c);
        delete h;
        return rc;
      }
    }
  }
  CHK(cudaStreamSynchronize(c->stream));
#undef CHK
  l2_persist_setup(c);
  // slab contexts: device-signalled collectives over peer memory when every
  // rank can map its neighbours (peer.cu); otherwise the base transport
  if (c->comm && c->comm->want_peer && c->kind != GADI_CSR) {
    if (peer_enable(c) != 0 && getenv("GADI_COMM_VERBOSE"))
      fprintf(stderr, "gadi: peer transport off (%s), using %s\n", gadi_last_error(), c->comm->kind());
  }
  *out = h;
  return 0;
}

int gadi_ctx_create(const gadi_problem_desc* desc, int device, gadi_ctx** out) {
  return ctx_create(desc, device, nullptr, 0, 0, out);
}

int gadi_ctx_create_slab(const gadi_problem_desc* desc, int device, gadi_comm* comm, int64_t x0, int64_t x1,
                         gadi_ctx** out) {
  if (!comm) return set_error("slab context needs a communicator", GADI_ERR_ARG);
  return ctx_create(desc, device, comm, x0, x1, out);
}

int gadi_ctx_slab(gadi_ctx* h, int64_t* x0, int64_t* x1, int64_t* n_local) {
  Ctx* c = &h->c;
  if (x0) *x0 = c->x0;
  if (x1) *x1 = c->x0 + c->nx;
  if (n_local) *n_local = c->n;
  return 0;
}

int gadi_ctx_destroy(gadi_ctx* h) {
  if (!h) return 0;
  free_ctx(&h->c);
  delete h;
  return 0;
}

int gadi_set_rhs(gadi_ctx* h, const double* b) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  GADI_TRY(upload(c, b, c->b));
  GADI_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int gadi_gen_rhs_ones(gadi_ctx* h) {
  Ctx* c = &h->c;
  if (c->kind == GADI_CSR) return set_error("b = A 1 is generated for stencil families only", GADI_ERR_UNSUPPORTED);
  GADI_CUDA(cudaSetDevice(c->device));
  RhsOnes p;
  p.nx = c->gnx;
  p.x0 = c->x0;
  p.ny = c->ny;
  p.nz = c->nz;
  p.zs = c->kind == GADI_COMPLEX ? 2 : 1;
  p.plane = (long long)c->ny * c->nz;
  p.A = c->A;
  p.v = c->v64;
  p.b = c->b;
  rhs_ones_kernel<<<launch_1d(c, c->n), 256, 0, c->stream>>>(p, c->n);
  c->launches++;
  GADI_CUDA(cudaGetLastError());
  GADI_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

int gadi_get_rhs(gadi_ctx* h, double* b) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  return download(c, c->b, b);
}

int gadi_set_exact(gadi_ctx* h, const double* xs, int all_ones) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  if (xs) {
    if (!c->xs) GADI_CUDA(guarded_malloc(c, (void**)&c->xs, sizeof(double) * (size_t)c->n, 8));
    GADI_TRY(upload(c, xs, c->xs));
    GADI_TRY(halo(c, c->xs, 8));
    GADI_CUDA(cudaStreamSynchronize(c->stream));
    c->has_exact = 1;
    c->ones = 0;
  } else {
    c->has_exact = all_ones ? 1 : 0;
    c->ones = all_ones ? 1 : 0;
  }
  return 0;
}

int gadi_norm2(gadi_ctx* h, const double* v0, uint64_t seed, double tol, int maxit, double* sigma, int* iterations) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  double* w = c->x[0];
  double* t = c->x[1];
  const bool fused = norm_fused_ok(c);
  GADI_CUDA(cudaEventRecord(c->ev[6], c->stream));
  if (v0) {
    GADI_TRY(upload(c, v0, w));  // this slab's rows of the normalised start vector
  } else {
    // N(0,1) by global index, normalised over all slabs (analysis.py:54-57)
    const int nb = launch_1d(c, c->n);
    const int rank = c->comm ? c->comm->rank : 0, nranks = c->comm ? c->comm->nranks : 1;
    randn_kernel<<<nb, 256, 0, c->stream>>>(w, c->n, (unsigned long long)seed, (long long)c->x0 * c->ny * c->nz);
    sumsq_kernel<<<nb, 256, 0, c->stream>>>(w, c->n, c->partials);
    partials_total_kernel<<<1, 32, 0, c->stream>>>(c->partials, nb, c->gbuf + (size_t)rank * GROW);
    c->launches += 3;
    GADI_CUDA(cudaGetLastError());
    if (c->comm) GADI_TRY(c->comm->gather(c->gbuf, 1, c->stream));
    scale_by_norm_kernel<<<nb, 256, 0, c->stream>>>(w, c->n, c->gbuf, nranks, GROW);
    c->launches++;
    GADI_CUDA(cudaGetLastError());
  }
  GADI_TRY(halo(c, w, 8));
  norm_state_init<<<1, 1, 0, c->stream>>>(c->nst, tol, maxit);
  c->launches++;
  int launched = 0, batch = 64;
  bool polled = false;
  while (launched < maxit) {
    const int nb = std::min(batch, maxit - launched);
    for (int j = 0; j < nb; ++j) {
      if (fused) {
        // every coefficient of A nonzero (cd3d): the branch-free ordered stencil
        const bool dense = c->A.d != 0.0 && c->A.lo[0] != 0.0 && c->A.lo[1] != 0.0 && c->A.lo[2] != 0.0 &&
                           c->A.up[0] != 0.0 && c->A.up[1] != 0.0 && c->A.up[2] != 0.0;
        const int rc = c->ndim == 3 ? (dense ? norm_fused_step<3, true>(c, w, t) : norm_fused_step<3, false>(c, w, t))
                                    : norm_fused_step<2, false>(c, w, t);
        if (rc) return rc;
        std::swap(w, t);
        continue;
      }
      if (c->comm && c->kind != GADI_CSR) {  // slabs: the passes push their halo planes
        GADI_TRY(norm_pass_h<false>(c, w, t));
        GADI_TRY(norm_pass_h<true>(c, t, w));
      } else {
        GADI_TRY(norm_pass_d<false>(c, w, t));
        GADI_TRY(halo(c, t, 8));
        GADI_TRY(norm_pass_d<true>(c, t, w));
        GADI_TRY(halo(c, w, 8));
      }
    }
    launched += nb;
    GADI_CUDA(cudaMemcpyAsync(c->h_nst, c->nst, sizeof(NormState), cudaMemcpyDeviceToHost, c->stream));
    GADI_CUDA(cudaStreamSynchronize(c->stream));
    prof_collect(c);
    polled = true;
    if (c->h_nst->done) break;
    batch = 128;
  }
  if (!polled) {
    GADI_CUDA(cudaMemcpyAsync(c->h_nst, c->nst, sizeof(NormState), cudaMemcpyDeviceToHost, c->stream));
    GADI_CUDA(cudaStreamSynchronize(c->stream));
  }
  GADI_CUDA(cudaEventRecord(c->ev[7], c->stream));
  GADI_CUDA(cudaEventSynchronize(c->ev[7]));
  float ms = 0.f;
  GADI_CUDA(cudaEventElapsedTime(&ms, c->ev[6], c->ev[7]));
  c->last_norm_ms = ms;
  *sigma = c->h_nst->sigma;
  if (iterations) *iterations = c->h_nst->it;
  // leave x = 0 (halo planes included) for the solve
  GADI_TRY(zero_vec(c, c->x[0], 8));
  GADI_TRY(zero_vec(c, c->x[1], 8));
  GADI_CUDA(cudaStreamSynchronize(c->stream));
  return 0;
}

static void fill_scalars(const OuterSums* s, gadi_outer_scalars* o) {
  o->sum_r2 = s->v[0];
  o->max_r = s->v[1];
  o->sum_ralg2 = s->v[2];
  o->sum_x2 = s->v[3];
  o->sum_e2 = s->v[4];
  o->sum_ae2 = s->v[5];
}

static void fill_stats(const InnerState* s, gadi_inner_stats* o) {
  o->iterations = s->it;
  o->converged = s->converged;
  o->breakdown = s->breakdown;
  o->pad = 0;
  o->final_relative_residual = s->relres;
}

int gadi_outer_begin(gadi_ctx* h, gadi_outer_scalars* out) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  GADI_TRY(zero_vec(c, c->x[c->xcur], 8));
  GADI_TRY(zero_vec(c, c->Y, c->ssz));
  GADI_TRY(c->vt->outer(c, 1.0, c->has_exact));
  GADI_CUDA(cudaMemcpyAsync(c->h_osum, c->osum, sizeof(OuterSums), cudaMemcpyDeviceToHost, c->stream));
  GADI_CUDA(cudaStreamSynchronize(c->stream));
  if (out) fill_scalars(c->h_osum, out);
  c->pred_h = 4;
  c->pred_s = 4;
  return 0;
}

int gadi_outer_step(gadi_ctx* h, const gadi_step_args* a, gadi_outer_scalars* out, gadi_inner_stats* hs,
                    gadi_inner_stats* ss, gadi_phase_times* t) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  GADI_CUDA(cudaEventRecord(c->ev[0], c->stream));
  if (c->rounding == 2) {
    GADI_TRY(exact_h_solve(c, c->r, a->scale, a->inner_tol, a->maxit_h));
    GADI_CUDA(cudaEventRecord(c->ev[1], c->stream));
    GADI_TRY(exact_s_solve(c, c->ex[EX_Z], a->coeff, a->inner_tol, a->maxit_s));
    GADI_TRY(c->vt->quantize(c, c->ex[EX_Y], c->Y, c->n));  // exact: y holds u_s images
  } else {
    GADI_TRY(c->vt->h_solve(c, a->scale, a->inner_tol, a->maxit_h));
    GADI_CUDA(cudaEventRecord(c->ev[1], c->stream));
    GADI_TRY(c->vt->s_solve(c, a->coeff, a->inner_tol, a->maxit_s));
  }
  GADI_CUDA(cudaEventRecord(c->ev[2], c->stream));
  GADI_TRY(c->vt->outer(c, a->scale, c->has_exact));
  GADI_CUDA(cudaEventRecord(c->ev[3], c->stream));
  GADI_CUDA(cudaMemcpyAsync(c->h_osum, c->osum, sizeof(OuterSums), cudaMemcpyDeviceToHost, c->stream));
  GADI_CUDA(cudaStreamSynchronize(c->stream));
  prof_collect(c);
  if (out) fill_scalars(c->h_osum, out);
  if (hs) fill_stats(c->h_hst, hs);
  if (ss) fill_stats(c->h_sst, ss);
  if (t) {
    float m0 = 0.f, m1 = 0.f, m2 = 0.f;
    GADI_CUDA(cudaEventElapsedTime(&m0, c->ev[0], c->ev[1]));
    GADI_CUDA(cudaEventElapsedTime(&m1, c->ev[1], c->ev[2]));
    GADI_CUDA(cudaEventElapsedTime(&m2, c->ev[2], c->ev[3]));
    t->inner_h = m0;
    t->inner_s = m1;
    t->residual = m2;  // fused update + residual + monitor pass
    t->update = 0.0;
    t->monitor = 0.0;
  }
  return 0;
}

int gadi_get_x(gadi_ctx* h, double* x) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  return download(c, c->x[c->xcur], x);
}

int gadi_h_solve(gadi_ctx* h, const double* rhs, double tol, int maxit, double* x, gadi_inner_stats* st) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  GADI_TRY(upload(c, rhs, c->r));
  if (c->rounding == 2) {
    GADI_TRY(exact_h_solve(c, c->r, 1.0, tol, maxit));
    GADI_TRY(download(c, c->ex[EX_Z], x));
  } else {
    c->pred_h = std::min(maxit, 16);
    GADI_TRY(c->vt->h_solve(c, 1.0, tol, maxit));
    GADI_TRY(c->vt->widen(c, c->Z, c->x[c->xcur ^ 1], c->n));
    GADI_TRY(download(c, c->x[c->xcur ^ 1], x));
  }
  if (st) fill_stats(c->h_hst, st);
  return 0;
}

int gadi_s_solve(gadi_ctx* h, const double* rhs, double tol, int maxit, double* x, gadi_inner_stats* st) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  GADI_TRY(upload(c, rhs, c->r));
  if (c->rounding == 2) {
    GADI_TRY(exact_s_solve(c, c->r, 1.0, tol, maxit));
    GADI_TRY(download(c, c->ex[EX_Y], x));
  } else {
    GADI_TRY(c->vt->quantize(c, c->r, c->Z, c->n));
    GADI_TRY(halo(c, c->Z, c->ssz));
    c->pred_s = std::min(maxit, 16);
    GADI_TRY(c->vt->s_solve(c, 1.0, tol, maxit));
    GADI_TRY(c->vt->widen(c, c->Y, c->x[c->xcur ^ 1], c->n));
    GADI_TRY(download(c, c->x[c->xcur ^ 1], x));
  }
  if (st) fill_stats(c->h_sst, st);
  return 0;
}

int gadi_spmv(gadi_ctx* h, int op, int strict, const double* x, double* y) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  if (op < 0 || op > 3) return set_error("op must be 0..3", GADI_ERR_ARG);
  GADI_TRY(upload(c, x, c->r));
  GADI_TRY(halo(c, c->r, 8));
  if (op == 0) {
    norm_state_init<<<1, 1, 0, c->stream>>>(c->nst, 0.0, 1);
    c->launches++;
    GADI_TRY(norm_pass_d<false>(c, c->r, c->x[c->xcur ^ 1]));
  } else {
    GADI_TRY(c->vt->apply(c, op, strict, c->r, c->x[c->xcur ^ 1]));
  }
  GADI_TRY(download(c, c->x[c->xcur ^ 1], y));
  return 0;
}

int gadi_residual(gadi_ctx* h, const double* x, double* r) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  GADI_TRY(upload(c, x, c->x[c->xcur]));
  GADI_TRY(halo(c, c->x[c->xcur], 8));
  GADI_TRY(zero_vec(c, c->Y, c->ssz));
  GADI_TRY(c->vt->outer(c, 1.0, 0));  // x_new = x + 0 ; r = b - A x
  return download(c, c->r, r);
}

int gadi_prof_enable(gadi_ctx* h, int on) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaSetDevice(c->device));
  GADI_CUDA(cudaStreamSynchronize(c->stream));
  prof_collect(c);
  c->prof = on ? 1 : 0;
  for (int k = 0; k < K_NKID; ++k) {
    c->prof_ms[k] = 0.0;
    c->prof_n[k] = 0;
  }
  return 0;
}

int gadi_prof_read(gadi_ctx* h, int kid, double* total_ms, int64_t* launches) {
  Ctx* c = &h->c;
  if (kid < 0 || kid >= K_NKID) return set_error("kernel id out of range", GADI_ERR_ARG);
  GADI_CUDA(cudaStreamSynchronize(c->stream));
  prof_collect(c);
  *total_ms = c->prof_ms[kid];
  *launches = c->prof_n[kid];
  return 0;
}

int gadi_timer_start(gadi_ctx* h) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaEventRecord(c->ev[4], c->stream));
  return 0;
}

int gadi_timer_stop(gadi_ctx* h, double* ms) {
  Ctx* c = &h->c;
  GADI_CUDA(cudaEventRecord(c->ev[5], c->stream));
  GADI_CUDA(cudaEventSynchronize(c->ev[5]));
  float m = 0.f;
  GADI_CUDA(cudaEventElapsedTime(&m, c->ev[4], c->ev[5]));
  *ms = m;
  return 0;
}

int gadi_set_rounding(gadi_ctx* h, int mode, int dot_fmt) {
  Ctx* c = &h->c;
  if (mode < 0 || mode > 2)
    return set_error("rounding mode must be 0 (storage), 1 (reference, fused) or 2 (reference, per operation)",
                     GADI_ERR_ARG);
  if (dot_fmt < GADI_BF16 || dot_fmt > GADI_FP64) return set_error("bad dot format", GADI_ERR_ARG);
  GADI_CUDA(cudaSetDevice(c->device));
  if (mode == 2 && c->comm) return set_error("per-operation reference rounding runs on a single domain", GADI_ERR_UNSUPPORTED);
  if (mode == 1 && c->comm && c->us != GADI_FP64) {
    // the fl_dot trees of the slabs must be whole subtrees of the global tree:
    // 2^k ranks, equal slabs of a power-of-two number of (complex) points
    const int P = c->comm->nranks;
    const long long pts = c->kind == GADI_COMPLEX ? c->n / 2 : c->n;
    const bool pow2 = (P & (P - 1)) == 0 && (pts & (pts - 1)) == 0 && c->gnx % P == 0;
    if (!pow2)
      return set_error("reference rounding on slabs needs 2^k ranks and equal slabs of 2^m points", GADI_ERR_UNSUPPORTED);
  }
  // the fused reference passes cover the stencil families; general CSR
  // operators (and u_s = fp64, whose per-operation emulation is not needed
  // for mode 2) keep the per-operation path
  if (mode == 1 && c->kind == GADI_CSR) mode = c->us == GADI_FP64 ? 0 : 2;
  if (mode == 2 && c->us == GADI_FP64) mode = 0;
  if (mode != c->graph_mode) {  // loop graphs were captured with the other passes
    GADI_CUDA(cudaStreamSynchronize(c->stream));
    if (c->gexec_h) cudaGraphExecDestroy(c->gexec_h);
    if (c->gexec_s) cudaGraphExecDestroy(c->gexec_s);
    if (c->graph_h) cudaGraphDestroy(c->graph_h);
    if (c->graph_s) cudaGraphDestroy(c->graph_s);
    c->gexec_h = c->gexec_s = nullptr;
    c->graph_h = c->graph_s = nullptr;
    c->graph_mode = mode;
  }
  c->rounding = mode;
  c->dot_fmt = dot_fmt;
  c->dk = dot_fmt == GADI_BF16 ? DK_BF16 : (dot_fmt == GADI_FP16 ? DK_F16 : DK_F32);
  if (mode == 2) return exact_alloc(c);
  if (mode == 1 && !c->tree) {
    const long long lv = 2 * ((c->n + TF_BLK - 1) / TF_BLK) + 64;
    GADI_CUDA(cudaMalloc((void**)&c->tree, sizeof(float) * (size_t)(c->n + 64)));
    GADI_CUDA(cudaMalloc((void**)&c->tlvl, sizeof(float) * (size_t)lv));
    GADI_CUDA(cudaMalloc((void**)&c->tticket, sizeof(unsigned int)));
    GADI_CUDA(cudaMalloc((void**)&c->taux, 8 * sizeof(double)));
    GADI_CUDA(cudaMemsetAsync(c->tticket, 0, sizeof(unsigned int), c->stream));
    GADI_CUDA(cudaMemsetAsync(c->taux, 0, 8 * sizeof(double), c->stream));
  }
  return 0;
}

double gadi_last_norm_ms(gadi_ctx* h) { return h->c.last_norm_ms; }
const char* gadi_ctx_comm_kind(gadi_ctx* h) { return h->c.comm ? h->c.comm->kind() : "none"; }
int64_t gadi_kernel_launches(gadi_ctx* h) { return h->c.launches; }

}  // extern "C"
