// Host-side context of one solve: device buffers, stream, device-resident
// scalar states and their pinned host mirrors.  Shared by the per-precision
// engines (engine_*.cu) and the C-ABI (api.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <array>
#include <map>
#include <memory>
#include <string>
#include <vector>
#include "../../include/gadi_b200.h"
#include "comm.h"
#include "passes.cuh"

#ifndef GADI_TRY
#define GADI_TRY(x)      \
  do {                   \
    int rc_ = (x);       \
    if (rc_) return rc_; \
  } while (0)
#endif

namespace gadi {

struct Ctx;

// general-CSR operators (kind GADI_CSR): A, A^T (power iteration), H, S, S^T
enum CsrSlot { CS_A = 0, CS_AT, CS_H, CS_S, CS_ST, CS_N };
struct CsrDev {
  long long* rp = nullptr;  // nrows + 1
  int* ci = nullptr;        // nnz
  double* v64 = nullptr;    // fp64 values (u_s images for H, S, S^T)
  void* vs = nullptr;       // values in u_s storage (H, S, S^T)
  long long nnz = 0;
};

// fp64 work vectors of the reference-rounding inner solvers (exact.cu)
enum ExactBuf { EX_Z = 0, EX_R, EX_P, EX_Q, EX_RB, EX_Y, EX_T0, EX_T1, EX_N };

// Per-u_s-precision entry points (one table per storage type).
struct EngineVT {
  int (*h_solve)(Ctx*, double scale, double tol, int maxit);  // rhs: c->r (fp64)
  int (*s_solve)(Ctx*, double coeff, double tol, int maxit);  // rhs: coeff * c->Z
  int (*outer)(Ctx*, double scale, int has_e);                // x += y/scale ; r ; sums
  int (*apply)(Ctx*, int op, int strict, const double* xdev, double* ydev);
  int (*quantize)(Ctx*, const double* in, void* out, long long n);
  int (*widen)(Ctx*, const void* in, double* out, long long n);
};

struct Ctx {
  gadi_problem_desc d;  // copy (host pointers are not retained)
  int device = 0;
  cudaStream_t stream = nullptr;
  int kind = 0, ndim = 2;
  int nx = 1, ny = 1, nz = 1;  // device grid of this slab (complex: nz = 2 n_g)
  long long n = 0;             // unknowns of this slab
  // slab decomposition: this context owns global planes
  // [x0, x0 + nx) of gnx along the slowest axis; hlo / hhi say whether a
  // neighbour slab exists below / above (one halo plane each, stored just
  // before plane 0 and just after plane nx-1 of every stencil-input vector)
  Comm* comm = nullptr;
  int x0 = 0, gnx = 1, hlo = 0, hhi = 0;
  long long gn = 0;             // global unknowns
  double* gbuf = nullptr;       // gather buffer [nranks][GROW]
  std::vector<void*> raws;      // raw device allocations (vectors with guards/halos)
  struct GVec {
    void* base;
    void* raw;
  };
  std::vector<GVec> gvec;       // the halo'd vectors, in allocation order (peer transport)
  // peer transport (peer.cu): the device-signalled collectives replace the
  // base communicator once every rank has mapped its neighbours' buffers
  std::unique_ptr<Comm> peer;
  Comm* base_comm = nullptr;
  unsigned long long* pflags = nullptr;  // epoch flags written by the peers
  unsigned long long* pcnt = nullptr;    // this rank's epoch counters
  int us = GADI_FP64, u = GADI_FP64, ur = GADI_FP64;
  size_t ssz = 8;  // bytes per u_s element
  int sms = 148;

  // fp64 vectors
  double* b = nullptr;
  double* x[2] = {nullptr, nullptr};
  int xcur = 0;
  double* r = nullptr;
  double* xs = nullptr;
  double* v64 = nullptr;  // crd potential
  double* tmp = nullptr;  // staging for host<->device permutations
  struct HostStager* stager = nullptr;  // pinned host staging (hostcopy.h), large n only
  // u_s vectors (typed by the engine)
  void* R = nullptr;
  void* P[2] = {nullptr, nullptr};
  void* Z = nullptr;
  void* RB = nullptr;
  void* Y = nullptr;
  void* VS = nullptr;  // crd potential in u_s

  double* partials = nullptr;
  int pstride = 0;
  unsigned int* ticket = nullptr;
  InnerState* hst = nullptr;
  InnerState* sst = nullptr;
  OuterSums* osum = nullptr;
  NormState* nst = nullptr;
  // pinned mirrors
  InnerState* h_hst = nullptr;
  InnerState* h_sst = nullptr;
  OuterSums* h_osum = nullptr;
  NormState* h_nst = nullptr;

  cudaEvent_t ev[8] = {};
  int has_exact = 0, ones = 0;
  int pred_h = 4, pred_s = 4;  // iteration-count predictions for launch batching
  long long launches = 0;
  int no_tma = 0;  // force the register-prefetch sweep (testing)
  int waves = 1;      // grid size in waves of resident CTAs (TMA sweep)
  int wavefront = 0;  // wavefront schedule (one CTA per tile) when the tiles fit in one wave
  int batch_cap = 0;  // max inner iterations enqueued per poll (0: the adaptive batch alone)
  int tma2 = 1;       // barrier-free TMA consumers (sweep_tma2.cuh); 0: f-plane form
  int tall = 1;       // GADI_TALL=0: HcgA keeps the default 8-row tiles (passes.cuh GeoT TALL)
  int zlag_on = 0;    // GADI_ZLAG=1: z updated in the next HcgA (engine.cuh zlag_ok)
  // device-driven inner loops: CUDA graphs whose conditional WHILE node
  // repeats two captured iterations until the solve state is done
  int graphs = 1;
  // TMA tensor maps of the 3-D sweeps (tmap.cuh), encoded once per
  // (buffer, element size, box); tmap = 0 (GADI_TMAP=0) keeps row copies
  int tmap = 1;
  // CUtensorMapL2promotion (GADI_TM_PROMO): 0 none, 1 64B (measured best: HcgA 205 -> 197 us vs 256B), 2 128B, 3 256B
  int tm_promo = 1;
  void* tm_encode = nullptr;
  std::map<std::array<long long, 4>, CUtensorMap> tmcache;
  cudaGraph_t graph_h = nullptr, graph_s = nullptr;
  int graph_mode = -1;  // rounding mode the loop graphs were captured with
  cudaGraphExec_t gexec_h = nullptr, gexec_s = nullptr;
  unsigned* wavecnt = nullptr;  // 2 x nx per-plane counters (alternating parity)
  int wpar = 0;
  int min_chunk = 8;  // lower bound on planes per CTA
  int lockstep = 0;   // TMA sweep: align x-chunks across tiles (L2 halo reuse; slower on B200)
  double last_norm_ms = 0.0;

  // live per-kernel timers: event pairs around every launch while enabled,
  // folded into per-kernel totals at each host synchronisation point
  int prof = 0;
  std::vector<cudaEvent_t> evpool;
  std::vector<int> evkid;
  int evused = 0;
  double prof_ms[K_NKID] = {};
  long long prof_n[K_NKID] = {};

  // inner-solver arithmetic: 0 storage model (engine.cuh); 1 the reference's
  // per-operation rounding inside the fused passes (strict.cuh); 2 the same
  // emulation host-driven per operation (exact.cu: CSR operators, and a
  // cross-check of mode 1).  dot_fmt: the reference's fl_dot format.
  int rounding = 0, dot_fmt = GADI_FP64;
  double* ex[EX_N] = {};
  // mode 1: fl_dot leaves, the finisher's level buffer / ticket, the passes'
  // fp64 totals handed to the finisher
  float* tree = nullptr;
  float* tlvl = nullptr;
  unsigned int* tticket = nullptr;
  double* taux = nullptr;
  int dk = 0;  // DotKind of dot_fmt
  CsrDev csr[CS_N];

  CoefT<double> A, AT, H, S, ST;
  CoefT<float> A32;
  EngineVT* vt = nullptr;
};

int set_error(const std::string& msg, int code);

// Per-(kernel, device) launch setup: the dynamic shared-memory opt-in applies
// to the device current when it is set, so it is made once per device (and
// the resulting occupancy cached) under a lock -- slab ranks may run as
// threads of one process (SlabComm.local).
int kernel_occupancy(const void* fn, int device, int nthreads, size_t smem, bool carveout, int* occ);
template <class K>
inline int occupancy_of(Ctx* c, K* kernel, int nthreads, size_t smem, int* occ, bool carveout = false) {
  return kernel_occupancy(reinterpret_cast<const void*>(kernel), c->device, nthreads, smem, carveout, occ);
}

#define GADI_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return ::gadi::set_error(std::string(#call) + ": " + cudaGetErrorString(e_), GADI_ERR_CUDA); \
  } while (0)

inline CoefT<double> coef_of(const gadi_coef& c) {
  CoefT<double> o;
  o.d = c.d;
  for (int i = 0; i < 3; ++i) {
    o.lo[i] = c.lo[i];
    o.up[i] = c.up[i];
  }
  return o;
}
inline CoefT<double> transpose_coef(const CoefT<double>& c) {
  CoefT<double> o = c;
  for (int i = 0; i < 3; ++i) {
    o.lo[i] = c.up[i];
    o.up[i] = c.lo[i];
  }
  return o;
}
template <class CT>
inline CoefT<CT> cast_coef(const CoefT<double>& c) {
  CoefT<CT> o;
  o.d = (CT)c.d;
  for (int i = 0; i < 3; ++i) {
    o.lo[i] = (CT)c.lo[i];
    o.up[i] = (CT)c.up[i];
  }
  return o;
}

// Sweep geometry for a pass with tile TZ x TY.  `slots` = CTAs resident on
// the whole GPU (occupancy x SMs): the x-chunks are sized so the grid is
// about `waves` full waves (long chunks amortise the pipeline fill and the
// two overlap planes of every chunk); 0 keeps the legacy target.
inline SweepGeom make_geom(const Ctx* c, int TZ, int TY, int VZ, long long slots = 0) {
  SweepGeom g;
  g.nx = c->nx;
  g.ny = c->ny;
  g.nz = c->nz;
  g.plane = (long long)c->ny * c->nz;
  g.nzt = (c->nz + TZ - 1) / TZ;
  g.nyt = (c->ny + TY - 1) / TY;
  const long long tiles = (long long)g.nzt * g.nyt;
  long long xc;
  if (slots > 0) {
    const long long want = slots * (long long)c->waves;
    const long long chunks = std::max(1LL, want / tiles);
    xc = (c->nx + chunks - 1) / chunks;
    xc = std::max(xc, std::min<long long>(c->nx, c->min_chunk));
  } else {
    const long long target = (long long)c->sms * 12;
    xc = (c->nx * tiles + target - 1) / target;
  }
  if (xc < 1) xc = 1;
  if (xc > c->nx) xc = c->nx;
  g.xchunk = (int)xc;
  g.pstride = c->pstride;
  g.vec = (c->nz % VZ) == 0 ? 1 : 0;
  g.hlo = c->hlo;
  g.hhi = c->hhi;
  return g;
}
inline int geom_blocks(const SweepGeom& g) {
  return g.nzt * g.nyt * ((g.nx + g.xchunk - 1) / g.xchunk);
}

inline void prof_begin(Ctx* c, int kid) {
  if (!c->prof) return;
  if ((size_t)(2 * c->evused + 2) > c->evpool.size()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      c->evpool.push_back(e);
    }
    c->evkid.resize(c->evpool.size() / 2);
  }
  c->evkid[c->evused] = kid;
  cudaEventRecord(c->evpool[2 * c->evused], c->stream);
}
inline void prof_end(Ctx* c) {
  if (!c->prof) return;
  cudaEventRecord(c->evpool[2 * c->evused + 1], c->stream);
  c->evused++;
}
// call after the stream has been synchronised
inline void prof_collect(Ctx* c) {
  for (int i = 0; i < c->evused; ++i) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->evpool[2 * i], c->evpool[2 * i + 1]) == cudaSuccess) {
      c->prof_ms[c->evkid[i]] += ms;
      c->prof_n[c->evkid[i]] += 1;
    }
  }
  c->evused = 0;
}

int peer_enable(Ctx* c);
int peer_check(Ctx* c);
int peer_export(Ctx* c, void* out, size_t cap, size_t* len);
int peer_import(Ctx* c, const void* blobs, size_t blob_len);

int exact_alloc(Ctx* c);
void exact_free(Ctx* c);
int exact_h_solve(Ctx* c, const double* r64, double scale, double tol, int maxit);
int exact_s_solve(Ctx* c, const double* z, double coeff, double tol, int maxit);

// Halo exchange of one stencil-input vector (no-op on a single domain).
inline int halo(Ctx* c, void* base, size_t esz) {
  if (!c->comm) return 0;
  return c->comm->halo(base, esz * (size_t)c->ny * c->nz, c->nx, c->stream);
}

extern EngineVT engine_bf16, engine_fp16, engine_fp32, engine_fp64;

}  // namespace gadi

struct gadi_ctx {
  gadi::Ctx c;
};
