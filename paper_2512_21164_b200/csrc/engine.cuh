// Per-u_s-precision engine: launches the fused passes of the inner solves and
// of the outer step for one storage type ST, dispatching on the operator
// family (2-D / 3-D real stencil, crd complex).  Instantiated once per ST in
// engine_<st>.cu so the precisions compile in parallel.
//
// Inner Krylov loops run device-driven: every pass reads the solve state
// (alpha, beta, it, done) from device memory and the last CTA of each pass
// writes the next scalars, so the host only enqueues.  Kernels launched after
// convergence exit at their first instruction.  The host enqueues a predicted
// number of iterations (the count of the previous outer step), then polls the
// `done` flag once per batch.
#pragma once
#include <algorithm>
#include "csr.cuh"
#include "ctx.h"

namespace gadi {

// Passes may opt out of the barrier-free consumer form (static TMA2_OK =
// false): the fp64 outer pass measured faster with the f-plane form.
template <class P, class = void> struct TmaForm2 : std::true_type {};
template <class P> struct TmaForm2<P, std::void_t<decltype(P::TMA2_OK)>> : std::bool_constant<P::TMA2_OK> {};

// True when every input row of pass P starts 16-byte aligned (TMA path).
// One 3-D tensor map over a vector of esz-byte elements laid out [x][y][z]
// (planes -hlo .. nx+hhi-1 of a slab context's allocation), box {bw, bh, 1}.
// Cached per (pointer, esz, box); false if the driver entry point or the
// encoding is unavailable (the caller keeps the row-copy producer).
inline bool tm_map(Ctx* c, const void* ptr, int esz, int bw, int bh, CUtensorMap* out) {
  const std::array<long long, 4> key{(long long)(uintptr_t)ptr, esz, bw, bh};
  auto itc = c->tmcache.find(key);
  if (itc != c->tmcache.end()) {
    *out = itc->second;
    return true;
  }
  if (!c->tm_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
      cudaGetLastError();
      c->tmap = 0;
      return false;
    }
    c->tm_encode = fn;
  }
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  const CUtensorMapDataType dt = esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                 : esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  const long long plane = (long long)c->ny * c->nz;
  const int hlo = c->hlo, hhi = c->hhi;
  const char* base = static_cast<const char*>(ptr) - (long long)hlo * plane * esz;
  const cuuint64_t dims[3] = {(cuuint64_t)c->nz, (cuuint64_t)c->ny, (cuuint64_t)(c->nx + hlo + hhi)};
  const cuuint64_t strides[2] = {(cuuint64_t)c->nz * esz, (cuuint64_t)plane * esz};
  const cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMap m;
  const CUresult r = reinterpret_cast<EncodeFn>(c->tm_encode)(
      &m, dt, 3, const_cast<char*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, (CUtensorMapL2promotion)c->tm_promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  c->tmcache.emplace(key, m);
  *out = m;
  return true;
}

template <class P, int TM>
inline bool tm_fill(Ctx* c, const P& p, TmapSet& tm) {
  using TS = TmaShape2<P, TM>;
  using BX = TmBox<P, TmaShape<P>>;
  if (c->ndim != 3 || ((long long)c->ny * c->nz) % 16) return false;
  for (int j = 0; j < P::NIN; ++j) {
    if (!p.in_active(j) || (TM != 1 && TM != 3)) continue;
    if ((uintptr_t)p.in_ptr(j) % 16 || !tm_map(c, p.in_ptr(j), P::in_esz(j), BX::BW(j), TS::TY + 2, &tm.in[j]))
      return false;
  }
  for (int j = 0; j < P::NE && (TM == 2 || TM == 3); ++j)
    if ((uintptr_t)p.epi_ptr(j) % 16 || !tm_map(c, p.epi_ptr(j), P::epi_esz(j), TS::TZ, TS::TY, &tm.epi[j]))
      return false;
  return true;
}

template <class P>
inline bool tma_aligned(const Ctx* c) {
  if (!P::TMA_OK || c->no_tma) return false;
  for (int j = 0; j < P::NIN; ++j)
    if (((long long)c->nz * P::in_esz(j)) % 16) return false;
  for (int j = 0; j < P::NE; ++j)
    if (((long long)c->nz * P::epi_esz(j)) % 16) return false;
  return (c->nz % P::VZ) == 0;
}

// Z-lag H-CG (passes.cuh HcgA): compiled in, selected per process by the
// environment (GADI_ZLAG=1) when the pass runs on the barrier-free TMA form.
// Measured at 512^3 bf16 (profiles/ab_zlag_r2.jsonl): HcgA 204 -> 278 us,
// HcgB 256 -> 190 us, one H-CG iteration 460 -> 468 us -- off by default.
#ifndef GADI_TALL_ROWCOPY_OK
#define GADI_TALL_ROWCOPY_OK 0  // let 16-row passes use the row-copy producer (bitwise the boxes: scripts/tall_diag2.py)
#endif
template <class P>
inline bool zlag_ok(const Ctx* c) {
  if (!c->zlag_on) return false;
  return tma_aligned<P>(c) && c->tma2 != 0 && TmaForm2<P>::value;
}

// Slab decomposition: after a reducing pass, gather every rank's totals and
// run the pass's scalar recurrence on them (finalize_kernel).
template <class P>
inline int post_reduce(Ctx* c, const P& p) {
  if constexpr (TreeSlot<P>::value >= 0) {
    if (p.tout.tree) return 0;  // reference rounding: launch_tree gathers after its finisher
  }
  if constexpr (P::HAS_RED) {
    if (c->comm) {
      GADI_TRY(c->comm->gather(c->gbuf, P::NR, c->stream));
      finalize_kernel<P><<<1, 1, 0, c->stream>>>(p, c->gbuf, c->comm->nranks, GROW);
      c->launches++;
      GADI_CUDA(cudaGetLastError());
    }
  }
  return 0;
}

inline double* defer_row(Ctx* c) { return c->comm ? c->gbuf + (size_t)c->comm->rank * GROW : nullptr; }

inline int ilog2(long long v) {
  int l = 0;
  while ((1LL << (l + 1)) <= v) ++l;
  return l;
}

// Reference rounding: after a pass that wrote fl_dot leaves, sum them and run
// its scalar recurrence (tree_finish_kernel, strict.cuh).
template <class P>
inline int launch_tree(Ctx* c, const P& p, long long leaves) {
  auto finish = [&](const float* lv, long long m, int slot) -> int {
    const long long nb = std::max(1LL, (m + TF_BLK - 1) / TF_BLK);
    prof_begin(c, K_TREE);
    tree_finish_kernel<P><<<(int)nb, TF_NT, 0, c->stream>>>(p, lv, m, c->tlvl, c->tticket, slot);
    prof_end(c);
    c->launches++;
    GADI_CUDA(cudaGetLastError());
    return 0;
  };
  if (!c->comm) return finish(c->tree, leaves, -1);
  // slabs: this rank's subtree(s) into its gather row, then the tree across
  // ranks (complex: the real and imaginary halves are separate subtrees)
  const bool cplx = p.tout.cm > 0;
  if (cplx) {
    GADI_TRY(finish(c->tree, leaves / 2, P::TS));
    GADI_TRY(finish(c->tree + leaves / 2, leaves / 2, P::NR));
  } else {
    GADI_TRY(finish(c->tree, leaves, P::TS));
  }
  GADI_TRY(c->comm->gather(c->gbuf, P::NR + 1, c->stream));
  tree_combine_kernel<P><<<1, 1, 0, c->stream>>>(p, c->gbuf, c->comm->nranks, GROW, cplx ? 1 : 0);
  c->launches++;
  GADI_CUDA(cudaGetLastError());
  return 0;
}
template <class P>
inline void tree_setup(Ctx* c, P& p) {
  p.tout = TreeOut{nullptr, -1, 0, nullptr, 0};
  if constexpr (TreeSlot<P>::value >= 0)
    p.tout = TreeOut{c->tree, -1, c->dk, c->taux, c->kind == GADI_COMPLEX ? c->n / 2 : 0};
}
// leaves of one dot: one per element, else one per aligned block (two per
// block of an interleaved complex vector: the real and imaginary halves)
inline long long tree_leaves(const Ctx* c, const TreeOut& t) {
  if (t.tlog < 0) return c->n;
  if (t.cm) return 2 * (t.cm >> (t.tlog - 1));
  return (c->n + (1LL << t.tlog) - 1) >> t.tlog;
}

// Split-phase halo of the vector a pass produces (peer transport): before
// the pass the neighbours' halo slots are claimed and their plane pointers
// go into the pass (HaloOut); after it, halo_end publishes the data.  Other
// transports: the ordinary halo exchange after the pass.
inline bool halo_begin(Ctx* c, void* base, size_t esz, HaloOut& h) {
  h = HaloOut{nullptr, nullptr};
  if (!c->comm) return false;
  return c->comm->halo_begin(base, esz * (size_t)c->ny * c->nz, c->nx, &h.lo, &h.hi, c->stream);
}
inline int halo_end(Ctx* c, void* base, size_t esz, bool fused) {
  if (!c->comm) return 0;
  if (fused) return c->comm->halo_end(base, c->stream);
  return halo(c, base, esz);
}

template <class P>
inline int launch_sweep(Ctx* c, P& p, const HaloOut* hout = nullptr) {
  using S = SweepShape<P>;
  p.hout = hout ? *hout : HaloOut{nullptr, nullptr};
  p.partials = c->partials;
  p.ticket = c->ticket;
  p.defer = defer_row(c);
  p.wave = p.wave_clear = nullptr;
  p.wlead = 0;
  tree_setup(c, p);
  if (tma_aligned<P>(c)) {
    // one resident wave of CTAs; the kernel splits the (tile, plane) units
    // evenly among them (SegIter).  Barrier-free consumers (sweep_tma2.cuh)
    // unless GADI_TMA2=0 selects the f-plane form (sweep_tma.cuh).
    const bool v2 = c->tma2 != 0 && TmaForm2<P>::value;
    if constexpr (HasSide<P>::value) {
      if (!v2) return set_error("z-lag pass off the barrier-free sweep form", GADI_ERR_ARG);
    }
    if constexpr (P::TALL != 0) {
      if (!v2) return set_error("16-row tile pass off the barrier-free sweep form", GADI_ERR_ARG);
    }
    // tensor-map producer for the 3-D barrier-free passes (tmap.cuh): mode 1
    // boxes for two haloed inputs, mode 2 boxes for the epilogue inputs
    constexpr int TMM = TmaTm<P>::value ? (TmaTmBoth<P>::value ? 3 : 1) : (TmaTmEpi<P>::value ? 2 : 0);
    TmapSet tm;
    tm.ok = 0;
    if constexpr (TMM != 0) {
      if (v2 && c->tmap) tm.ok = tm_fill<P, TMM>(c, p, tm) ? 1 : 0;
    }
    if constexpr (P::TALL != 0 && !GADI_TALL_ROWCOPY_OK) {
      // 16-row passes are measured with their tensor maps only (the row-copy
      // producer issues 2 x 18 copies per stage from one warp)
      if (!tm.ok) return set_error("16-row tile pass without its tensor maps", GADI_ERR_ARG);
    }
    const size_t smem = v2 ? (tm.ok ? TmaShape2<P, TMM>::SMEM : TmaShape2<P>::SMEM) : TmaShape<P>::SMEM;
    const int NTH = v2 ? Tma2Threads<P>::value : TmaThreads<P>::NTOT;
    int occ = 1;
    if (v2 && tm.ok) {
      if constexpr (TMM != 0) GADI_TRY(occupancy_of(c, sweep_tma2_kernel<P, TMM>, NTH, smem, &occ));
    } else if (v2) {
      GADI_TRY(occupancy_of(c, sweep_tma2_kernel<P, 0>, NTH, smem, &occ));
    } else {
      GADI_TRY(occupancy_of(c, sweep_tma_kernel<P>, NTH, smem, &occ));
    }
    // reference rounding on the barrier-free form: one fl_dot leaf per
    // aligned block of G = min(2^v2(nz), 32 VZ) elements (strict.cuh)
    if constexpr (TreeSlot<P>::value >= 0) {
      if (v2) {
        const int a = c->nz & -c->nz, gb = std::min(a, 32 * P::VZ);
        if (gb >= P::VZ) p.tout.tlog = ilog2(gb);
      }
    }
    p.g = make_geom(c, S::TZ, S::TY, P::VZ, (long long)occ * c->sms);
    const long long tiles = (long long)p.g.nzt * p.g.nyt;
    const long long units = tiles * p.g.nx;
    const long long slots = (long long)occ * c->sms * c->waves;
    long long nbl = std::min(units, slots);
    if (c->wavefront && c->wavecnt && tiles <= (long long)occ * c->sms && c->nx >= 4) {
      nbl = tiles;  // one CTA per tile through all planes (SegIter with nblocks == tiles)
      p.wave = c->wavecnt + (size_t)c->wpar * c->nx;
      p.wave_clear = c->wavecnt + (size_t)(c->wpar ^ 1) * c->nx;
      p.wlead = (v2 ? (tm.ok ? TmaShape2<P, TMM>::NST : TmaShape2<P>::NST) : TmaShape<P>::NST) + 4;
      c->wpar ^= 1;
    }
    if (c->lockstep && tiles <= slots) {
      // every tile split into the same k x-chunks: CTAs on neighbouring tiles
      // sweep the same planes at the same time, so y-halo rows hit in L2
      const long long k = std::max(1LL, std::min(slots / tiles, (long long)p.g.nx / std::max(1, c->min_chunk)));
      nbl = tiles * k;
    }
    const int nb = (int)nbl;
    if (nb > c->pstride) return set_error("sweep grid exceeds partials buffer", GADI_ERR_ARG);
    prof_begin(c, P::KID);
    if (v2 && tm.ok) {
      if constexpr (TMM != 0) sweep_tma2_kernel<P, TMM><<<nb, NTH, smem, c->stream>>>(p, tm);
    } else if (v2) {
      sweep_tma2_kernel<P, 0><<<nb, NTH, smem, c->stream>>>(p, TmapNone{0});
    }
    else
      sweep_tma_kernel<P><<<nb, NTH, smem, c->stream>>>(p);
    prof_end(c);
  } else {
    if constexpr (HasSide<P>::value) return set_error("z-lag pass off the TMA sweep path", GADI_ERR_ARG);
    if constexpr (P::TALL != 0) return set_error("16-row tile pass off the TMA sweep path", GADI_ERR_ARG);
    p.g = make_geom(c, S::TZ, S::TY, P::VZ);
    const int nb = geom_blocks(p.g);
    if (nb > c->pstride) return set_error("sweep grid exceeds partials buffer", GADI_ERR_ARG);
    const size_t smem = S::SMEM;
    if (smem > 48 * 1024) {
      int occ = 1;
      GADI_TRY(occupancy_of(c, sweep_kernel<P>, P::NT, smem, &occ));
    }
    prof_begin(c, P::KID);
    sweep_kernel<P><<<nb, P::NT, smem, c->stream>>>(p);
    prof_end(c);
  }
  c->launches++;
  GADI_CUDA(cudaGetLastError());
  GADI_TRY(post_reduce(c, p));
  if constexpr (TreeSlot<P>::value >= 0) GADI_TRY(launch_tree(c, p, tree_leaves(c, p.tout)));
  return 0;
}

template <class P>
inline int launch_pw(Ctx* c, P& p) {
  p.n = c->n;
  p.partials = c->partials;
  p.ticket = c->ticket;
  p.pstride = c->pstride;
  p.defer = defer_row(c);
  tree_setup(c, p);
  if constexpr (TreeSlot<P>::value >= 0) {
    p.tout.tlog = ilog2(32 * P::VZ);
    if (p.tout.cm && p.tout.cm % (16 * P::VZ)) p.tout.tlog = -1;  // halves not block-aligned
  }
  const long long chunks = (c->n + (long long)PW_NT * P::VZ - 1) / ((long long)PW_NT * P::VZ);
  int nb = (int)std::min<long long>(chunks, (long long)c->sms * 8);
  nb = std::max(nb, 1);
  prof_begin(c, P::KID);
  pointwise_kernel<P><<<nb, PW_NT, 0, c->stream>>>(p);
  prof_end(c);
  c->launches++;
  GADI_CUDA(cudaGetLastError());
  GADI_TRY(post_reduce(c, p));
  if constexpr (TreeSlot<P>::value >= 0) GADI_TRY(launch_tree(c, p, tree_leaves(c, p.tout)));
  return 0;
}


// Poll the device state of an inner solve.
inline int poll_state(Ctx* c, InnerState* dev, InnerState* host) {
  GADI_CUDA(cudaMemcpyAsync(host, dev, sizeof(InnerState), cudaMemcpyDeviceToHost, c->stream));
  GADI_CUDA(cudaStreamSynchronize(c->stream));
  prof_collect(c);
  return peer_check(c);
}

// Enqueue inner iterations in batches (the previous solve's count + 1 first,
// then a quarter of it), polling the device `done` flag once per batch.
// iter(k) enqueues iteration k; passes launched after convergence are no-ops.
// A batch cap (GADI_BATCH_CAP) bounds the no-op launches enqueued past
// convergence when the count drops between solves, at one poll per cap.
template <class F>
inline int run_batched(Ctx* c, InnerState* dev, InnerState* host, int& pred, int maxit, F&& iter) {
  auto capped = [&](int b) { return c->batch_cap > 0 ? std::min(b, c->batch_cap) : b; };
  int launched = 0, batch = capped(std::max(1, pred + 1));
  bool polled = false;
  while (launched < maxit) {
    const int nb = std::min(batch, maxit - launched);
    for (int j = 0; j < nb; ++j) GADI_TRY(iter(launched + j));
    launched += nb;
    GADI_TRY(poll_state(c, dev, host));
    polled = true;
    if (host->done) break;
    batch = capped(std::max(2, pred / 4 + 1));
  }
  if (!polled) GADI_TRY(poll_state(c, dev, host));
  pred = host->it;
  return 0;
}

// ---------------------------------------------------------------- device-driven loops
// The inner solvers' scalars and stop tests already live on the device; a
// CUDA graph with a conditional WHILE node removes the host from the loop:
// its body is two captured iterations followed by a one-thread kernel that
// sets the loop condition from the solve state.  Used on a single domain when
// the per-launch timers are off; the host enqueues the graph once per inner
// solve and reads the state once at the end.
static __global__ void loop_cond_kernel(cudaGraphConditionalHandle h, const InnerState* st) {
  cudaGraphSetConditional(h, st->done ? 0u : 1u);
}

// graph loops need collectives without the host: a single domain, or slabs on
// the peer transport (peer.cu)
inline bool use_graphs(const Ctx* c) { return c->graphs && (!c->comm || c->comm->device_only()) && !c->prof; }

// Build (once per context) the graph whose WHILE body is `body` (which
// enqueues the kernels of two iterations on c->stream).
template <class F>
inline int build_loop_graph(Ctx* c, cudaGraph_t& graph, cudaGraphExec_t& exec, const InnerState* st, F&& body) {
  GADI_CUDA(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle h;
  GADI_CUDA(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  GADI_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &np));
  cudaGraph_t bodyg = np.conditional.phGraph_out[0];
  const long long launches = c->launches;
  GADI_CUDA(cudaStreamBeginCaptureToGraph(c->stream, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  int rc = body();
  loop_cond_kernel<<<1, 1, 0, c->stream>>>(h, st);
  cudaGraph_t captured = nullptr;
  const cudaError_t e = cudaStreamEndCapture(c->stream, &captured);
  c->launches = launches;  // captured, not executed
  if (rc) return rc;
  GADI_CUDA(e);
  GADI_CUDA(cudaGraphInstantiate(&exec, graph, 0));
  return 0;
}

// Run the remaining iterations of an inner solve (iteration 0 already
// enqueued) through the loop graph, then read the state.  `kernels_per_iter`
// counts launches for the statistics.
inline int run_loop_graph(Ctx* c, cudaGraphExec_t exec, InnerState* dev, InnerState* host, int& pred,
                          int kernels_per_iter) {
  GADI_CUDA(cudaGraphLaunch(exec, c->stream));
  GADI_TRY(poll_state(c, dev, host));
  pred = host->it;
  const long long pairs = std::max(1, (host->it - 1 + 1) / 2);
  c->launches += pairs * (2LL * kernels_per_iter + 1);
  return 0;
}

template <class ST>
struct Engine {
  typedef typename CTOf<ST>::type CT;

  // ------------------------------------------------------------ general CSR (csr.cuh)
  static CsrT<ST> csr_s(const Ctx* c, int slot) {
    return CsrT<ST>{c->csr[slot].rp, c->csr[slot].ci, (const ST*)c->csr[slot].vs};
  }
  static CsrT<double> csr_d(const Ctx* c, int slot) {
    return CsrT<double>{c->csr[slot].rp, c->csr[slot].ci, c->csr[slot].v64};
  }
  static int h_solve_csr(Ctx* c, double scale, double tol, int maxit) {
    HcgInit<ST> hi;
    hi.r64 = c->r;
    hi.rs = (ST*)c->R;
    hi.z = (ST*)c->Z;
    hi.st = c->hst;
    hi.scale = scale;
    hi.tol = tol;
    hi.maxit = maxit;
    GADI_TRY(launch_pw(c, hi));
    const CsrT<ST> H = csr_s(c, CS_H);
    ST* p = (ST*)c->P[0];
    ST* q = (ST*)c->P[1];
    return run_batched(c, c->hst, c->h_hst, c->pred_h, maxit, [&](int k) {
      CsrDir<ST> d;
      d.st = c->hst;
      d.f = (const ST*)c->R;
      d.p = p;
      d.first = k == 0;
      GADI_TRY(launch_pw(c, d));
      CsrSpmv<ST, 0> s;
      s.st = c->hst;
      s.m = H;
      s.x = p;
      s.q = q;
      GADI_TRY(launch_pw(c, s));
      CsrUpdate<ST, 0> u;
      u.st = c->hst;
      u.p = p;
      u.q = q;
      u.u = (ST*)c->Z;
      u.r = (ST*)c->R;
      return launch_pw(c, u);
    });
  }
  static int s_solve_csr(Ctx* c, double coeff, double tol, int maxit) {
    CsrCgnrRhs<ST> rh;
    rh.z = (const ST*)c->Z;
    rh.r = (ST*)c->R;
    rh.y = (ST*)c->Y;
    rh.coeff = (CT)coeff;
    GADI_TRY(launch_pw(c, rh));
    const CsrT<ST> S = csr_s(c, CS_S), STm = csr_s(c, CS_ST);
    CsrSpmv<ST, 3> in;
    in.st = c->sst;
    in.m = STm;
    in.x = (const ST*)c->R;
    in.q = (ST*)c->RB;
    in.tol = tol;
    in.maxit = maxit;
    GADI_TRY(launch_pw(c, in));
    ST* p = (ST*)c->P[0];
    ST* w = (ST*)c->P[1];
    return run_batched(c, c->sst, c->h_sst, c->pred_s, maxit, [&](int k) {
      CsrDir<ST> d;
      d.st = c->sst;
      d.f = (const ST*)c->RB;
      d.p = p;
      d.first = k == 0;
      GADI_TRY(launch_pw(c, d));
      CsrSpmv<ST, 1> s;
      s.st = c->sst;
      s.m = S;
      s.x = p;
      s.q = w;
      GADI_TRY(launch_pw(c, s));
      CsrUpdate<ST, 1> u;
      u.st = c->sst;
      u.p = p;
      u.q = w;
      u.u = (ST*)c->Y;
      u.r = (ST*)c->R;
      GADI_TRY(launch_pw(c, u));
      CsrSpmv<ST, 2> t;
      t.st = c->sst;
      t.m = STm;
      t.x = (const ST*)c->R;
      t.q = (ST*)c->RB;
      return launch_pw(c, t);
    });
  }
  template <int UR, bool HAS_E>
  static int outer_csr_t(Ctx* c, double scale) {
    CsrOuterX<ST> ox;
    ox.x = c->x[c->xcur];
    ox.y = (const ST*)c->Y;
    ox.xout = c->x[c->xcur ^ 1];
    ox.scale = scale;
    ox.inv_scale = 1.0 / scale;
    ox.u32 = (c->u != GADI_FP64 && c->u != GADI_FP64X2) ? 1 : 0;
    GADI_TRY(launch_pw(c, ox));
    CsrOuterR<UR, HAS_E> o;
    o.A = csr_d(c, CS_A);
    o.x = c->x[c->xcur ^ 1];
    o.xs = c->xs;
    o.b = c->b;
    o.r = c->r;
    o.out = c->osum;
    o.ones = c->ones;
    GADI_TRY(launch_pw(c, o));
    c->xcur ^= 1;
    return 0;
  }
  static int outer_csr(Ctx* c, double scale, int has_e) {
    const int ur = c->ur == GADI_FP64 ? 0 : (c->ur == GADI_FP64X2 ? 2 : 1);
    if (ur == 0) return has_e ? outer_csr_t<0, true>(c, scale) : outer_csr_t<0, false>(c, scale);
    if (ur == 1) return has_e ? outer_csr_t<1, true>(c, scale) : outer_csr_t<1, false>(c, scale);
    return has_e ? outer_csr_t<2, true>(c, scale) : outer_csr_t<2, false>(c, scale);
  }
  static int apply_csr(Ctx* c, int op, int strict, const double* in, double* out) {
    const int slot = op == 1 ? CS_H : (op == 2 ? CS_S : CS_ST);
    if (strict) {
      CsrApply<ST, true> a;
      a.m = csr_d(c, slot);
      a.in = in;
      a.outv = out;
      return launch_pw(c, a);
    }
    CsrApply<ST, false> a;
    a.m = csr_d(c, slot);
    a.in = in;
    a.outv = out;
    return launch_pw(c, a);
  }

  // ------------------------------------------------------------ H-solve (CG)
  // RF: the reference's per-operation rounding (strict.cuh), else the storage model
  template <int DIM, int ZS, bool RF>
  static int h_solve_t(Ctx* c, double scale, double tol, int maxit) {
    typedef GeoT<ST, DIM, ZS> G;
    HcgInit<ST, RF> hi;
    hi.r64 = c->r;
    hi.rs = (ST*)c->R;
    hi.z = (ST*)c->Z;
    hi.st = c->hst;
    hi.scale = scale;
    hi.tol = tol;
    hi.maxit = maxit;
    GADI_TRY(launch_pw(c, hi));
    GADI_TRY(halo(c, c->R, sizeof(ST)));
    // z-lag (passes.cuh HcgA): only where every H-CG pass runs the barrier-free form
    // HcgA on 16-row tiles (passes.cuh GeoT TALL) where it gets the tensor-map producer
    typedef GeoT<ST, DIM, ZS, 1> GT;
    const bool tall = DIM == 3 && c->tall && (c->tmap || GADI_TALL_ROWCOPY_OK) && c->tma2 != 0 && tma_aligned<HcgA<GT>>(c) &&
                      ((long long)c->ny * c->nz) % 16 == 0;  // tm_fill's plane-stride condition
    if (zlag_ok<HcgA<G, false, RF, true>>(c) && zlag_ok<HcgB<G, RF, true>>(c))
      return tall ? h_loop_t<G, GT, RF, true>(c, maxit) : h_loop_t<G, G, RF, true>(c, maxit);
    return tall ? h_loop_t<G, GT, RF, false>(c, maxit) : h_loop_t<G, G, RF, false>(c, maxit);
  }
  // GA: the geometry of the HcgA passes (G or its 16-row TALL form);
  // GADI_TALL_HCGB = 1 (experiment) runs HcgB on it too
#ifndef GADI_TALL_HCGB
#define GADI_TALL_HCGB 0
#endif
  template <class G, class GA, bool RF, bool ZL>
  static int h_loop_t(Ctx* c, int maxit) {
    using GB = typename std::conditional<GADI_TALL_HCGB != 0, GA, G>::type;
    const CoefT<CT> H = cast_coef<CT>(c->H);
    ST* P[2] = {(ST*)c->P[0], (ST*)c->P[1]};
    auto iter = [&](int k) -> int {
        HaloOut ho;
        bool hf = false;
        if (k == 0) {
          HcgA<GA, true, RF> a;
          a.st = c->hst;
          a.r = (const ST*)c->R;
          a.pin = P[0];
          a.pout = P[1];
          a.H = H;
          hf = halo_begin(c, P[1], sizeof(ST), ho);
          GADI_TRY(launch_sweep(c, a, &ho));
        } else {
          HcgA<GA, false, RF, ZL> a;
          a.st = c->hst;
          a.r = (const ST*)c->R;
          a.pin = P[k & 1];
          a.pout = P[(k + 1) & 1];
          a.z = (ST*)c->Z;
          a.H = H;
          hf = halo_begin(c, P[(k + 1) & 1], sizeof(ST), ho);
          GADI_TRY(launch_sweep(c, a, &ho));
        }
        GADI_TRY(halo_end(c, P[(k + 1) & 1], sizeof(ST), hf));
        HcgB<GB, RF, ZL> b;
        b.st = c->hst;
        b.p = P[(k + 1) & 1];
        b.z = (ST*)c->Z;
        b.r = (ST*)c->R;
        b.H = H;
        hf = halo_begin(c, c->R, sizeof(ST), ho);
        GADI_TRY(launch_sweep(c, b, &ho));
        return halo_end(c, c->R, sizeof(ST), hf);
    };
    if (use_graphs(c) && maxit > 1) {
      GADI_TRY(iter(0));
      if (!c->gexec_h)
        GADI_TRY(build_loop_graph(c, c->graph_h, c->gexec_h, c->hst, [&]() -> int {
          GADI_TRY(iter(1));
          return iter(2);
        }));
      GADI_TRY(run_loop_graph(c, c->gexec_h, c->hst, c->h_hst, c->pred_h, 2));
    } else {
      GADI_TRY(run_batched(c, c->hst, c->h_hst, c->pred_h, maxit, iter));
    }
    if constexpr (ZL) {
      HcgZFinal<ST, RF> zf;
      zf.st = c->hst;
      zf.P0 = P[0];
      zf.P1 = P[1];
      zf.z = (ST*)c->Z;
      GADI_TRY(launch_pw(c, zf));
    }
    return halo(c, c->Z, sizeof(ST));  // z is the stencil input of the CGNR init
  }

  // ------------------------------------------------------------ S-solve (CGNR)
  template <int DIM, bool RF>
  static int s_solve_real(Ctx* c, double coeff, double tol, int maxit) {
    typedef GeoT<ST, DIM, 1> G;
    const CoefT<CT> S = cast_coef<CT>(c->S), STc = cast_coef<CT>(c->ST);
    CgnrInit<G, RF> ci;
    ci.st = c->sst;
    ci.z = (const ST*)c->Z;
    ci.r = (ST*)c->R;
    ci.rbar = (ST*)c->RB;
    ci.y = (ST*)c->Y;
    ci.ST_ = STc;
    ci.coeff = (CT)coeff;
    ci.tol = tol;
    ci.maxit = maxit;
    GADI_TRY(launch_sweep(c, ci));
    GADI_TRY(halo(c, c->RB, sizeof(ST)));
    ST* P[2] = {(ST*)c->P[0], (ST*)c->P[1]};
    auto iter = [&](int k) -> int {
        HaloOut ho;
        bool hf = false;
        if (k == 0) {
          CgnrP1<G, true, RF> p1;
          p1.st = c->sst;
          p1.rbar = (const ST*)c->RB;
          p1.pin = P[0];
          p1.pout = P[1];
          p1.S = S;
          hf = halo_begin(c, P[1], sizeof(ST), ho);
          GADI_TRY(launch_sweep(c, p1, &ho));
        } else {
          CgnrP1<G, false, RF> p1;
          p1.st = c->sst;
          p1.rbar = (const ST*)c->RB;
          p1.pin = P[k & 1];
          p1.pout = P[(k + 1) & 1];
          p1.S = S;
          hf = halo_begin(c, P[(k + 1) & 1], sizeof(ST), ho);
          GADI_TRY(launch_sweep(c, p1, &ho));
        }
        GADI_TRY(halo_end(c, P[(k + 1) & 1], sizeof(ST), hf));
        CgnrP2<G, RF> p2;
        p2.st = c->sst;
        p2.p = P[(k + 1) & 1];
        p2.y = (ST*)c->Y;
        p2.r = (ST*)c->R;
        p2.S = S;
        hf = halo_begin(c, c->R, sizeof(ST), ho);
        GADI_TRY(launch_sweep(c, p2, &ho));
        GADI_TRY(halo_end(c, c->R, sizeof(ST), hf));
        CgnrP3<G, RF> p3;
        p3.st = c->sst;
        p3.r = (const ST*)c->R;
        p3.rbar = (ST*)c->RB;
        p3.ST_ = STc;
        hf = halo_begin(c, c->RB, sizeof(ST), ho);
        GADI_TRY(launch_sweep(c, p3, &ho));
        return halo_end(c, c->RB, sizeof(ST), hf);
    };
    if (use_graphs(c) && maxit > 1) {
      GADI_TRY(iter(0));
      if (!c->gexec_s)
        GADI_TRY(build_loop_graph(c, c->graph_s, c->gexec_s, c->sst, [&]() -> int {
          GADI_TRY(iter(1));
          return iter(2);
        }));
      GADI_TRY(run_loop_graph(c, c->gexec_s, c->sst, c->h_sst, c->pred_s, 3));
    } else {
      GADI_TRY(run_batched(c, c->sst, c->h_sst, c->pred_s, maxit, iter));
    }
    return halo(c, c->Y, sizeof(ST));  // y is a field input of the outer pass
  }

  template <bool RF>
  static int s_solve_cplx(Ctx* c, double coeff, double tol, int maxit) {
    const CT al = (CT)c->d.alpha_s;
    CInit<ST, RF> ci;
    ci.vs = (const ST*)c->VS;
    ci.al = al;
    ci.z = (const ST*)c->Z;
    ci.r = (ST*)c->R;
    ci.y = (ST*)c->Y;
    ci.st = c->sst;
    ci.coeff = (CT)coeff;
    ci.tol = tol;
    ci.maxit = maxit;
    GADI_TRY(launch_pw(c, ci));
    auto iter = [&](int) -> int {
        CP1<ST, RF> p1;
        p1.vs = (const ST*)c->VS;
        p1.al = al;
        p1.r = (const ST*)c->R;
        p1.p = (ST*)c->P[0];
        p1.st = c->sst;
        GADI_TRY(launch_pw(c, p1));
        CP2<ST, RF> p2;
        p2.vs = (const ST*)c->VS;
        p2.al = al;
        p2.p = (const ST*)c->P[0];
        p2.y = (ST*)c->Y;
        p2.r = (ST*)c->R;
        p2.st = c->sst;
        return launch_pw(c, p2);
    };
    if (use_graphs(c) && maxit > 1) {
      GADI_TRY(iter(0));
      if (!c->gexec_s)
        GADI_TRY(build_loop_graph(c, c->graph_s, c->gexec_s, c->sst, [&]() -> int {
          GADI_TRY(iter(1));
          return iter(2);
        }));
      GADI_TRY(run_loop_graph(c, c->gexec_s, c->sst, c->h_sst, c->pred_s, 2));
    } else {
      GADI_TRY(run_batched(c, c->sst, c->h_sst, c->pred_s, maxit, iter));
    }
    return halo(c, c->Y, sizeof(ST));
  }

  // ------------------------------------------------------------ outer pass
  template <int DIM, int ZS, int UR, bool HAS_E, bool CPLX>
  static int outer_t(Ctx* c, double scale) {
    // GADI_TALL_OUTER = 1 (experiment): the outer pass on 16-row tiles
#ifndef GADI_TALL_OUTER
#define GADI_TALL_OUTER 0
#endif
    if constexpr (GADI_TALL_OUTER && DIM == 3) {
      typedef GeoT<double, DIM, ZS, 1> GT;
      if (c->tall && c->tmap && c->tma2 != 0 && tma_aligned<Outer<GT, ST, UR, HAS_E, CPLX>>(c) &&
          ((long long)c->ny * c->nz) % 16 == 0)
        return outer_g<GT, UR, HAS_E, CPLX>(c, scale);
    }
    return outer_g<GeoT<double, DIM, ZS>, UR, HAS_E, CPLX>(c, scale);
  }
  template <class G, int UR, bool HAS_E, bool CPLX>
  static int outer_g(Ctx* c, double scale) {
    Outer<G, ST, UR, HAS_E, CPLX> o;
    o.x = c->x[c->xcur];
    o.y = (const ST*)c->Y;
    o.xs = c->xs;
    o.b = c->b;
    o.v = c->v64;
    o.xout = c->x[c->xcur ^ 1];
    o.r = c->r;
    o.out = c->osum;
    o.A = c->A;
    o.A32 = c->A32;
    o.scale = scale;
    o.inv_scale = 1.0 / scale;
    o.ones = c->ones;
    o.u32 = (c->u != GADI_FP64 && c->u != GADI_FP64X2) ? 1 : 0;
    HaloOut ho;
    const bool hf = halo_begin(c, c->x[c->xcur ^ 1], sizeof(double), ho);
    GADI_TRY(launch_sweep(c, o, &ho));
    c->xcur ^= 1;
    return halo_end(c, c->x[c->xcur], sizeof(double), hf);
  }

  template <int DIM, int ZS, bool CPLX>
  static int outer_d(Ctx* c, double scale, int has_e) {
    if constexpr (CPLX) {
      return has_e ? outer_t<DIM, ZS, 0, true, true>(c, scale) : outer_t<DIM, ZS, 0, false, true>(c, scale);
    } else {
      const int ur = c->ur == GADI_FP64 ? 0 : (c->ur == GADI_FP64X2 ? 2 : 1);
      if (ur == 0) return has_e ? outer_t<DIM, ZS, 0, true, false>(c, scale) : outer_t<DIM, ZS, 0, false, false>(c, scale);
      if (ur == 1) return has_e ? outer_t<DIM, ZS, 1, true, false>(c, scale) : outer_t<DIM, ZS, 1, false, false>(c, scale);
      return has_e ? outer_t<DIM, ZS, 2, true, false>(c, scale) : outer_t<DIM, ZS, 2, false, false>(c, scale);
    }
  }

  // ------------------------------------------------------------ Op x
  template <int DIM, int ZS, bool STRICT>
  static int apply_sweep(Ctx* c, const CoefT<double>& C, const double* in, double* out) {
    typedef GeoT<ST, DIM, ZS> G;
    ApplyOp<G, STRICT> a;
    a.in = in;
    a.outv = out;
    a.C = cast_coef<CT>(C);
    return launch_sweep(c, a);
  }
  template <bool TRANS, bool STRICT>
  static int apply_cplx(Ctx* c, const double* in, double* out) {
    CApply<ST, TRANS, STRICT> a;
    a.vs = (const ST*)c->VS;
    a.al = (CT)c->d.alpha_s;
    a.in = in;
    a.outv = out;
    return launch_pw(c, a);
  }

  // ------------------------------------------------------------ vtable
  template <bool RF>
  static int h_solve_m(Ctx* c, double scale, double tol, int maxit) {
    if (c->kind == GADI_COMPLEX)
      return c->ndim == 3 ? h_solve_t<3, 2, RF>(c, scale, tol, maxit) : h_solve_t<2, 2, RF>(c, scale, tol, maxit);
    if (c->ndim == 3) return h_solve_t<3, 1, RF>(c, scale, tol, maxit);
    return h_solve_t<2, 1, RF>(c, scale, tol, maxit);
  }
  static int h_solve(Ctx* c, double scale, double tol, int maxit) {
    if (c->kind == GADI_CSR) return h_solve_csr(c, scale, tol, maxit);
    return c->rounding == 1 ? h_solve_m<true>(c, scale, tol, maxit) : h_solve_m<false>(c, scale, tol, maxit);
  }
  template <bool RF>
  static int s_solve_m(Ctx* c, double coeff, double tol, int maxit) {
    if (c->kind == GADI_COMPLEX) return s_solve_cplx<RF>(c, coeff, tol, maxit);
    if (c->ndim == 3) return s_solve_real<3, RF>(c, coeff, tol, maxit);
    return s_solve_real<2, RF>(c, coeff, tol, maxit);
  }
  static int s_solve(Ctx* c, double coeff, double tol, int maxit) {
    if (c->kind == GADI_CSR) return s_solve_csr(c, coeff, tol, maxit);
    return c->rounding == 1 ? s_solve_m<true>(c, coeff, tol, maxit) : s_solve_m<false>(c, coeff, tol, maxit);
  }
  static int outer(Ctx* c, double scale, int has_e) {
    if (c->kind == GADI_CSR) return outer_csr(c, scale, has_e);
    if (c->kind == GADI_COMPLEX)
      return c->ndim == 3 ? outer_d<3, 2, true>(c, scale, has_e) : outer_d<2, 2, true>(c, scale, has_e);
    if (c->ndim == 3) return outer_d<3, 1, false>(c, scale, has_e);
    return outer_d<2, 1, false>(c, scale, has_e);
  }
  static int apply(Ctx* c, int op, int strict, const double* in, double* out) {
    if (c->kind == GADI_CSR) return apply_csr(c, op, strict, in, out);
    const CoefT<double>& C = op == 1 ? c->H : (op == 2 ? c->S : c->ST);
    if (c->kind == GADI_COMPLEX) {
      if (op == 1 && c->ndim == 3)
        return strict ? apply_sweep<3, 2, true>(c, C, in, out) : apply_sweep<3, 2, false>(c, C, in, out);
      if (op == 1)
        return strict ? apply_sweep<2, 2, true>(c, C, in, out) : apply_sweep<2, 2, false>(c, C, in, out);
      if (op == 2) return strict ? apply_cplx<false, true>(c, in, out) : apply_cplx<false, false>(c, in, out);
      return strict ? apply_cplx<true, true>(c, in, out) : apply_cplx<true, false>(c, in, out);
    }
    if (c->ndim == 3)
      return strict ? apply_sweep<3, 1, true>(c, C, in, out) : apply_sweep<3, 1, false>(c, C, in, out);
    return strict ? apply_sweep<2, 1, true>(c, C, in, out) : apply_sweep<2, 1, false>(c, C, in, out);
  }
  static int quantize(Ctx* c, const double* in, void* out, long long n) {
    const int nb = (int)std::min<long long>((n + 255) / 256, (long long)c->sms * 16);
    quantize_kernel<ST><<<std::max(nb, 1), 256, 0, c->stream>>>(in, (ST*)out, n);
    c->launches++;
    GADI_CUDA(cudaGetLastError());
    return 0;
  }
  static int widen(Ctx* c, const void* in, double* out, long long n) {
    const int nb = (int)std::min<long long>((n + 255) / 256, (long long)c->sms * 16);
    widen_kernel<ST><<<std::max(nb, 1), 256, 0, c->stream>>>((const ST*)in, out, n);
    c->launches++;
    GADI_CUDA(cudaGetLastError());
    return 0;
  }
  static EngineVT vt() { return EngineVT{&h_solve, &s_solve, &outer, &apply, &quantize, &widen}; }
};

}  // namespace gadi
