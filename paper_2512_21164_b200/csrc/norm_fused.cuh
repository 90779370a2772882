// One power-iteration step of ||A||_2 (analysis.py:58-66) in ONE sweep:
//     v = w / ||w|| ;  t = A v ;  w' = A^T t ;  sum w'^2
// The two-pass form (NormPass<false>, NormPass<true>) streams 4 fp64 vectors
// per iteration (read w, write t, read t, write w'); this kernel streams 2.
// t = A w * (1/||w||) (the normalisation applied once per t value instead
// of to each of the seven v reads: one rounding away from A (w/||w||) of the
// two-pass form; ||A||_2 is not pinned bitwise by the reference and agrees
// to ~1e-15).  t never leaves the SM: while the CTA marches along x it computes the
// t-plane x+1 on its tile plus a one-cell ring (helper warps own the two
// y-halo rows and the two z-halo columns) from the v-planes
// x, x+1, x+2 held in the TMA stage ring, keeps t for its own columns in a
// 3-plane register queue (x-neighbours) and the whole t-plane in a
// shared-memory ring of t-planes (y / z neighbours; 3-D: four planes handed
// over by one mbarrier each, 2-D: three behind a CTA barrier), and applies
// A^T to produce w'-plane x.
//
// Real 5-point (DIM 2: rows of 64 lanes) and 7-point (DIM 3: 32 lanes x TY
// rows) stencils on a single domain; the crd family and slab contexts keep
// the two-pass form.
#pragma once
#include "sweep_tma.cuh"
#include "tmap.cuh"

namespace gadi {

#ifndef GADI_VZNORM
#define GADI_VZNORM 4  // fp64 elements per lane (measured: 4 beats 2 here, not in the other fp64 passes)
#endif
// GADI_NORM_MBAR = 1: the per-plane CTA barrier between "t-plane x+1 stored"
// and "A^T reads t-plane x" becomes one mbarrier per t buffer (4 buffers):
// every consumer / helper warp arrives after storing its part of a t-plane
// and waits only for the plane it is about to read (stored one plane
// earlier), so warps drift within the ring instead of meeting every plane.
#ifndef GADI_NORM_MBAR
#define GADI_NORM_MBAR 1
#endif
// GADI_NORM_ILP = 1: the 7-term stencils as two independent FMA chains
// (depth 4 instead of 7) and one ||w'||^2 accumulator per vector element
// (the fp64 chain through `red` was one dependent DFMA per element)
#ifndef GADI_NORM_ILP
#define GADI_NORM_ILP 0
#endif
#ifndef GADI_NORM_XU
#define GADI_NORM_XU 1
#endif
// tile rows, CTAs per SM (register budget) and stage-count rule of the fused
// power iteration (GADI_NORM_NSTANY = 0: 8 or 4 stages, a power of two)
// 3-D default: 16-row tiles, one CTA per SM (107 registers: the mbarrier
// form no longer spills) -- 782 -> 708 us at 512^3 (profiles/ab_norm_tile2_r2.jsonl);
// 2-D keeps 2 CTAs per SM of one-row tiles and the CTA barrier.
#ifndef GADI_NORM_TY
#define GADI_NORM_TY 16
#endif
#ifndef GADI_NORM_MINB
#define GADI_NORM_MINB 1
#endif
#ifndef GADI_NORM_NSTANY
#define GADI_NORM_NSTANY 0
#endif
template <int DIM>
struct NFShape {
  static constexpr int VZ = GADI_VZNORM;
  static constexpr int BZ = DIM == 3 ? 32 : 64;
  static constexpr int TY = DIM == 3 ? GADI_NORM_TY : 1;
  static constexpr int MINB = DIM == 3 ? GADI_NORM_MINB : 2;  // CTAs per SM (register budget)
  static constexpr bool MB = GADI_NORM_MBAR && DIM == 3;      // mbarrier t-plane handoff
  static constexpr int TZ = BZ * VZ;
  static constexpr int HZ = 2;                       // 16-byte pad = 2 fp64 each side
  static constexpr int HV = DIM == 3 ? 2 : 0;        // v halo rows each side
  static constexpr int HT = DIM == 3 ? 1 : 0;        // t halo rows each side
  static constexpr int VROWS = TY + 2 * HV;
  static constexpr int ROW = TZ + 2 * HZ;            // elements per smem row (v and t)
  static constexpr int STAGE = VROWS * ROW * 8;
  static constexpr int TROWS = TY + 2 * HT;
  static constexpr int TPLANE = TROWS * ROW;         // elements per t buffer
  static constexpr int NT = BZ * TY;
  // helper warps: 3-D: one per t halo row, whose first TY lanes also compute
  // the two z-halo columns of the core rows; 2-D: one warp for the two z-halo
  // values (keeps the divergent single-column work off the core warps)
  static constexpr int NH = DIM == 3 ? 2 : 1;
  static constexpr int NCONS = NT + 32 * NH;
  static constexpr int NTOT = NCONS + 32;
  static constexpr int NTB = MB ? 4 : 3;                          // t buffers
  static constexpr int TBYTES = (NTB * TPLANE * 8 + 127) / 128 * 128;  // stages 128-byte aligned (TMA boxes)
  static constexpr int BUDGET = (MINB >= 3 ? 72 : (MINB >= 2 ? 100 : 200)) * 1024;
  static constexpr int NST_RAW = (BUDGET - TBYTES) / STAGE;
  static constexpr int NST = GADI_NORM_NSTANY ? (NST_RAW > 8 ? 8 : NST_RAW)
                                              : (NST_RAW >= 8 ? 8 : 4);  // power of two: cheap stage indexing
  static constexpr size_t SMEM = (size_t)TBYTES + (size_t)NST * STAGE + (2 * NST + NTB) * sizeof(uint64_t);
};

template <int DIM, bool DENSE>
struct NormFused {
  SweepGeom g;
  double* defer;
  double* partials;
  unsigned int* ticket;
  NormState* ns;
  const double* in;  // w
  double* outv;      // w'
  CoefT<double> A, AT;
  double rnw;
  int use_tm;  // the v tile of a stage is one tensor-map box (hardware zero fill), else row copies
  static constexpr int NR = 1;
  static constexpr bool HAS_RED = true;
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  __device__ bool prepare() {
    if (ns->done) return false;
    rnw = 1.0 / ns->nw;
    return true;
  }
  __device__ void finalize(const double (&t)[1]) const { fin_norm(ns, t[0]); }
};

// The power iteration only feeds the backward-error denominator ||A||_2; its
// bits are not pinned by the reference (scipy's order), so the
// dense case contracts each term into an FMA (half the fp64 instructions,
// half the dependent chain).  sigma agrees with the ordered form to ~1e-15
// (tests pin it to the reference at 1e-12).  GADI_NORM_ORDERED=1 keeps the
// non-contracted order.
#ifndef GADI_NORM_ORDERED
#define GADI_NORM_ORDERED 0
#endif
template <int DIM, bool DENSE>
__device__ __forceinline__ double nf_stencil(const CoefT<double>& c, double xm, double ym, double zm, double ce,
                                             double zp, double yp, double xp) {
  if constexpr (DENSE && !GADI_NORM_ORDERED && GADI_NORM_ILP) {
    double a = c.lo[0] * xm, b = c.up[0] * xp;
    a = fma_rn(c.lo[1], ym, a);
    b = fma_rn(c.up[1], yp, b);
    a = fma_rn(c.lo[2], zm, a);
    b = fma_rn(c.up[2], zp, b);
    a = fma_rn(c.d, ce, a);
    return a + b;
  } else if constexpr (DENSE && !GADI_NORM_ORDERED) {
    double acc = c.lo[0] * xm;
    acc = fma_rn(c.lo[1], ym, acc);
    acc = fma_rn(c.lo[2], zm, acc);
    acc = fma_rn(c.d, ce, acc);
    acc = fma_rn(c.up[2], zp, acc);
    acc = fma_rn(c.up[1], yp, acc);
    return fma_rn(c.up[0], xp, acc);
  } else if constexpr (DENSE) {
    return apply_stencil_dense(c, 0.0, xm, ym, zm, ce, zp, yp, xp);
  } else {
    return apply_stencil<true>(c, 0.0, xm, ym, zm, ce, zp, yp, xp);
  }
}

template <int DIM, bool DENSE>
__global__ void __launch_bounds__(NFShape<DIM>::NTOT, NFShape<DIM>::MINB)
    norm_fused_kernel(NormFused<DIM, DENSE> p, const __grid_constant__ CUtensorMap tmw) {
  using S = NFShape<DIM>;
  constexpr int VZ = S::VZ, BZ = S::BZ, TY = S::TY, TZ = S::TZ, HZ = S::HZ, HV = S::HV, HT = S::HT;
  constexpr int ROW = S::ROW, NST = S::NST, NT = S::NT, NCONS = S::NCONS, NWCONS = NCONS / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* tbuf = reinterpret_cast<double*>(smem_raw);
  unsigned char* stages = smem_raw + S::TBYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + (size_t)NST * S::STAGE);
  uint64_t* empty = full + NST;
  uint64_t* twr = empty + NST;  // GADI_NORM_MBAR: "t buffer b stored" (all consumer + helper warps)

  if (!p.prepare()) return;
  const SweepGeom g = p.g;
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWCONS);
    }
    for (int b = 0; b < S::NTB; ++b) mbar_init(&twr[b], NWCONS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double red[1] = {0.0};
  double redk[VZ];
#pragma unroll
  for (int k = 0; k < VZ; ++k) redk[k] = 0.0;

  if (tid >= NCONS) {
    // ---------------------------------------------------------------- producer
    constexpr int NCOPY = S::VROWS;
    SegIter it(g, gridDim.x, blockIdx.x);
    int tile, xa, xb, gs = 0;
    while (it.next(tile, xa, xb)) {
      const int zt0 = (tile % g.nzt) * TZ, y0 = (tile / g.nzt) * TY;
      const int za = max(zt0 - HZ, 0), zbnd = min(zt0 + TZ + HZ, g.nz);
      const unsigned rowbytes = (unsigned)((zbnd - za) * 8), dst0 = (unsigned)((za - (zt0 - HZ)) * 8);
      for (int xp = xa - 2; xp <= xb + 1; ++xp, ++gs) {
        const int st = gs % NST;
        if (gs >= NST) mbar_wait(&empty[st], (unsigned)(((gs / NST) - 1) & 1));
        unsigned char* sb = stages + (size_t)st * S::STAGE;
        const bool pv = xp >= 0 && xp < g.nx;
        if (p.use_tm) {
          // one (TZ + 2 HZ) x (TY + 2 HV) box: rows / columns outside the grid arrive as zeros
          if (lane == 0) {
            mbar_expect_tx(&full[st], pv ? (unsigned)S::STAGE : 0u);
            if (pv) tma_load_3d(sb, &tmw, zt0 - HZ, y0 - HV, xp, &full[st]);
          }
          __syncwarp();
          continue;
        }
        unsigned bytes = 0;
        if (pv)
          for (int r = 0; r < NCOPY; ++r) {
            const int yy = y0 - HV + r;
            if (yy >= 0 && yy < g.ny) bytes += rowbytes;
          }
        if (lane == 0) mbar_expect_tx(&full[st], bytes);
        __syncwarp();
        if (pv)
          for (int r = lane; r < NCOPY; r += 32) {
            const int yy = y0 - HV + r;
            if (yy < 0 || yy >= g.ny) continue;
            const long long e0 = (long long)xp * g.plane + (long long)yy * g.nz + za;
            bulk_g2s(sb + (size_t)r * ROW * 8 + dst0, p.in + e0, rowbytes, &full[st]);
          }
      }
    }
  } else {
    // ---------------------------------------------------------------- consumers
    const bool halo = tid >= NT;
    const int hw = (tid - NT) / 32;  // helper warp index
    const int tz = halo ? lane : tid % BZ;
    const int trow = halo ? (hw == 0 ? 0 : TY + 2 * HT - 1) : tid / BZ + HT;  // row in the t buffer
    const int vrow = trow - HT + HV;                                          // same y in a v stage
    const bool has_row = !halo || DIM == 3;  // computes t on its own columns of `trow`
    // z-halo column duty (helper lanes): t buffer row zrow, tile column zcol
    const bool has_zcol = halo && (DIM == 3 ? lane < TY : lane < 2);
    const int zrow = DIM == 3 ? 1 + lane : 0;
    const int zcol = (DIM == 3 ? hw == 0 : lane == 0) ? -1 : TZ;
    const double rnw = p.rnw;
    auto wait_full = [&](int s) { mbar_wait(&full[s % NST], (unsigned)((s / NST) & 1)); };
    auto release = [&](int s) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s % NST]);
    };
    auto vrowp = [&](int s, int r) {
      return reinterpret_cast<const double*>(stages + (size_t)(s % NST) * S::STAGE) + (size_t)r * ROW;
    };

    SegIter it(g, gridDim.x, blockIdx.x);
    int tile, xa, xb, gs = 0;
    int tq = 0;  // GADI_NORM_MBAR: t-planes stored by this CTA before the segment
    while (it.next(tile, xa, xb)) {
      const int zt0 = (tile % g.nzt) * TZ, y0 = (tile / g.nzt) * TY;
      const int y = y0 + trow - HT;
      const bool yok = y >= 0 && y < g.ny;
      const int zb = zt0 + tz * VZ;
      const bool zok = zb < g.nz;          // nz % VZ == 0: a lane's vector is all in or all out
      const bool own = has_row && yok && zok;
      // validity of v rows y-1, y, y+1 and of the z-halo columns
      const bool ym_ok = y - 1 >= 0 && y - 1 < g.ny, yp_ok = y + 1 >= 0 && y + 1 < g.ny;
      const int gs0 = gs;  // stage of plane xa-2
      auto st_of = [&](int x) { return gs0 + (x - (xa - 2)); };

      // v (scaled, masked) at stage s, stage row r, tile column c (-HZ .. TZ+HZ-1)
      auto vat = [&](int s, int x, int r, int c) -> double {
        const int yy = y0 - HV + r, zz = zt0 + c;
        if (x < 0 || x >= g.nx || yy < 0 || yy >= g.ny || zz < 0 || zz >= g.nz) return 0.0;
        return vrowp(s, r)[c + HZ];
      };
      auto vown = [&](int x, double (&o)[VZ]) {
        if (x < 0 || x >= g.nx || !own) {
#pragma unroll
          for (int k = 0; k < VZ; ++k) o[k] = 0.0;
          return;
        }
        const double* q = vrowp(st_of(x), vrow) + HZ + tz * VZ;
#pragma unroll
        for (int k = 0; k < VZ; ++k) o[k] = q[k];
      };
      // t at plane x+1 for this thread's columns (vA, vB, vC = v planes x, x+1, x+2)
      // (every lane of the warp runs the shuffles; invalid lanes get t = 0)
      auto t_own = [&](int x, const double (&vA)[VZ], const double (&vB)[VZ], const double (&vC)[VZ],
                       double (&t)[VZ]) {
        double left = __shfl_up_sync(0xffffffffu, vB[VZ - 1], 1);
        double right = __shfl_down_sync(0xffffffffu, vB[0], 1);
        const bool ok = x + 1 >= 0 && x + 1 < g.nx && own;
        if (!ok) {
#pragma unroll
          for (int k = 0; k < VZ; ++k) t[k] = 0.0;
          return;
        }
        const int s = st_of(x + 1);
        const double* rm = vrowp(s, vrow - 1) + HZ + tz * VZ;
        const double* rp = vrowp(s, vrow + 1) + HZ + tz * VZ;
        if (lane == 0) left = vat(s, x + 1, vrow, tz * VZ - 1);
        if (lane == 31) right = vat(s, x + 1, vrow, tz * VZ + VZ);
#pragma unroll
        for (int k = 0; k < VZ; ++k) {
          const double zm = k > 0 ? vB[k - 1] : left;
          const double zp = k < VZ - 1 ? vB[k + 1] : right;
          const double ym = (DIM == 3 && ym_ok) ? rm[k] : 0.0;
          const double yp = (DIM == 3 && yp_ok) ? rp[k] : 0.0;
          t[k] = nf_stencil<DIM, DENSE>(p.A, vA[k], ym, zm, vB[k], zp, yp, vC[k]) * rnw;
        }
      };
      // t at plane x+1, t buffer row rt, tile column c (the z-halo columns)
      auto t_col = [&](int x, int rt, int c) -> double {
        const int zz = zt0 + c, yy = y0 + rt - HT, vr = rt - HT + HV;
        if (x + 1 < 0 || x + 1 >= g.nx || yy < 0 || yy >= g.ny || zz < 0 || zz >= g.nz) return 0.0;
        const int s = st_of(x + 1);
        return nf_stencil<DIM, DENSE>(p.A, vat(st_of(x), x, vr, c), vat(s, x + 1, vr - 1, c),
                                      vat(s, x + 1, vr, c - 1), vat(s, x + 1, vr, c), vat(s, x + 1, vr, c + 1),
                                      vat(s, x + 1, vr + 1, c), vat(st_of(x + 2), x + 2, vr, c)) * rnw;
      };
      // t-plane x (x >= xa) is the CTA's stored plane tq + x - xa
      auto tbuf_of = [&](int x) -> double* {
        if constexpr (S::MB) return tbuf + (size_t)((tq + x - xa) % S::NTB) * S::TPLANE + HZ;
        else return tbuf + (size_t)((x - (xa - 1)) % 3) * S::TPLANE + HZ;
      };
      auto t_published = [&](int x) {  // this warp's part of t-plane x is in its buffer
        if constexpr (S::MB) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&twr[(tq + x - xa) % S::NTB]);
        }
      };
      auto t_wait = [&](int x) {  // every warp's part of t-plane x is in its buffer
        if constexpr (S::MB) {
          const int q = tq + x - xa;
          mbar_wait(&twr[q % S::NTB], (unsigned)((q / S::NTB) & 1));
        }
      };
      auto t_store = [&](int x, const double (&t)[VZ]) {  // t-plane x+1 -> its buffer
        double* b = tbuf_of(x + 1);
        if (has_row) {
#pragma unroll
          for (int k = 0; k < VZ; ++k) b[(size_t)trow * ROW + tz * VZ + k] = t[k];
        }
        if (has_zcol) b[(size_t)zrow * ROW + zcol] = t_col(x, zrow, zcol);
      };

      double vA[VZ], vB[VZ], vC[VZ], tp[VZ], tc[VZ], tn[VZ];
      // prologue: t(xa-1) (own columns), t(xa) (own columns + buffer)
      wait_full(st_of(xa - 2));
      wait_full(st_of(xa - 1));
      wait_full(st_of(xa));
      vown(xa - 2, vA);
      vown(xa - 1, vB);
      vown(xa, vC);
      t_own(xa - 2, vA, vB, vC, tp);
      release(st_of(xa - 2));
#pragma unroll
      for (int k = 0; k < VZ; ++k) {
        vA[k] = vB[k];
        vB[k] = vC[k];
      }
      wait_full(st_of(xa + 1));
      vown(xa + 1, vC);
      t_own(xa - 1, vA, vB, vC, tc);
      // (mbarrier form) the buffers this segment overwrites first were last
      // read before every warp stored the previous segment's final t-plane
      if (S::MB && tq > 0) t_wait(xa - 1);
      t_store(xa - 1, tc);
      t_published(xa);
      release(st_of(xa - 1));
      if constexpr (!S::MB) consumer_sync(NCONS);

      long long gidx = (long long)xa * g.plane + (long long)y * g.nz + zb;
      // GADI_NORM_XU = 3 unrolls by the period of the v / t register queues
#if GADI_NORM_XU == 3
#pragma unroll 3
#elif GADI_NORM_XU == 2
#pragma unroll 2
#endif
      for (int x = xa; x < xb; ++x, gidx += g.plane) {
        // t-plane x+1 from v-planes x, x+1, x+2
#pragma unroll
        for (int k = 0; k < VZ; ++k) {
          vA[k] = vB[k];
          vB[k] = vC[k];
        }
        wait_full(st_of(x + 2));
        vown(x + 2, vC);
        t_own(x, vA, vB, vC, tn);
        t_store(x, tn);
        if constexpr (S::MB) {
          t_published(x + 1);
          release(st_of(x));
          t_wait(x);
        } else {
          consumer_sync(NCONS);
          release(st_of(x));
        }
        // w'-plane x = A^T t from t(x-1), t(x), t(x+1)
        if (!halo) {
          double left = __shfl_up_sync(0xffffffffu, tc[VZ - 1], 1);
          double right = __shfl_down_sync(0xffffffffu, tc[0], 1);
          if (own) {
            const double* b = tbuf_of(x);
            const double* rc = b + (size_t)trow * ROW + tz * VZ;
            const double* rm = rc - ROW;
            const double* rp = rc + ROW;
            if (lane == 0) left = rc[-1];
            if (lane == 31) right = rc[VZ];
            double o[VZ];
#pragma unroll
            for (int k = 0; k < VZ; ++k) {
              const double zm = k > 0 ? tc[k - 1] : left;
              const double zp = k < VZ - 1 ? tc[k + 1] : right;
              const double ym = DIM == 3 ? rm[k] : 0.0;
              const double yp = DIM == 3 ? rp[k] : 0.0;
              o[k] = nf_stencil<DIM, DENSE>(p.AT, tp[k], ym, zm, tc[k], zp, yp, tn[k]);
              if constexpr (GADI_NORM_ILP) redk[k] = fma_rn(o[k], o[k], redk[k]);
              else red[0] += o[k] * o[k];
            }
            store_any<double, VZ>(p.outv, gidx, VZ, o, true);
          }
        }
#pragma unroll
        for (int k = 0; k < VZ; ++k) {
          tp[k] = tc[k];
          tc[k] = tn[k];
        }
      }
      release(st_of(xb));
      release(st_of(xb + 1));
      gs += xb - xa + 4;
      tq += xb - xa + 1;
    }
  }
  if constexpr (GADI_NORM_ILP) {
#pragma unroll
    for (int k = 0; k < VZ; ++k) red[0] += redk[k];
  }

  double tot[1];
  const int ops[1] = {RED_SUM};
  if (grid_finish<1, S::NTOT>(red, ops, p.partials, g.pstride, p.ticket, tot)) {
    if (threadIdx.x == 0) finish_pass(p, tot);
  }
}

}  // namespace gadi
