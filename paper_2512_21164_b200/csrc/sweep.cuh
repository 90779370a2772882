// Generic 2.5-D stencil sweep for constant-coefficient 5-point (2-D) and
// 7-point (3-D) operators, matrix-free.
//
// Layout: a vector is the reference's lexicographic grid order
// (gadimp/problems.py:62-65, 88-92): element (x, y, z) lives at
// x*ny*nz + y*nz + z with z fastest.  2-D problems use ny = 1 (x = slow
// index, z = fast index); the interleaved complex layout of the crd family
// doubles nz and uses a z-stride ZS = 2 so each component sees its own
// 5-point Laplacian.
//
// Each CTA owns a TY x TZ tile of the (y, z) plane and marches along x over a
// chunk of planes.  Every input element is read from HBM once per sweep
// (plus the 2-plane overlap of neighbouring x-chunks and the in-plane halo,
// which L2 serves):
//   * x-neighbours come from a 3-deep register queue (prev/cur/next plane);
//   * y-neighbours from a double-buffered shared-memory copy of the plane;
//   * z-neighbours from the thread's own VZ-vector, warp shuffles, and the
//     shared-memory row at warp/tile edges.
// Loads of plane x+2 are issued before the stencil of plane x is evaluated so
// global latency overlaps compute.  Vector loads are 16 B wide.
//
// A "pass" P supplies: how to turn raw inputs into the stencil field(s) f
// (pointwise, e.g. f = r + beta*p), the coefficients of the operator applied
// to each field, and an epilogue that consumes the centre values, the
// stencil results and per-point extra inputs, writes outputs and
// accumulates partial sums.  Partial sums go through the deterministic
// last-block reduction (common.cuh) into P::finalize, which runs the scalar
// logic of the Krylov recurrences on the device.
#pragma once
#include "common.cuh"

namespace gadi {

struct SweepGeom {
  int nx, ny, nz;      // nz fastest, in elements
  long long plane;     // ny * nz
  int nzt, nyt;        // tile counts along z and y
  int xchunk;          // planes per CTA
  int pstride;         // partials row stride (>= number of CTAs)
  int vec;             // 16-byte vector path usable (nz % VZ == 0)
  int hlo, hhi;        // slab decomposition: plane -1 / plane nx is a valid halo plane
};

// The seven neighbour values of one point, plus its centre.
template <class CT> struct Nb { CT xm, ym, zm, ce, zp, yp, xp; };

template <class CT> struct CoefT {
  CT d;
  CT lo[3];  // neighbour with the smaller index, axis order x, y, z
  CT up[3];
};

// Ascending-column accumulation starting from `acc`: lo_x, lo_y, lo_z, d,
// up_z, up_y, up_x (gadimp/sparsemat.py:193-198 with scipy's CSR order).
// Zero coefficients are skipped exactly as the CSR has no stored zeros.
template <bool ORD, class CT>
__device__ __forceinline__ CT apply_stencil(const CoefT<CT>& c, CT acc, CT xm, CT ym, CT zm, CT ce, CT zp, CT yp,
                                            CT xp) {
  if constexpr (!ORD) {
    // storage model: a zero coefficient contributes an exact 0 (finite
    // operands), so the fused chain needs no presence tests
    acc = fma_rn(c.lo[0], xm, acc);
    acc = fma_rn(c.lo[1], ym, acc);
    acc = fma_rn(c.lo[2], zm, acc);
    acc = fma_rn(c.d, ce, acc);
    acc = fma_rn(c.up[2], zp, acc);
    acc = fma_rn(c.up[1], yp, acc);
    return fma_rn(c.up[0], xp, acc);
  }
  if (c.lo[0] != CT(0)) acc = madd<ORD>(c.lo[0], xm, acc);
  if (c.lo[1] != CT(0)) acc = madd<ORD>(c.lo[1], ym, acc);
  if (c.lo[2] != CT(0)) acc = madd<ORD>(c.lo[2], zm, acc);
  if (c.d != CT(0)) acc = madd<ORD>(c.d, ce, acc);
  if (c.up[2] != CT(0)) acc = madd<ORD>(c.up[2], zp, acc);
  if (c.up[1] != CT(0)) acc = madd<ORD>(c.up[1], yp, acc);
  if (c.up[0] != CT(0)) acc = madd<ORD>(c.up[0], xp, acc);
  return acc;
}

// Passes whose epilogue needs a per-point coefficient indexed differently
// from the grid (the crd potential v, one per complex point) load it from
// global memory in the TMA forms (load_epi_v), next to the staged inputs.
template <class P, class = void> struct HasEpiV : std::false_type {};
template <class P> struct HasEpiV<P, std::void_t<decltype(&P::load_epi_v)>> : std::true_type {};

// Optional per-vector hooks: a pass may process a lane's whole VZ-vector at
// once (packed fp32x2 arithmetic) instead of element by element.
template <class P, class = void> struct HasStencilVec : std::false_type {};
template <class P> struct HasStencilVec<P, std::void_t<decltype(&P::stencil_vec)>> : std::true_type {};
template <class P, class = void> struct HasFieldVec : std::false_type {};
template <class P> struct HasFieldVec<P, std::void_t<decltype(&P::field_vec)>> : std::true_type {};

// Storage-model 7-point stencil on a lane's vector with packed fp32x2 FMAs
// for the x, y and centre terms (pairs of adjacent z-elements) and scalar
// FMAs for the z-neighbours (which straddle pairs).  HASY = 3-D.
template <bool HASY, int VZ, int ZS>
__device__ __forceinline__ void stencil_packed(const CoefT<float>& c, const float (&xm)[VZ], const float (&ym)[VZ],
                                               const float (&ce)[VZ], const float (&left)[ZS],
                                               const float (&right)[ZS], const float (&yp)[VZ],
                                               const float (&xp)[VZ], float (&out)[VZ]) {
  const float2 clx = bcast2(c.lo[0]), cd = bcast2(c.d), cux = bcast2(c.up[0]);
  const float2 cly = bcast2(c.lo[1]), cuy = bcast2(c.up[1]);
#pragma unroll
  for (int j = 0; j < VZ; j += 2) {
    float2 acc = fmul2(cd, make_float2(ce[j], ce[j + 1]));
    acc = ffma2(clx, make_float2(xm[j], xm[j + 1]), acc);
    acc = ffma2(cux, make_float2(xp[j], xp[j + 1]), acc);
    if constexpr (HASY) {
      acc = ffma2(cly, make_float2(ym[j], ym[j + 1]), acc);
      acc = ffma2(cuy, make_float2(yp[j], yp[j + 1]), acc);
    }
    const float zm0 = (j >= ZS) ? ce[j - ZS] : left[j];
    const float zm1 = (j + 1 >= ZS) ? ce[j + 1 - ZS] : left[j + 1];
    const float zp0 = (j + ZS < VZ) ? ce[j + ZS] : right[j + ZS - VZ];
    const float zp1 = (j + 1 + ZS < VZ) ? ce[j + 1 + ZS] : right[j + 1 + ZS - VZ];
    out[j] = fmaf(c.up[2], zp0, fmaf(c.lo[2], zm0, acc.x));
    out[j + 1] = fmaf(c.up[2], zp1, fmaf(c.lo[2], zm1, acc.y));
  }
}

// Tiling constants shared by a pass and its host launcher.
template <class P> struct SweepShape {
  using CT = typename P::CT;
  static constexpr int VZ = P::VZ, BZ = P::BZ, BY = P::BY, ZS = P::ZS, NF = P::NF;
  static constexpr int TZ = BZ * VZ, TY = BY;
  static constexpr int PAD = (16 / (int)sizeof(CT)) > ZS ? (16 / (int)sizeof(CT)) : ZS;
  static constexpr int ROW = TZ + 2 * PAD;
  static constexpr int PLANE = NF * (TY + 2) * ROW;  // elements per buffer
  static constexpr size_t SMEM = 2 * (size_t)PLANE * sizeof(CT);
};

// Ordered form without the presence tests, for operators whose seven
// coefficients are all nonzero (then the CSR stores every term and the two
// forms are the same operations); saves the per-term branches.
template <class CT>
__device__ __forceinline__ CT apply_stencil_dense(const CoefT<CT>& c, CT acc, CT xm, CT ym, CT zm, CT ce, CT zp, CT yp,
                                                  CT xp) {
  acc = add_rn(acc, mul_rn(c.lo[0], xm));
  acc = add_rn(acc, mul_rn(c.lo[1], ym));
  acc = add_rn(acc, mul_rn(c.lo[2], zm));
  acc = add_rn(acc, mul_rn(c.d, ce));
  acc = add_rn(acc, mul_rn(c.up[2], zp));
  acc = add_rn(acc, mul_rn(c.up[1], yp));
  return add_rn(acc, mul_rn(c.up[0], xp));
}

template <bool ORD, class CT>
__device__ __forceinline__ CT apply_stencil(const CoefT<CT>& c, CT acc, const Nb<CT>& n) {
  return apply_stencil<ORD>(c, acc, n.xm, n.ym, n.zm, n.ce, n.zp, n.yp, n.xp);
}

// End of a reducing pass: run the scalar recurrence in place (one rank), or
// deposit this rank's totals for the gather + finalize_kernel (slabs).
// Slot of a pass's reference-rounding fl_dot (strict.cuh), or -1.
template <class P, class = void> struct TreeSlot : std::integral_constant<int, -1> {};
template <class P> struct TreeSlot<P, std::void_t<decltype(P::TS)>> : std::integral_constant<int, P::TS> {};

template <class P, int NR>
__device__ __forceinline__ void finish_pass(const P& p, const double (&tot)[NR]) {
  if constexpr (TreeSlot<P>::value >= 0) {
    if (p.tout.aux) {  // the tree finisher (strict.cuh) completes the reduction
#pragma unroll
      for (int s = 0; s < NR; ++s) p.tout.aux[s] = tot[s];
      return;
    }
  }
  if (p.defer) {
#pragma unroll
    for (int s = 0; s < NR; ++s) p.defer[s] = tot[s];
  } else {
    p.finalize(tot);
  }
}

// Slab decomposition: reduce the gathered per-rank totals in rank order (the
// same order on every rank) and run the pass's scalar recurrence.
template <class P>
__global__ void finalize_kernel(P p, const double* __restrict__ gbuf, int nranks, int row) {
  if (!p.prepare()) return;
  constexpr int NR = P::NR;
  double tot[NR];
#pragma unroll
  for (int s = 0; s < NR; ++s) tot[s] = gbuf[s];
  for (int r = 1; r < nranks; ++r)
#pragma unroll
    for (int s = 0; s < NR; ++s) tot[s] = red_combine(P::op(s), tot[s], gbuf[(size_t)r * row + s]);
  p.finalize(tot);
}

template <class P>
__global__ void __launch_bounds__(P::NT) sweep_kernel(P p) {
  using S = SweepShape<P>;
  using CT = typename P::CT;
  constexpr int VZ = S::VZ, BZ = S::BZ, BY = S::BY, ZS = S::ZS, NF = S::NF;
  constexpr int TZ = S::TZ, TY = S::TY, PAD = S::PAD, ROW = S::ROW;
  constexpr int NR = P::NR, NT = P::NT;
  static_assert(BZ % 32 == 0, "BZ must be a multiple of the warp size");
  static_assert(VZ % ZS == 0 && VZ >= ZS, "vector must hold whole z-stencil strides");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  CT* sm = reinterpret_cast<CT*>(smem_raw);

  if (!p.prepare()) return;  // device-side convergence flag: whole grid is a no-op

  const SweepGeom g = p.g;
  const int tid = threadIdx.x, tz = tid % BZ, ty = tid / BZ, lane = tid & 31;
  int bidx = blockIdx.x;
  const int ztile = bidx % g.nzt;
  bidx /= g.nzt;
  const int ytile = bidx % g.nyt;
  bidx /= g.nyt;
  const int xa = bidx * g.xchunk;
  const int xb = min(g.nx, xa + g.xchunk);
  const int zt0 = ztile * TZ, zb = zt0 + tz * VZ;
  const int y0 = ytile * TY, y = y0 + ty;
  const bool yok = y < g.ny;
  const int nvz = yok ? max(0, min(VZ, g.nz - zb)) : 0;
  // halo rows owned by the first/last thread row
  const bool own_hm = (ty == 0), own_hp = (ty == BY - 1);
  const int yhm = y0 - 1, yhp = y0 + TY;
  const int nvhm = (own_hm && yhm >= 0) ? max(0, min(VZ, g.nz - zb)) : 0;
  const int nvhp = (own_hp && yhp < g.ny) ? max(0, min(VZ, g.nz - zb)) : 0;
  const bool own_zl = (tz == 0), own_zr = (tz == BZ - 1);

  auto gidx = [&](int xx, int yy, int zz) -> long long {
    return (long long)xx * g.plane + (long long)yy * g.nz + zz;
  };

  // ---- raw state of the plane in flight
  typename P::Raw R, RHm, RHp;
  typename P::RawS RSl[ZS], RSr[ZS];
  int r_nv = 0, r_nvhm = 0, r_nvhp = 0;
  bool r_zl[ZS], r_zr[ZS];

  auto load_plane = [&](int xp) {
    const bool pv = (xp >= -g.hlo && xp < g.nx + g.hhi);
    r_nv = pv ? nvz : 0;
    r_nvhm = pv ? nvhm : 0;
    r_nvhp = pv ? nvhp : 0;
    if (r_nv > 0) p.load_raw(R, gidx(xp, y, zb), r_nv);
    if (r_nvhm > 0) p.load_raw(RHm, gidx(xp, yhm, zb), r_nvhm);
    if (r_nvhp > 0) p.load_raw(RHp, gidx(xp, yhp, zb), r_nvhp);
#pragma unroll
    for (int j = 0; j < ZS; ++j) {
      const int zl = zt0 - ZS + j, zr = zt0 + TZ + j;
      r_zl[j] = pv && own_zl && yok && zl >= 0;
      r_zr[j] = pv && own_zr && yok && zr < g.nz;
      if (r_zl[j]) p.load_raw_s(RSl[j], gidx(xp, y, zl));
      if (r_zr[j]) p.load_raw_s(RSr[j], gidx(xp, y, zr));
    }
  };

  auto fields = [&](const typename P::Raw& raw, int nv, CT (&f)[NF][VZ]) {
    if constexpr (HasFieldVec<P>::value) {
      if (nv == VZ) {
        p.field_vec(raw, f);
        return;
      }
    }
#pragma unroll
    for (int k = 0; k < VZ; ++k) {
      CT t[NF];
      if (k < nv) {
        p.field(raw, k, t);
      } else {
#pragma unroll
        for (int q = 0; q < NF; ++q) t[q] = CT(0);
      }
#pragma unroll
      for (int q = 0; q < NF; ++q) f[q][k] = t[q];
    }
  };

  // write the in-flight plane (fields already computed for the core) to smem
  auto write_smem = [&](CT* buf, const CT (&fc)[NF][VZ]) {
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      CT* rowc = buf + ((size_t)q * (TY + 2) + (ty + 1)) * ROW + PAD + tz * VZ;
#pragma unroll
      for (int k = 0; k < VZ; ++k) rowc[k] = fc[q][k];
    }
    if (own_hm) {
      CT fh[NF][VZ];
      fields(RHm, r_nvhm, fh);
#pragma unroll
      for (int q = 0; q < NF; ++q) {
        CT* row = buf + ((size_t)q * (TY + 2) + 0) * ROW + PAD + tz * VZ;
#pragma unroll
        for (int k = 0; k < VZ; ++k) row[k] = fh[q][k];
      }
    }
    if (own_hp) {
      CT fh[NF][VZ];
      fields(RHp, r_nvhp, fh);
#pragma unroll
      for (int q = 0; q < NF; ++q) {
        CT* row = buf + ((size_t)q * (TY + 2) + (TY + 1)) * ROW + PAD + tz * VZ;
#pragma unroll
        for (int k = 0; k < VZ; ++k) row[k] = fh[q][k];
      }
    }
    if (own_zl || own_zr) {
#pragma unroll
      for (int j = 0; j < ZS; ++j) {
        CT tl[NF], tr[NF];
        if (r_zl[j]) p.field_s(RSl[j], tl);
        else {
#pragma unroll
          for (int q = 0; q < NF; ++q) tl[q] = CT(0);
        }
        if (r_zr[j]) p.field_s(RSr[j], tr);
        else {
#pragma unroll
          for (int q = 0; q < NF; ++q) tr[q] = CT(0);
        }
#pragma unroll
        for (int q = 0; q < NF; ++q) {
          CT* row = buf + ((size_t)q * (TY + 2) + (ty + 1)) * ROW;
          if (own_zl) row[PAD - ZS + j] = tl[q];
          if (own_zr) row[PAD + TZ + j] = tr[q];
        }
      }
    }
  };

  CT fprev[NF][VZ], fcur[NF][VZ], fnext[NF][VZ];
  typename P::Epi E, En;
  static_assert(NR >= 1, "passes carry at least one reduction slot");
  double red[NR];
#pragma unroll
  for (int s = 0; s < NR; ++s) red[s] = 0.0;

  // ---- prologue: plane xa-1 (core only), plane xa (haloed, smem buffer 0)
  {
    const int xp = xa - 1;
    const int nv = (xp >= -g.hlo) ? nvz : 0;
    typename P::Raw Rp;
    if (nv > 0) p.load_raw(Rp, gidx(xp, y, zb), nv);
    fields(Rp, nv, fprev);
  }
  load_plane(xa);
  fields(R, r_nv, fcur);
  write_smem(sm, fcur);
  load_plane(xa + 1);
  if (nvz > 0) p.load_epi(E, gidx(xa, y, zb), nvz);
  __syncthreads();

  for (int x = xa; x < xb; ++x) {
    CT* bcur = sm + (size_t)((x - xa) & 1) * S::PLANE;
    CT* bnxt = sm + (size_t)(((x - xa) + 1) & 1) * S::PLANE;
    // 1. fields of plane x+1 (raw data loaded one step ago) -> registers + smem
    fields(R, r_nv, fnext);
    write_smem(bnxt, fnext);
    // 2. prefetch plane x+2 and the epilogue inputs of plane x+1
    if (x + 2 <= xb) {
      load_plane(x + 2);
    } else {
      r_nv = r_nvhm = r_nvhp = 0;
#pragma unroll
      for (int j = 0; j < ZS; ++j) r_zl[j] = r_zr[j] = false;
    }
    if (x + 1 < xb && nvz > 0) p.load_epi(En, gidx(x + 1, y, zb), nvz);
    // 3. stencil(s) and epilogue of plane x
    CT st[NF][VZ];
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      const CT* rowm = bcur + ((size_t)q * (TY + 2) + ty) * ROW + PAD + tz * VZ;
      const CT* rowc = rowm + ROW;
      const CT* rowp = rowc + ROW;
      CT left[ZS], right[ZS];
#pragma unroll
      for (int j = 0; j < ZS; ++j) {
        CT fromprev = __shfl_up_sync(0xffffffffu, fcur[q][VZ - ZS + j], 1);
        CT fromnext = __shfl_down_sync(0xffffffffu, fcur[q][j], 1);
        left[j] = (lane == 0) ? rowc[-ZS + j] : fromprev;
        right[j] = (lane == 31) ? rowc[VZ + j] : fromnext;
      }
      if constexpr (HasStencilVec<P>::value) {
        CT ym[VZ], yp[VZ];
#pragma unroll
        for (int k = 0; k < VZ; ++k) {
          ym[k] = rowm[k];
          yp[k] = rowp[k];
        }
        p.stencil_vec(q, fprev[q], ym, fcur[q], left, right, yp, fnext[q], st[q]);
      } else {
#pragma unroll
        for (int k = 0; k < VZ; ++k) {
          const CT zm = (k >= ZS) ? fcur[q][k - ZS] : left[k];
          const CT zp = (k + ZS < VZ) ? fcur[q][k + ZS] : right[k + ZS - VZ];
          const Nb<CT> nb{fprev[q][k], rowm[k], zm, fcur[q][k], zp, rowp[k], fnext[q][k]};
          st[q][k] = p.stencil(q, k, nb, fcur, E);
        }
      }
    }
    if (nvz > 0) p.epilogue(gidx(x, y, zb), nvz, fcur, st, E, red);
    // 4. rotate the register queue
#pragma unroll
    for (int q = 0; q < NF; ++q)
#pragma unroll
      for (int k = 0; k < VZ; ++k) {
        fprev[q][k] = fcur[q][k];
        fcur[q][k] = fnext[q][k];
      }
    E = En;
    __syncthreads();
  }

  if constexpr (P::HAS_RED) {
    double tot[NR];
    int ops[NR];
#pragma unroll
    for (int s = 0; s < NR; ++s) ops[s] = P::op(s);
    if (grid_finish<NR, NT>(red, ops, p.partials, g.pstride, p.ticket, tot)) {
      if (threadIdx.x == 0) finish_pass(p, tot);
    }
  }
}

}  // namespace gadi
