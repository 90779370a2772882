// Barrier-free consumer form of the TMA sweep (default; GADI_TMA2=0 selects
// the f-plane form of sweep_tma.cuh).
//
// The f-plane form computes each plane's stencil fields once, stores them to
// a shared-memory plane (plus two halo warps for the y-halo rows) and
// synchronises all consumer warps at every plane.  Here a consumer reads
// everything it needs straight from the TMA stage ring, which already holds
// the (TY+2) haloed rows of every input: its own row's fields for x+1 (kept
// in the 3-plane register queue), the y-neighbour rows' fields recomputed
// from their raw inputs, the z-edge scalars from the row pads.  The stages
// are read-only, so there is no named barrier, no halo warp and no f-plane
// buffer: each warp only waits on the stage it needs and releases it when
// done, and warps drift freely inside the ring.  Field recomputation costs
// ALU (two extra field evaluations per element) that the barrier stalls of
// the f-plane form cost in issue slots.
#pragma once
#include "sweep_tma.cuh"
#include "tmap.cuh"
#include "strict.cuh"

namespace gadi {

// GADI_EPI_LDG: consumers load the epilogue-only inputs (no halo) with
// 16-byte global loads one plane ahead instead of through the TMA ring
#ifndef GADI_EPI_LDG
#define GADI_EPI_LDG 0
#endif

// In-place fields (GADI_INPLACE, passes declaring INPLACE): for passes whose
// field is a rounded function of its raw inputs (HcgA, CgnrP1: p <- r + beta p,
// rounded to u_s), each consumer warp writes its own row's field back over
// the raw p row of the stage it has just computed it from, and one helper
// warp does the same for the tile's two y-halo rows.  The y-neighbour fields
// are then loaded instead of recomputed (one field evaluation per element
// instead of three).  A third mbarrier per slot ("fields written", all
// consumer warps + helper) orders the writes before the neighbour reads; a
// warp writes plane x+1 before it waits for plane x, so the wait is lagged by
// one plane and rarely stalls.
// GADI_ZPAD_FIELDS (in-place passes): the helper warp also writes the fields
// of the tile's two z-pad columns
#ifndef GADI_ZPAD_FIELDS
#define GADI_ZPAD_FIELDS 1
#endif
#ifndef GADI_XUNROLL
#define GADI_XUNROLL 1
#endif
#ifndef GADI_INPLACE
#define GADI_INPLACE 1
#endif
template <class P, class = void>
struct HasInplace : std::false_type {};
template <class P>
struct HasInplace<P, std::void_t<decltype(P::INPLACE)>>
    : std::integral_constant<bool, P::INPLACE && GADI_INPLACE != 0 && P::NF == 1 && (SweepShape<P>::BY > 1)> {};

// Passes with a field-time side update of their own rows (HcgA under
// GADI_ZLAG: z += alpha p_in, passes.cuh); barrier-free form only.
template <class P, class = void>
struct HasSide : std::false_type {};
template <class P>
struct HasSide<P, std::void_t<decltype(P::SIDE)>> : std::integral_constant<bool, P::SIDE> {};

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// address of element 0 (of the tile core) of row r of input j in stage st,
// as seen by lane tz (tensor-map layout: the lane's box)
template <class P, class TS>
__device__ __forceinline__ unsigned char* stage_in_row(unsigned char* stages, int st, int j, int r, int tz) {
  return TS::in_row_ptr(stages, st, j, r, tz);
}

// field of one lane's VZ-vector at row r of stage st (zeros unless ok)
template <class P, class TS>
__device__ __forceinline__ void stage_fields(const P& p, unsigned char* stages, int st, int r, int zo, bool ok,
                                             typename P::CT (&f)[P::NF][SweepShape<P>::VZ]) {
  using CT = typename P::CT;
  constexpr int VZ = SweepShape<P>::VZ;
  if (ok) {
    SmRow R;
#pragma unroll
    for (int j = 0; j < 4; ++j) R.p[j] = nullptr;
#pragma unroll
    for (int j = 0; j < P::NIN; ++j) R.p[j] = stage_in_row<P, TS>(stages, st, j, r, zo / VZ);
    typename P::Raw a;
    p.load_raw_sm(a, R, zo);
    p.field_vec(a, f);
  } else {
#pragma unroll
    for (int k = 0; k < VZ; ++k) f[0][k] = CT(0);
  }
}

// the helper warp of the in-place form: fields of the tile's two y-halo rows
// (stage rows 0 and TY+1) for every plane whose stencils the CTA computes
template <class P, class TS>
__device__ void inplace_halo_rows(const P& p, const SweepGeom& g, unsigned char* stages, uint64_t* full,
                                  uint64_t* empty, uint64_t* fdone, int lane) {
  using CT = typename P::CT;
  using ST = typename P::ST;
  constexpr int VZ = SweepShape<P>::VZ, TZ = SweepShape<P>::TZ, TY = SweepShape<P>::TY, NST = TS::NST;
  constexpr int BZ_ = SweepShape<P>::BZ;
  SegIter it(g, gridDim.x, blockIdx.x);
  int tile, xa, xb;
  int gs = 0;
  while (it.next(tile, xa, xb)) {
    const int zt0 = (tile % g.nzt) * TZ, y0 = (tile / g.nzt) * TY;
    const bool zok = zt0 + lane * VZ < g.nz;
    const bool top_ok = zok && y0 - 1 >= 0;
    const bool bot_ok = zok && y0 + TY < g.ny;
    int slot = gs % NST;
    unsigned ph = (unsigned)((gs / NST) & 1);
    for (int x = xa - 1; x <= xb; ++x) {
      mbar_wait(&full[slot], ph);
      if (x >= xa && x < xb) {
        CT f[1][VZ];
        stage_fields<P, TS>(p, stages, slot, 0, lane * VZ, top_ok, f);
        store_exact<ST, VZ>(reinterpret_cast<ST*>(stage_in_row<P, TS>(stages, slot, P::FIELD_IN, 0, lane)), lane * VZ,
                          VZ, f[0], true);
        stage_fields<P, TS>(p, stages, slot, TY + 1, lane * VZ, bot_ok, f);
        store_exact<ST, VZ>(reinterpret_cast<ST*>(stage_in_row<P, TS>(stages, slot, P::FIELD_IN, TY + 1, lane)),
                          lane * VZ, VZ, f[0], true);
#if GADI_ZPAD_FIELDS
        // the z-neighbour fields just outside the tile (columns -1 and TZ) of
        // every row, so the consumers' edge lanes load them instead of
        // evaluating the field in a divergent branch
        for (int q = lane; q < 2 * (TY + 2); q += 32) {
          const int r = q >> 1, right = q & 1;
          const int tzl = right ? BZ_ - 1 : 0, zo = right ? TZ : -1;
          const int zz = zt0 + zo, yy = y0 - 1 + r;
          const bool ok = zz >= 0 && zz < g.nz && yy >= 0 && yy < g.ny;
          CT fs[1];
          if (ok) {
            SmRow R;
#pragma unroll
            for (int j = 0; j < 4; ++j) R.p[j] = nullptr;
#pragma unroll
            for (int j = 0; j < P::NIN; ++j) R.p[j] = stage_in_row<P, TS>(stages, slot, j, r, tzl);
            typename P::RawS a;
            p.load_raw_s_sm(a, R, zo);
            p.field_s(a, fs);
          } else {
            fs[0] = CT(0);
          }
          reinterpret_cast<ST*>(stage_in_row<P, TS>(stages, slot, P::FIELD_IN, r, tzl))[zo] = Store<ST>::from(fs[0]);
        }
#endif
        fence_proxy_async_smem();
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&fdone[slot]);
        mbar_arrive(&empty[slot]);
      }
      if (++slot == NST) {
        slot = 0;
        ph ^= 1u;
      }
    }
    gs += xb - xa + 2;
  }
}

template <class P>
struct Tma2Threads {
  static constexpr int value = P::NT + 32 + (HasInplace<P>::value ? 32 : 0);
};

// Stage layouts: TM = false, rows of (TZ + 2 hz) elements per input (the
// row-copy producer); TM = true, the tensor-map boxes of tmap.cuh, each box
// 128-byte aligned.
template <class P, int TM = 0>
struct TmaShape2 : TmaShape<P> {
  using Base = TmaShape<P>;
  using BX = TmBox<P, Base>;
  static constexpr int TZ = Base::TZ, TY = Base::TY;
  static constexpr int r128(int b) { return (b + 127) / 128 * 128; }
  static constexpr int boxb(int j) { return r128((TY + 2) * BX::BW(j) * P::in_esz(j)); }
  static constexpr int off_in_tm(int j) {
    int o = 0;
    for (int i = 0; i < j; ++i) o += BX::NB(i) * boxb(i);
    return o;
  }
  static constexpr int off_epi_tm(int j) {
    int o = (TM == 1 || TM == 3) ? off_in_tm(P::NIN) : r128(Base::off_in(P::NIN));
    for (int i = 0; i < j; ++i) o += r128(TY * TZ * P::epi_esz(i));
    return o;
  }
  static constexpr int STAGE = TM ? r128(off_epi_tm(P::NE)) : Base::STAGE;
  static constexpr int in_box_off(int j, int k) { return off_in_tm(j) + k * boxb(j); }
  static __device__ __forceinline__ unsigned char* in_row_ptr(unsigned char* stages, int st, int j, int r, int tz) {
    const int esz = P::in_esz(j), hz = Base::hz(esz);
    unsigned char* sb = stages + (size_t)st * STAGE;
    if constexpr (TM == 1 || TM == 3) {
      const int k = (BX::NB(j) == 2 && tz >= 16) ? 1 : 0;
      return sb + in_box_off(j, k) + r * BX::BW(j) * esz + (hz - k * BX::BW(j)) * esz;
    } else {
      return sb + Base::off_in(j) + r * Base::rb_in(j) + hz * esz;
    }
  }
  static __device__ __forceinline__ unsigned char* epi_row_ptr(unsigned char* stages, int st, int j, int r) {
    unsigned char* sb = stages + (size_t)st * STAGE;
    if constexpr (TM) return sb + off_epi_tm(j) + r * TZ * P::epi_esz(j);
    else return sb + Base::off_epi(j) + r * Base::rb_epi(j);
  }
  static constexpr int BUDGET = (P::MINB >= 3 ? GADI_TMA_BUDGET_KB : (P::MINB == 2 ? GADI_TMA_BUDGET1_KB : GADI_TMA_BUDGET_TALL_KB)) * 1024;
  static constexpr int NST_RAW = BUDGET / STAGE;
  static constexpr int NST = NST_RAW < 2 ? 2 : (NST_RAW > 12 ? 12 : NST_RAW);
  static constexpr size_t SMEM = (size_t)NST * STAGE + 3 * NST * sizeof(uint64_t);
};

template <class P, int TM>
__global__ void __launch_bounds__(Tma2Threads<P>::value, P::MINB)
    sweep_tma2_kernel(P p, const __grid_constant__ TmParam<TM> tm) {
  using S = SweepShape<P>;
  using TS = TmaShape2<P, TM>;
  using CT = typename P::CT;
  constexpr int VZ = S::VZ, BZ = S::BZ, BY = S::BY, ZS = S::ZS, NF = S::NF;
  constexpr int TZ = S::TZ, TY = S::TY;
  constexpr int NR = P::NR, NT = P::NT, NIN = P::NIN, NE = P::NE, NST = TS::NST;
  constexpr int NWCONS = NT / 32;
  constexpr bool INPL = HasInplace<P>::value;
  constexpr int NPART = NWCONS + (INPL ? 1 : 0);  // warps that release a stage
  static_assert(NIN <= 4 && NE <= 4, "at most four inputs of each kind");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* stages = smem_raw;
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + (size_t)NST * TS::STAGE);
  uint64_t* empty = full + NST;
  uint64_t* fdone = empty + NST;

  if (!p.prepare()) return;
  const SweepGeom g = p.g;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NPART);
      mbar_init(&fdone[s], NPART);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double red[NR];
#pragma unroll
  for (int s = 0; s < NR; ++s) red[s] = 0.0;
  if (p.wave)
    for (int i = blockIdx.x * (NT + 32) + tid; i < g.nx; i += gridDim.x * (NT + 32)) p.wave_clear[i] = 0u;

  if (tid >= NT + (INPL ? 32 : 0)) {
    if constexpr (TM != 0)
      produce_stages_tm<P, TS, TM>(p, g, stages, full, empty, lane, tm);
    else
      produce_stages<P, TS, !GADI_EPI_LDG>(p, g, stages, full, empty, lane);
  } else if (INPL && tid >= NT) {
    if constexpr (INPL) inplace_halo_rows<P, TS>(p, g, stages, full, empty, fdone, lane);
  } else {
    const int tz = tid % BZ, ty = tid / BZ;
    // stages are addressed by ring slot; (slot, phase) advance incrementally
    struct Pos {
      int slot;
      unsigned ph;
      __device__ void next() {
        if (++slot == NST) {
          slot = 0;
          ph ^= 1u;
        }
      }
    };
    auto in_row = [&](int st, int r) {
      SmRow R;
#pragma unroll
      for (int j = 0; j < 4; ++j) R.p[j] = nullptr;
#pragma unroll
      for (int j = 0; j < NIN; ++j) R.p[j] = TS::in_row_ptr(stages, st, j, r, tz);
      return R;
    };
    auto epi_row = [&](int st, int r) {
      SmRow R;
#pragma unroll
      for (int j = 0; j < 4; ++j) R.p[j] = nullptr;
#pragma unroll
      for (int j = 0; j < NE; ++j) R.p[j] = TS::epi_row_ptr(stages, st, j, r);
      return R;
    };
    // fields of this lane's vector in stage row r; zeros unless valid (nv == VZ)
    auto fields_at = [&](int st, int r, bool ok, CT (&f)[NF][VZ]) {
      if (ok) {
        typename P::Raw a;
        p.load_raw_sm(a, in_row(st, r), tz * VZ);
        if constexpr (HasFieldVec<P>::value) {
          p.field_vec(a, f);
        } else {
#pragma unroll
          for (int k = 0; k < VZ; ++k) {
            CT t[NF];
            p.field(a, k, t);
#pragma unroll
            for (int q = 0; q < NF; ++q) f[q][k] = t[q];
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < VZ; ++k)
#pragma unroll
          for (int q = 0; q < NF; ++q) f[q][k] = CT(0);
      }
    };
    // fields of this lane's own row (stage row ty + 1), plus the pass's side
    // update of the owned plane (element index i) when `side`
    auto own_fields_at = [&](int st, bool ok, bool side, long long i, CT (&f)[NF][VZ]) {
      if constexpr (HasSide<P>::value) {
        static_assert(!GADI_EPI_LDG, "side updates read the staged epilogue row");
        if (ok) {
          typename P::Raw a;
          p.load_raw_sm(a, in_row(st, ty + 1), tz * VZ);
          p.field_vec(a, f);
          if (side) p.side(a, epi_row(st, ty), tz * VZ, i);
        } else {
#pragma unroll
          for (int k = 0; k < VZ; ++k) f[0][k] = CT(0);
        }
      } else {
        fields_at(st, ty + 1, ok, f);
      }
    };
    // scalar field at element offset zo of stage row r (z-edges)
    auto field_scalar = [&](int st, int r, int zo, bool ok, CT (&f)[NF]) {
      if (ok) {
        typename P::RawS a;
        p.load_raw_s_sm(a, in_row(st, r), zo);
        p.field_s(a, f);
      } else {
#pragma unroll
        for (int q = 0; q < NF; ++q) f[q] = CT(0);
      }
    };
    auto release = [&](const Pos& q) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[q.slot]);
    };
    auto wait_full = [&](const Pos& q) { mbar_wait(&full[q.slot], q.ph); };
    // in-place form: publish this row's field of stage st over its raw p row
    auto put_field = [&](int st, const CT (&f)[NF][VZ]) {
      if constexpr (INPL) {
        using ST = typename P::ST;
        store_exact<ST, VZ>(reinterpret_cast<ST*>(stage_in_row<P, TS>(stages, st, P::FIELD_IN, ty + 1, tz)), tz * VZ, VZ,
                          f[0], true);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&fdone[st]);
      }
    };

    SegIter it(g, gridDim.x, blockIdx.x);
    int tile, xa, xb;
    int gs = 0;  // stage sequence number of plane xa-1 of the current segment
    while (it.next(tile, xa, xb)) {
      const int zt0 = (tile % g.nzt) * TZ, y0 = (tile / g.nzt) * TY;
      const int zb = zt0 + tz * VZ;
      const int y = y0 + ty;
      const bool yok = y < g.ny;
      const bool own = yok && zb < g.nz;  // nz % VZ == 0 on this path
      const bool ym_ok = BY > 1 && own && y - 1 >= 0;
      const bool yp_ok = BY > 1 && own && y + 1 < g.ny;
      const long long rowbase = (long long)y * g.nz + zb;

      CT fprev[NF][VZ], fcur[NF][VZ], fnext[NF][VZ];
      Pos ps{gs % NST, (unsigned)((gs / NST) & 1)};  // plane xa-1
      wait_full(ps);
      fields_at(ps.slot, ty + 1, own && xa - 1 >= -g.hlo, fprev);
      if constexpr (INPL) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&fdone[ps.slot]);
      }
      release(ps);
      ps.next();  // plane xa
      wait_full(ps);
      long long gidx = (long long)xa * g.plane + rowbase;
      own_fields_at(ps.slot, own, own, gidx, fcur);
      put_field(ps.slot, fcur);
      Pos pn = ps;

#if GADI_EPI_LDG
      typename P::Epi En;
      if (own) p.load_epi(En, gidx, VZ);
#endif
      // GADI_XUNROLL = 3 unrolls the plane loop by the depth of the register
      // queue (fprev / fcur / fnext), letting the compiler rename instead of
      // moving the queue every plane
      // 16-row (TALL) passes unroll by 3 at any GADI_XUNROLL: with their
      // register headroom the renaming pays (HcgA 196.5 -> 189.6 us); at 3
      // CTAs per SM it does not (profiles/ab_xunroll_r2.jsonl)
      constexpr int XU = P::TALL ? 3 : GADI_XUNROLL;
#pragma unroll XU
      for (int x = xa; x < xb; ++x, gidx += g.plane) {
        const int s = ps.slot;  // stage slot of plane x
        pn.next();              // plane x+1
        wait_full(pn);
        own_fields_at(pn.slot, own && x + 1 < g.nx + g.hhi, own && x + 1 < xb, gidx + g.plane, fnext);
        put_field(pn.slot, fnext);
        CT fym[NF][VZ], fyp[NF][VZ];
        if constexpr (INPL) {
          // neighbours' fields of plane x (written one plane ago)
          mbar_wait(&fdone[s], ps.ph);
          lds_vec<typename P::ST, VZ>(stage_in_row<P, TS>(stages, s, P::FIELD_IN, ty, tz), tz * VZ, fym[0]);
          lds_vec<typename P::ST, VZ>(stage_in_row<P, TS>(stages, s, P::FIELD_IN, ty + 2, tz), tz * VZ, fyp[0]);
        } else {
          fields_at(s, ty, ym_ok, fym);
          fields_at(s, ty + 2, yp_ok, fyp);
        }
        typename P::Epi E;
#if GADI_EPI_LDG
        E = En;
        if (own && x + 1 < xb) p.load_epi(En, gidx + g.plane, VZ);
#else
        p.load_epi_sm(E, epi_row(s, ty), tz * VZ);
#endif
        if constexpr (HasEpiV<P>::value) {
          if (own) p.load_epi_v(E, gidx, VZ);
        }
        CT st[NF][VZ];
        // z-neighbours: shuffles inside a warp, the stage row at warp edges
        CT zl[ZS][NF], zr[ZS][NF];
        if constexpr (INPL && GADI_ZPAD_FIELDS && ZS == 1 && NF == 1) {
          // the helper warp wrote the tile's z-pad fields in place (columns
          // -1 and TZ); interior warp edges read the neighbour lane's field row
          using ST = typename P::ST;
          const ST* row = reinterpret_cast<const ST*>(stage_in_row<P, TS>(stages, s, P::FIELD_IN, ty + 1, tz));
          zl[0][0] = (lane == 0) ? cvt_in<CT>(row[tz * VZ - 1]) : CT(0);
          zr[0][0] = (lane == 31) ? cvt_in<CT>(row[tz * VZ + VZ]) : CT(0);
        } else {
#pragma unroll
          for (int j = 0; j < ZS; ++j) {
            field_scalar(s, ty + 1, tz * VZ - ZS + j, lane == 0 && own && zb - ZS + j >= 0, zl[j]);
            field_scalar(s, ty + 1, tz * VZ + VZ + j, lane == 31 && own && zb + VZ + j < g.nz, zr[j]);
          }
        }
#pragma unroll
        for (int q = 0; q < NF; ++q) {
          CT left[ZS], right[ZS];
#pragma unroll
          for (int j = 0; j < ZS; ++j) {
            const CT fromprev = __shfl_up_sync(0xffffffffu, fcur[q][VZ - ZS + j], 1);
            const CT fromnext = __shfl_down_sync(0xffffffffu, fcur[q][j], 1);
            left[j] = (lane == 0) ? zl[j][q] : fromprev;
            right[j] = (lane == 31) ? zr[j][q] : fromnext;
          }
          if constexpr (HasStencilVec<P>::value) {
            p.stencil_vec(q, fprev[q], fym[q], fcur[q], left, right, fyp[q], fnext[q], st[q]);
          } else {
#pragma unroll
            for (int k = 0; k < VZ; ++k) {
              const CT zm = (k >= ZS) ? fcur[q][k - ZS] : left[k];
              const CT zp = (k + ZS < VZ) ? fcur[q][k + ZS] : right[k + ZS - VZ];
              const Nb<CT> nb{fprev[q][k], fym[q][k], zm, fcur[q][k], zp, fyp[q][k], fnext[q][k]};
              st[q][k] = p.stencil(q, k, nb, fcur, E);
            }
          }
        }
        if (own) p.epilogue(gidx, VZ, fcur, st, E, red);
        if constexpr (TreeSlot<P>::value >= 0) {
          // reference rounding: this warp's aligned fl_dot blocks (strict.cuh)
          if (p.tout.tlog >= 0) {
            tree_emit<VZ, (ZS == 2 ? 1 : 0)>(p.tout, gidx, own, lane, red[TreeSlot<P>::value]);
            red[TreeSlot<P>::value] = 0.0;
          }
        }
#pragma unroll
        for (int q = 0; q < NF; ++q)
#pragma unroll
          for (int k = 0; k < VZ; ++k) {
            fprev[q][k] = fcur[q][k];
            fcur[q][k] = fnext[q][k];
          }
        release(ps);
        ps = pn;
        if (p.wave && tid == 0) {
          __threadfence();
          atomicAdd(p.wave + x, 1u);
        }
      }
      release(ps);  // plane xb
      gs += xb - xa + 2;
    }
  }

  if constexpr (P::HAS_RED) {
    double tot[NR];
    int ops[NR];
#pragma unroll
    for (int s = 0; s < NR; ++s) ops[s] = P::op(s);
    if (grid_finish<NR, P::NT + 32>(red, ops, p.partials, g.pstride, p.ticket, tot)) {
      if (threadIdx.x == 0) finish_pass(p, tot);
    }
  }
}

}  // namespace gadi
