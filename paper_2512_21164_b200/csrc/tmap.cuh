// TMA tensor-map loads for the barrier-free 3-D sweeps (sweep_tma2.cuh).
//
// The row-copy producer issues one cp.async.bulk per stage row and input
// (20 for HcgA, 26 for HcgB per plane of a 256 x 8 tile), and the measured
// pass time follows the number of bulk copies per stage (splitting every
// input row into two copies: HcgA 232 -> 328 us, profiles/tiling_r01.md).
// With a 3-D tensor map per vector the whole (TY+2)-row haloed tile of an
// input is one or two box loads (box width <= 256 elements: 2 x 136 bf16 /
// fp16, 1 x 136 fp32, 1 x 68 fp64) and an epilogue tile one box, so a stage
// is 3-5 loads; rows and columns outside the grid (y-halo at the domain
// edge, z-pads at the first and last tile, planes beyond the slab) arrive
// zero-filled by the hardware.  The maps are encoded on the host
// (cuTensorMapEncodeTiled through the runtime's driver entry point, cached
// per buffer in the context) and passed by value as a __grid_constant__
// kernel parameter, so CUDA-graph capture records them with the launch.
//
// Shared-memory layout of an input with two boxes: box k holds elements
// [k*W/2, (k+1)*W/2) of each of the TY+2 rows, W = TZ + 2*hz; lanes 0-15 of
// a row read box 0 and lanes 16-31 box 1 (their z-edge pads included), so a
// lane's row base pointer selects its box once.
#pragma once
#include <cuda.h>
#include "sweep_tma.cuh"

namespace gadi {

struct TmapSet {
  CUtensorMap in[4];
  CUtensorMap epi[4];
  int ok;
};
struct TmapNone {  // the row-copy instances take no maps (keeps their parameter block small)
  int ok;
};
template <int TM>
using TmParam = typename std::conditional<TM != 0, TmapSet, TmapNone>::type;

// compile-time eligibility: 3-D tiles of 32 lanes per row, and passes with
// at least two haloed inputs (HcgA, CgnrP1).  Measured per pass (cd3d 512^3
// bf16, us): HcgA 232 -> 207, CgnrP1 199 -> 181 with tensor maps, but HcgB
// 262 -> 275-280 and CgnrP2 / CgnrInit / CgnrP3 slower too: for a single
// haloed input the ten parallel row copies finish a stage sooner than its
// two box loads (profiles/tiling_r01.md)
// GADI_TM_SINGLE = 1 (default): passes with ONE haloed input (HcgB, CgnrInit,
// CgnrP2, CgnrP3) load it as tensor-map boxes too (2 box loads per stage
// instead of TY + 2 row copies).  Measured at 512^3 bf16: HcgB 270.6 -> 256.4
// us, CgnrP2 291.9 -> 256.9 us, CgnrInit 290 -> 303 us (profiles/exp_r2e_*.json)
#ifndef GADI_TM_SINGLE
#define GADI_TM_SINGLE 1
#endif
template <class P>
struct TmaTm {
  static constexpr bool value = SweepShape<P>::BZ == 32 && SweepShape<P>::BY > 1 && P::NIN >= (GADI_TM_SINGLE ? 1 : 2);
};
// GADI_TM_EPIBOX = 1: the other 3-D passes with epilogue inputs load those
// as one box each (TM = 2).  Measured: HcgB 263 -> 271 us, CgnrP2 280 ->
// 277 us -- off by default.
#ifndef GADI_TM_EPIBOX
#define GADI_TM_EPIBOX 0
#endif
template <class P>
struct TmaTmEpi {
  static constexpr bool value =
      GADI_TM_EPIBOX && SweepShape<P>::BZ == 32 && SweepShape<P>::BY > 1 && !TmaTm<P>::value && P::NE > 0;
};

// GADI_TALL_EPIBOX = 1: a 16-row (TALL) pass with epilogue inputs loads
// haloed inputs AND epilogue tiles as boxes (TM = 3): 2 * 16 epilogue row
// copies per stage from one producer warp are the alternative
#ifndef GADI_TALL_EPIBOX
#define GADI_TALL_EPIBOX 1
#endif
template <class P>
struct TmaTmBoth {
  static constexpr bool value = GADI_TALL_EPIBOX && TmaTm<P>::value && P::TALL != 0 && P::NE > 0;
};

template <class P, class TS>
struct TmBox {
  static constexpr int W(int j) { return TS::TZ + 2 * TS::hz(P::in_esz(j)); }
  static constexpr int NB(int j) { return W(j) > 256 ? 2 : 1; }
  static constexpr int BW(int j) { return W(j) / NB(j); }
};

#ifndef GADI_TM_EVICT_FIRST
#define GADI_TM_EVICT_FIRST 0
#endif
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
#if GADI_TM_EVICT_FIRST
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
  return;
#endif
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// Producer warp with tensor maps.  TM = 1: the haloed inputs load as boxes
// (lane 0) and the epilogue inputs as bulk row copies (lanes in parallel);
// TM = 2: the haloed inputs as row copies and each epilogue input as one
// [TY][TZ] box.  Same ring protocol and plane sequence as produce_stages
// (sweep_tma.cuh); lane 0 posts the stage's byte count (whole boxes, their
// zero-filled parts included; row copies clipped to the grid) first.
template <class P, class TS, int TM>
__device__ __forceinline__ void produce_stages_tm(const P& p, const SweepGeom& g, unsigned char* stages,
                                                  uint64_t* full, uint64_t* empty, int lane, const TmapSet& tm) {
  constexpr int TZ = TS::TZ, TY = TS::TY, NIN = P::NIN, NE = P::NE, NST = TS::NST;
  // TM 1: haloed inputs as boxes, epilogue rows copied; 2: the reverse;
  // 3: both as boxes (no row copies)
  constexpr bool INB = TM == 1 || TM == 3, EPB = TM == 2 || TM == 3;
  constexpr int NRC = TM == 1 ? NE * TY : (TM == 2 ? NIN * (TY + 2) : 0);  // row copies per stage
  using B = TmBox<P, TS>;
  SegIter it(g, gridDim.x, blockIdx.x);
  int tile, xa, xb;
  int gs = 0, slot = 0, round = 0;
  while (it.next(tile, xa, xb)) {
    const int zt0 = (tile % g.nzt) * TZ, y0 = (tile / g.nzt) * TY;
    for (int xp = xa - 1; xp <= xb; ++xp, ++gs) {
      const int st = slot;
      if (gs >= NST) mbar_wait(&empty[st], (unsigned)((round - 1) & 1));
      if (++slot == NST) {
        slot = 0;
        ++round;
      }
      if (p.wave && xp - p.wlead >= 0) {
        if (lane == 0) {
          const volatile unsigned* cnt = p.wave + (xp - p.wlead);
          while (*cnt < gridDim.x) __nanosleep(100);
        }
        __syncwarp();
      }
      const bool pv = (xp >= -g.hlo && xp < g.nx + g.hhi);
      const bool ev = pv && xp >= xa && xp < xb;
      const int xc = xp + g.hlo;  // the maps start at the lowest valid plane
      const int nyv = min(TY, g.ny - y0);                  // valid epilogue rows
      const int ylo = max(y0 - 1, 0), yhi = min(y0 + TY + 1, g.ny);  // valid haloed rows
      if (lane == 0) {
        unsigned bytes = 0;
        if (pv) {
#pragma unroll
          for (int j = 0; j < NIN; ++j) {
            if (!p.in_active(j)) continue;
            const int esz = P::in_esz(j), hz = TS::hz(esz);
            if (INB)
              bytes += (unsigned)((TY + 2) * B::W(j) * esz);
            else
              bytes += (unsigned)((yhi - ylo) * (min(zt0 + TZ + hz, g.nz) - max(zt0 - hz, 0)) * esz);
          }
          if (ev) {
#pragma unroll
            for (int j = 0; j < NE; ++j)
              bytes += (unsigned)((EPB ? TY : nyv) * (EPB ? TZ : min(zt0 + TZ, g.nz) - zt0) * P::epi_esz(j));
          }
        }
        mbar_expect_tx(&full[st], bytes);
        if (pv && INB) {
#pragma unroll
          for (int j = 0; j < NIN; ++j) {
            if (!p.in_active(j)) continue;
            const int hz = TS::hz(P::in_esz(j));
#pragma unroll
            for (int k = 0; k < B::NB(j); ++k)
              tma_load_3d(stages + (size_t)st * TS::STAGE + TS::in_box_off(j, k), &tm.in[j], zt0 - hz + k * B::BW(j),
                          y0 - 1, xc, &full[st]);
          }
        }
        if (ev && EPB) {
#pragma unroll
          for (int j = 0; j < NE; ++j) tma_load_3d(TS::epi_row_ptr(stages, st, j, 0), &tm.epi[j], zt0, y0, xc, &full[st]);
        }
      }
      __syncwarp();
      // row copies, one per lane
      if (NRC > 0 && (TM == 1 ? ev : pv)) {
        for (int q = lane; q < NRC; q += 32) {
          if constexpr (TM == 1) {
            const int j = q / TY, yy = y0 + q % TY;
            if (yy >= g.ny) continue;
            const int esz = P::epi_esz(j);
            const unsigned char* base = reinterpret_cast<const unsigned char*>(p.epi_ptr(j));
            bulk_g2s(TS::epi_row_ptr(stages, st, j, q % TY),
                     base + ((long long)xp * g.plane + (long long)yy * g.nz + zt0) * esz,
                     (unsigned)((min(zt0 + TZ, g.nz) - zt0) * esz), &full[st]);
          } else {
            const int j = q / (TY + 2), r = q % (TY + 2), yy = y0 - 1 + r;
            if (!p.in_active(j) || yy < 0 || yy >= g.ny) continue;
            const int esz = P::in_esz(j), hz = TS::hz(esz);
            const int a = max(zt0 - hz, 0), b = min(zt0 + TZ + hz, g.nz);
            const unsigned char* base = reinterpret_cast<const unsigned char*>(p.in_ptr(j));
            bulk_g2s(TS::in_row_ptr(stages, st, j, r, 0) + (a - zt0) * esz,
                     base + ((long long)xp * g.plane + (long long)yy * g.nz + a) * esz, (unsigned)((b - a) * esz),
                     &full[st]);
          }
        }
      }
    }
  }
}

}  // namespace gadi
