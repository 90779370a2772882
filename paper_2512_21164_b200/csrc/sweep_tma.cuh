// Warp-specialised, TMA-fed version of the 2.5-D stencil sweep (sweep.cuh).
//
// One producer warp streams every plane a CTA needs into a ring of NST
// shared-memory stages with cp.async.bulk (the TMA bulk-copy engine,
// SASS UBLKCP) completing on per-stage mbarriers; the consumer warps never
// issue global loads for the stencil inputs, so the number of bytes in
// flight is set by the ring depth, not by registers.  A stage holds, for one
// x-plane, the (TY+2) haloed rows of every stencil input (each row padded by
// 16 bytes on both sides so every bulk copy is 16-byte aligned) and the TY
// core rows of every epilogue input.
//
// Consumers keep the register queue (x-neighbours), the f-plane double
// buffer (y-neighbours) and warp shuffles (z-neighbours) of sweep.cuh; they
// synchronise among themselves with a named barrier and hand stages back to
// the producer through "empty" mbarriers.  Out-of-grid rows / planes are
// simply not copied and are masked by coordinates, so stage contents beyond
// the grid are never read.  Requires every input row to start 16-byte
// aligned (nz * elem_size % 16 == 0) and arrays padded on both sides
// (the context allocates every vector with guard bands).
#pragma once
#include "sweep.cuh"

namespace gadi {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp is parked by the
// hardware until the phase completes (or the hint expires) instead of
// spinning and taking issue slots from the warps that have work
#ifndef GADI_MBAR_SUSPEND_NS
#define GADI_MBAR_SUSPEND_NS 1000000
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
#if GADI_MBAR_SUSPEND_NS > 0
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity), "n"(GADI_MBAR_SUSPEND_NS)
      : "memory");
#else
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// GADI_L2PF > 0: the producer also prefetches the rows of plane xp + L2PF
// into L2 (more DRAM requests in flight than the stage ring holds)
#ifndef GADI_L2PF
#define GADI_L2PF 0
#endif
#ifndef GADI_SPLITCOPY
#define GADI_SPLITCOPY 0  // experiment: two bulk copies per input row
#endif
__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// per-row pointers handed to the pass loaders: element 0 of the tile core
struct SmRow {
  const unsigned char* p[4];
};

template <class T, int VZ, class CT>
__device__ __forceinline__ void lds_vec(const unsigned char* row, int zoff, CT (&out)[VZ]) {
  const T* q = reinterpret_cast<const T*>(row) + zoff;
  constexpr int BYTES = VZ * (int)sizeof(T);
  if constexpr (std::is_same<T, bf16>::value && std::is_same<CT, float>::value && BYTES % 16 == 0) {
#pragma unroll
    for (int c = 0; c < BYTES / 16; ++c) {
      const uint4 u = reinterpret_cast<const uint4*>(q)[c];
      const unsigned w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        out[c * 8 + 2 * j] = bf_lo(w[j]);
        out[c * 8 + 2 * j + 1] = bf_hi(w[j]);
      }
    }
  } else if constexpr (BYTES % 16 == 0) {
    constexpr int PER = 16 / (int)sizeof(T);
#pragma unroll
    for (int c = 0; c < BYTES / 16; ++c) {
      const uint4 u = reinterpret_cast<const uint4*>(q)[c];
      const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
      for (int j = 0; j < PER; ++j) out[c * PER + j] = cvt_in<CT>(e[j]);
    }
  } else if constexpr (BYTES == 8) {
    const uint2 u = *reinterpret_cast<const uint2*>(q);
    const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int j = 0; j < VZ; ++j) out[j] = cvt_in<CT>(e[j]);
  } else if constexpr (BYTES == 4) {
    const unsigned u = *reinterpret_cast<const unsigned*>(q);
    const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int j = 0; j < VZ; ++j) out[j] = cvt_in<CT>(e[j]);
  } else {
#pragma unroll
    for (int j = 0; j < VZ; ++j) out[j] = cvt_in<CT>(q[j]);
  }
}
template <class T, class CT>
__device__ __forceinline__ CT lds1(const unsigned char* row, int zoff) {
  return cvt_in<CT>(reinterpret_cast<const T*>(row)[zoff]);
}

template <class P> struct TmaShape {
  using B = SweepShape<P>;
  static constexpr int TZ = B::TZ, TY = B::TY;
  static constexpr int hz(int esz) { return 16 / esz; }
  static constexpr int rb_in(int j) { return (TZ + 2 * hz(P::in_esz(j))) * P::in_esz(j); }
  static constexpr int rb_epi(int j) { return TZ * P::epi_esz(j); }
  static constexpr int off_in(int j) {
    int o = 0;
    for (int i = 0; i < j; ++i) o += (TY + 2) * rb_in(i);
    return o;
  }
  static constexpr int off_epi(int j) {
    int o = off_in(P::NIN);
    for (int i = 0; i < j; ++i) o += TY * rb_epi(i);
    return o;
  }
  static constexpr int STAGE = off_epi(P::NE);
  static constexpr int FBYTES = (int)B::SMEM;  // two f-plane buffers
#ifndef GADI_TMA_BUDGET_KB
#define GADI_TMA_BUDGET_KB 74  // smem per CTA for passes run 3 per SM
#endif
#ifndef GADI_TMA_BUDGET1_KB
#define GADI_TMA_BUDGET1_KB 110  // passes budgeted for 2 CTAs per SM
#endif
#ifndef GADI_TMA_BUDGET_TALL_KB
#define GADI_TMA_BUDGET_TALL_KB 200  // one CTA per SM (GeoT TALL)
#endif
  static constexpr int BUDGET = (P::MINB >= 3 ? GADI_TMA_BUDGET_KB : (P::MINB == 2 ? GADI_TMA_BUDGET1_KB : GADI_TMA_BUDGET_TALL_KB)) * 1024;
  static constexpr int NST_RAW = (BUDGET - FBYTES) / STAGE;
  // a power of two: the consumers index the ring with % and / NST
  static constexpr int NST = NST_RAW >= 8 ? 8 : (NST_RAW >= 4 ? 4 : 2);
  static constexpr size_t SMEM = (size_t)FBYTES + (size_t)NST * STAGE + 2 * NST * sizeof(uint64_t);
};

// Threads: NT compute threads (BZ x BY), NH halo warps (3-D: one per y-halo
// row, so the compute warps stay balanced), one producer warp.
template <class P> struct TmaThreads {
  static constexpr int NH = P::BY > 1 ? 2 : 0;
  static constexpr int NCONS = P::NT + 32 * NH;  // consumer threads
  static constexpr int NTOT = NCONS + 32;
};

// Work decomposition: the (tile, x-plane) units are split into gridDim.x
// equal contiguous ranges (one CTA per resident slot, a single wave); a
// range is a list of x-segments of at most a few tiles.  Every segment
// re-primes the register queue from planes xa-1, xa; the stage ring and the
// mbarrier phases run on across segments.
struct SegIter {
  long long u, u1;
  int nx, tiles;
  __device__ SegIter(const SweepGeom& g, int nblocks, int b) {
    nx = g.nx;
    tiles = g.nzt * g.nyt;
    const long long T = (long long)tiles * nx;
    const long long W = (T + nblocks - 1) / nblocks;
    u = (long long)b * W;
    u1 = min(T, u + W);
  }
  __device__ bool next(int& tile, int& xa, int& xb) {
    if (u >= u1) return false;
    tile = (int)(u / nx);
    xa = (int)(u % nx);
    xb = (int)min((long long)nx, xa + (u1 - u));
    u += xb - xa;
    return true;
  }
};

// The producer warp: streams every plane of this CTA's segments into the
// stage ring (one bulk copy per row and input, issued one row per lane; lane
// 0 posts the byte count first).  Shared by both consumer designs.
template <class P, class TS, bool EPI = true>
__device__ __forceinline__ void produce_stages(const P& p, const SweepGeom& g, unsigned char* stages, uint64_t* full,
                                               uint64_t* empty, int lane) {
  constexpr int TZ = TS::TZ, TY = TS::TY, NIN = P::NIN, NE = EPI ? P::NE : 0, NST = TS::NST;
  constexpr int NCOPY = NIN * (TY + 2) + NE * TY;
  SegIter it(g, gridDim.x, blockIdx.x);
  int tile, xa, xb;
  int gs = 0, slot = 0, round = 0;
  while (it.next(tile, xa, xb)) {
    const int zt0 = (tile % g.nzt) * TZ, y0 = (tile / g.nzt) * TY;
    // Row spans clipped to the grid row [0, nz): the 16-byte pads and the
    // part of a last partial tile past nz are never read by the consumers,
    // and at a row boundary they would pull extra DRAM lines.  zt0, nz and
    // the pads are 16-byte multiples on this path, so clipped copies stay
    // aligned.  Input rows start at element zt0 - hz (smem offset 0).
    int in_bytes[NIN > 0 ? NIN : 1];
#pragma unroll
    for (int j = 0; j < NIN; ++j) {
      const int esz = P::in_esz(j), hz = TS::hz(esz);
      in_bytes[j] = (min(zt0 + TZ + hz, g.nz) - max(zt0 - hz, 0)) * esz;
    }
    int epi_bytes[NE > 0 ? NE : 1];
#pragma unroll
    for (int j = 0; j < NE; ++j) epi_bytes[j] = (min(zt0 + TZ, g.nz) - zt0) * P::epi_esz(j);
    for (int xp = xa - 1; xp <= xb; ++xp, ++gs) {
      // ring position of stage gs (incremental: no division in the loop)
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
      unsigned char* sb = stages + (size_t)st * TS::STAGE;
      const bool pv = (xp >= -g.hlo && xp < g.nx + g.hhi);
      const bool ev = pv && xp >= xa && xp < xb;
      unsigned bytes = 0;
      if (pv) {
#pragma unroll
        for (int j = 0; j < NIN; ++j)
          if (p.in_active(j))
            for (int r = 0; r < TY + 2; ++r) {
              const int yy = y0 - 1 + r;
              if (yy >= 0 && yy < g.ny) bytes += in_bytes[j];
            }
        if (ev) {
#pragma unroll
          for (int j = 0; j < NE; ++j)
            for (int r = 0; r < TY; ++r)
              if (y0 + r < g.ny) bytes += epi_bytes[j];
        }
      }
      if (lane == 0) mbar_expect_tx(&full[st], bytes);
      __syncwarp();
      if (pv) {
        for (int q = lane; q < NCOPY; q += 32) {
          if (q < NIN * (TY + 2)) {
            const int j = q / (TY + 2), r = q % (TY + 2);
            const int yy = y0 - 1 + r;
            if (!p.in_active(j) || yy < 0 || yy >= g.ny) continue;
            const int esz = P::in_esz(j), hz = TS::hz(esz);
            const int a = max(zt0 - hz, 0), b = min(zt0 + TZ + hz, g.nz);  // = in_e0 / in_bytes (j is runtime here)
            const unsigned char* base = reinterpret_cast<const unsigned char*>(p.in_ptr(j));
            const long long e0 = (long long)xp * g.plane + (long long)yy * g.nz + a;
#if GADI_SPLITCOPY
            {
              const int h = ((b - a) / 2) & ~(16 / esz - 1);
              bulk_g2s(sb + TS::off_in(j) + r * TS::rb_in(j) + (a - (zt0 - hz)) * esz, base + e0 * esz,
                       (unsigned)(h * esz), &full[st]);
              bulk_g2s(sb + TS::off_in(j) + r * TS::rb_in(j) + (a + h - (zt0 - hz)) * esz, base + (e0 + h) * esz,
                       (unsigned)((b - a - h) * esz), &full[st]);
            }
#else
            bulk_g2s(sb + TS::off_in(j) + r * TS::rb_in(j) + (a - (zt0 - hz)) * esz, base + e0 * esz,
                     (unsigned)((b - a) * esz), &full[st]);
#endif
          } else if (ev) {
            const int q2 = q - NIN * (TY + 2);
            const int j = q2 / TY, r = q2 % TY;
            const int yy = y0 + r;
            if (yy >= g.ny) continue;
            const int esz = P::epi_esz(j);
            const unsigned char* base = reinterpret_cast<const unsigned char*>(p.epi_ptr(j));
            const long long e0 = (long long)xp * g.plane + (long long)yy * g.nz + zt0;
            bulk_g2s(sb + TS::off_epi(j) + r * TS::rb_epi(j), base + e0 * esz,
                     (unsigned)((min(zt0 + TZ, g.nz) - zt0) * esz), &full[st]);
          }
        }
      }
#if GADI_L2PF > 0
      {
        const int xq = xp + GADI_L2PF;
        if (xq <= xb && xq >= -g.hlo && xq < g.nx + g.hhi) {
          const bool eq = xq >= xa && xq < xb;
          for (int q = lane; q < NCOPY; q += 32) {
            if (q < NIN * (TY + 2)) {
              const int j = q / (TY + 2), yy = y0 - 1 + q % (TY + 2);
              if (!p.in_active(j) || yy < 0 || yy >= g.ny) continue;
              const int esz = P::in_esz(j), hz = TS::hz(esz);
              const int a = max(zt0 - hz, 0), b = min(zt0 + TZ + hz, g.nz);
              const unsigned char* base = reinterpret_cast<const unsigned char*>(p.in_ptr(j));
              bulk_prefetch_l2(base + ((long long)xq * g.plane + (long long)yy * g.nz + a) * esz,
                               (unsigned)((b - a) * esz));
            } else if (eq) {
              const int q2 = q - NIN * (TY + 2);
              const int j = q2 / TY, yy = y0 + q2 % TY;
              if (yy >= g.ny) continue;
              const int esz = P::epi_esz(j);
              const unsigned char* base = reinterpret_cast<const unsigned char*>(p.epi_ptr(j));
              bulk_prefetch_l2(base + ((long long)xq * g.plane + (long long)yy * g.nz + zt0) * esz,
                               (unsigned)((min(zt0 + TZ, g.nz) - zt0) * esz));
            }
          }
        }
      }
#endif
    }
  }
}

template <class P>
__global__ void __launch_bounds__(TmaThreads<P>::NTOT, P::MINB) sweep_tma_kernel(P p) {
  using S = SweepShape<P>;
  using TS = TmaShape<P>;
  using TH = TmaThreads<P>;
  using CT = typename P::CT;
  constexpr int VZ = S::VZ, BZ = S::BZ, BY = S::BY, ZS = S::ZS, NF = S::NF;
  constexpr int TZ = S::TZ, TY = S::TY, PAD = S::PAD, ROW = S::ROW;
  constexpr int NR = P::NR, NT = P::NT, NIN = P::NIN, NE = P::NE, NST = TS::NST;
  constexpr int NCONS = TH::NCONS, NWCONS = NCONS / 32;
  static_assert(NIN <= 4 && NE <= 4, "at most four inputs of each kind");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  CT* fsm = reinterpret_cast<CT*>(smem_raw);
  unsigned char* stages = smem_raw + TS::FBYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + (size_t)NST * TS::STAGE);
  uint64_t* empty = full + NST;

  if (!p.prepare()) return;

  const SweepGeom g = p.g;
  const int tid = threadIdx.x;
  const int lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWCONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double red[NR];
#pragma unroll
  for (int s = 0; s < NR; ++s) red[s] = 0.0;

  // Wavefront schedule: every CTA sweeps its tile through all nx planes and
  // the producers may not run more than wlead planes ahead of the slowest CTA,
  // so neighbouring tiles read the same planes at the same time and their
  // halo rows / pad lines are served by L2 instead of DRAM.
  if (p.wave)
    for (int i = blockIdx.x * TH::NTOT + tid; i < g.nx; i += gridDim.x * TH::NTOT) p.wave_clear[i] = 0u;

  if (tid >= NCONS) {
    // ------------------------------------------------------------ producer
    // the whole warp issues the row copies of a stage (one row per lane),
    // lane 0 posts the byte count first
    produce_stages<P, TS>(p, g, stages, full, empty, lane);
  } else {
    // ------------------------------------------------------------ consumers
    const bool halo_warp = tid >= NT;  // 3-D only: warp NT/32 -> row y0-1, NT/32+1 -> row y0+TY
    const int hrow = halo_warp ? ((tid - NT) / 32 == 0 ? 0 : TY + 1) : 0;
    const int tz = halo_warp ? lane : tid % BZ;
    const int ty = halo_warp ? 0 : tid / BZ;
    const bool own_zl = !halo_warp && (tz == 0), own_zr = !halo_warp && (tz == BZ - 1);

    // row r (0 .. TY+1, 0 = y0-1) of stage st, pointing at core element 0
    auto in_row = [&](int st, int r) {
      SmRow R;
      const unsigned char* sb = stages + (size_t)st * TS::STAGE;
#pragma unroll
      for (int j = 0; j < 4; ++j) R.p[j] = nullptr;
#pragma unroll
      for (int j = 0; j < NIN; ++j)
        R.p[j] = sb + TS::off_in(j) + r * TS::rb_in(j) + TS::hz(P::in_esz(j)) * P::in_esz(j);
      return R;
    };
    auto epi_row = [&](int st, int r) {
      SmRow R;
      const unsigned char* sb = stages + (size_t)st * TS::STAGE;
#pragma unroll
      for (int j = 0; j < 4; ++j) R.p[j] = nullptr;
#pragma unroll
      for (int j = 0; j < NE; ++j) R.p[j] = sb + TS::off_epi(j) + r * TS::rb_epi(j);
      return R;
    };
    // nz % VZ == 0 on this path: a lane's vector is entirely valid or not
    auto fields_core = [&](int st, int r, int nv, CT (&f)[NF][VZ]) {
      if (nv == VZ) {
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
    auto store_row = [&](CT* buf, int rr, const CT (&fc)[NF][VZ]) {
#pragma unroll
      for (int q = 0; q < NF; ++q) {
        CT* row = buf + ((size_t)q * (TY + 2) + rr) * ROW + PAD + tz * VZ;
#pragma unroll
        for (int k = 0; k < VZ; ++k) row[k] = fc[q][k];
      }
    };
    // z-halo scalars of this thread's row (edge lanes only)
    auto store_zhalo = [&](CT* buf, int st, bool ok, int zt0) {
      const SmRow R = in_row(st, ty + 1);
#pragma unroll
      for (int j = 0; j < ZS; ++j) {
        const int zl = zt0 - ZS + j, zr = zt0 + TZ + j;
        CT tl[NF], tr[NF];
        if (own_zl && ok && zl >= 0) {
          typename P::RawS a;
          p.load_raw_s_sm(a, R, -ZS + j);
          p.field_s(a, tl);
        } else {
#pragma unroll
          for (int q = 0; q < NF; ++q) tl[q] = CT(0);
        }
        if (own_zr && ok && zr < g.nz) {
          typename P::RawS a;
          p.load_raw_s_sm(a, R, TZ + j);
          p.field_s(a, tr);
        } else {
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
    };
    auto release = [&](int s) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s % NST]);
    };
    auto wait_full = [&](int s) { mbar_wait(&full[s % NST], (unsigned)((s / NST) & 1)); };

    if constexpr (TH::NH == 0) {
      // 2-D: the y-halo rows of the f-plane buffers stay zero
      for (int i = tid; i < 2 * NF * 2 * ROW; i += NCONS) {
        const int buf = i / (NF * 2 * ROW), rem = i % (NF * 2 * ROW);
        const int q = rem / (2 * ROW), rr = (rem / ROW) % 2 == 0 ? 0 : TY + 1, c = rem % ROW;
        fsm[(size_t)buf * S::PLANE + ((size_t)q * (TY + 2) + rr) * ROW + c] = CT(0);
      }
    }
    SegIter it(g, gridDim.x, blockIdx.x);
    int tile, xa, xb;
    int gs = 0;  // stage sequence number of plane xa-1 of the current segment
    while (it.next(tile, xa, xb)) {
      const int zt0 = (tile % g.nzt) * TZ, y0 = (tile / g.nzt) * TY;
      const int zb = zt0 + tz * VZ;
      const int y = halo_warp ? (hrow == 0 ? y0 - 1 : y0 + TY) : y0 + ty;
      const bool yok = y >= 0 && y < g.ny;
      const int nvz = yok ? max(0, min(VZ, g.nz - zb)) : 0;
      const long long rowbase = (long long)y * g.nz + zb;

      if (halo_warp) {
        // plane xa-1 is never read by the halo warps: hand its stage back at
        // once (after it filled, so the arrival counts for this use), else a
        // segment longer than the ring would starve the producer
        wait_full(gs);
        release(gs);
        // halo rows of planes xa .. xb into the f-plane buffers
        for (int x = xa; x <= xb; ++x) {
          const int s = gs + (x - xa + 1);
          wait_full(s);
          CT fh[NF][VZ];
          const bool pv = x < g.nx + g.hhi;
          fields_core((int)(s % NST), hrow, pv ? nvz : 0, fh);
          store_row(fsm + (size_t)((x - xa) & 1) * S::PLANE, hrow, fh);
          if (x > xa) release(s - 1);
          consumer_sync(NCONS);
        }
        release(gs + (xb - xa + 1));
        gs += xb - xa + 2;
        continue;
      }

      CT fprev[NF][VZ], fcur[NF][VZ], fnext[NF][VZ];
      {
        wait_full(gs);
        fields_core((int)(gs % NST), ty + 1, (xa - 1 >= -g.hlo) ? nvz : 0, fprev);
        wait_full(gs + 1);
        fields_core((int)((gs + 1) % NST), ty + 1, nvz, fcur);
        store_row(fsm, ty + 1, fcur);
        if (own_zl || own_zr) store_zhalo(fsm, (int)((gs + 1) % NST), yok, zt0);
      }
      consumer_sync(NCONS);
      release(gs);

      long long gidx = (long long)xa * g.plane + rowbase;
      for (int x = xa; x < xb; ++x, gidx += g.plane) {
        const int s = gs + (x - xa + 1);  // stage of plane x
        CT* bcur = fsm + (size_t)((x - xa) & 1) * S::PLANE;
        CT* bnxt = fsm + (size_t)(((x - xa) + 1) & 1) * S::PLANE;
        // 1. plane x+1 -> fnext + f-plane buffer (halo warps add the y-halo rows)
        wait_full(s + 1);
        const bool pv1 = x + 1 < g.nx + g.hhi;
        fields_core((int)((s + 1) % NST), ty + 1, pv1 ? nvz : 0, fnext);
        store_row(bnxt, ty + 1, fnext);
        if (own_zl || own_zr) store_zhalo(bnxt, (int)((s + 1) % NST), pv1 && yok, zt0);
        // 2. stencil(s) and epilogue of plane x
        typename P::Epi E;
        p.load_epi_sm(E, epi_row((int)(s % NST), ty), tz * VZ);
        if constexpr (HasEpiV<P>::value) {
          if (nvz == VZ) p.load_epi_v(E, gidx, VZ);
        }
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
          CT ym[VZ], yp[VZ];
#pragma unroll
          for (int k = 0; k < VZ; ++k) {
            ym[k] = rowm[k];
            yp[k] = rowp[k];
          }
          if constexpr (HasStencilVec<P>::value) {
            p.stencil_vec(q, fprev[q], ym, fcur[q], left, right, yp, fnext[q], st[q]);
          } else {
#pragma unroll
            for (int k = 0; k < VZ; ++k) {
              const CT zm = (k >= ZS) ? fcur[q][k - ZS] : left[k];
              const CT zp = (k + ZS < VZ) ? fcur[q][k + ZS] : right[k + ZS - VZ];
              const Nb<CT> nb{fprev[q][k], ym[k], zm, fcur[q][k], zp, yp[k], fnext[q][k]};
              st[q][k] = p.stencil(q, k, nb, fcur, E);
            }
          }
        }
        if (nvz == VZ) p.epilogue(gidx, VZ, fcur, st, E, red);
#pragma unroll
        for (int q = 0; q < NF; ++q)
#pragma unroll
          for (int k = 0; k < VZ; ++k) {
            fprev[q][k] = fcur[q][k];
            fcur[q][k] = fnext[q][k];
          }
        consumer_sync(NCONS);
        release(s);
        if (p.wave && tid == 0) {
          __threadfence();
          atomicAdd(p.wave + x, 1u);
        }
      }
      release(gs + (xb - xa + 1));  // plane xb
      gs += xb - xa + 2;
    }
  }

  if constexpr (P::HAS_RED) {
    double tot[NR];
    int ops[NR];
#pragma unroll
    for (int s = 0; s < NR; ++s) ops[s] = P::op(s);
    if (grid_finish<NR, TH::NTOT>(red, ops, p.partials, g.pstride, p.ticket, tot)) {
      if (threadIdx.x == 0) finish_pass(p, tot);
    }
  }
}

}  // namespace gadi
