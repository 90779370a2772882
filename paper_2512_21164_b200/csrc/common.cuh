// Device-side building blocks shared by every GADI kernel: storage <-> compute
// conversions with the reference's rounding contract (RNE, no FTZ, overflow to
// +-inf; gadimp/precision.py:136-165), vectorised 16-byte loads/stores,
// ordered (non-contracted) multiply-add, and the deterministic
// "last block finishes the reduction" pattern used to keep every inner-solver
// scalar (alpha, beta, convergence flags) on the device.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <type_traits>

namespace gadi {

typedef __nv_bfloat16 bf16;
typedef __half fp16;

// ---------------------------------------------------------------- conversions
template <class CT> __device__ __forceinline__ CT cvt_in(bf16 v) { return (CT)__bfloat162float(v); }
template <class CT> __device__ __forceinline__ CT cvt_in(fp16 v) { return (CT)__half2float(v); }
template <class CT> __device__ __forceinline__ CT cvt_in(float v) { return (CT)v; }
template <class CT> __device__ __forceinline__ CT cvt_in(double v) { return (CT)v; }

// Round a compute-type value onto the storage grid (RNE).  An fp64 value goes
// to bf16 through fp32 exactly as the reference does (precision.py:113-125):
// for an arbitrary fp64 value (e.g. 2^-e r, or a quotient) the two-step
// rounding can differ from a direct cvt.rn.bf16.f64 at bf16 midpoints.
template <class ST> struct Store;
template <> struct Store<bf16> {
  static __device__ __forceinline__ bf16 from(float v) { return __float2bfloat16_rn(v); }
  static __device__ __forceinline__ bf16 from(double v) { return __float2bfloat16_rn(__double2float_rn(v)); }
};
template <> struct Store<fp16> {
  static __device__ __forceinline__ fp16 from(float v) { return __float2half_rn(v); }
  static __device__ __forceinline__ fp16 from(double v) { return __double2half(v); }
};
template <> struct Store<float> {
  static __device__ __forceinline__ float from(float v) { return v; }
  static __device__ __forceinline__ float from(double v) { return __double2float_rn(v); }
};
template <> struct Store<double> {
  static __device__ __forceinline__ double from(float v) { return (double)v; }
  static __device__ __forceinline__ double from(double v) { return v; }
};

template <class ST, class CT>
__device__ __forceinline__ CT round_to(CT v) { return cvt_in<CT>(Store<ST>::from(v)); }

// ------------------------------------------------------------ ordered madd
// ORD=true: product and sum each rounded separately (no FMA contraction);
// this is the reference's scipy/emulated order (gadimp/sparsemat.py:193-198).
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }

template <bool ORD, class CT>
__device__ __forceinline__ CT madd(CT c, CT v, CT acc) {
  if (ORD) return add_rn(acc, mul_rn(c, v));
  return fma_rn(c, v, acc);
}

// ------------------------------------------------------------ packed fp32x2
// Blackwell executes fp32 add/mul/fma on register pairs (SASS FFMA2/FADD2/
// FMUL2): half the instruction count of the scalar forms for the
// storage-model arithmetic.  Pairs are (element 2j, element 2j+1).
__device__ __forceinline__ unsigned long long f2u(float2 a) {
  unsigned long long u;
  asm("mov.b64 %0, {%1, %2};" : "=l"(u) : "f"(a.x), "f"(a.y));
  return u;
}
__device__ __forceinline__ float2 u2f(unsigned long long u) {
  float2 a;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(u));
  return a;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(r);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}
__device__ __forceinline__ float2 bcast2(float a) { return make_float2(a, a); }

// bf16x2 word -> two floats with one integer op each (bf16 is the top half
// of an fp32 pattern): lo = w << 16, hi = w & 0xffff0000.
__device__ __forceinline__ float bf_lo(unsigned w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(unsigned w) { return __uint_as_float(w & 0xffff0000u); }

// RNE-round a pair of floats onto the storage grid (packed conversion for
// bf16/fp16: one F2FP per pair) and return the rounded values as floats.
template <class ST>
__device__ __forceinline__ float2 round2(float2 v) {
  if constexpr (std::is_same<ST, bf16>::value) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(v.x, v.y);
    const unsigned w = *reinterpret_cast<const unsigned*>(&h);
    return make_float2(bf_lo(w), bf_hi(w));
  } else if constexpr (std::is_same<ST, fp16>::value) {
    const __half2 h = __floats2half2_rn(v.x, v.y);
    return __half22float2(h);
  } else {
    return v;
  }
}

// ------------------------------------------------------------ vector memory
// Load VZ consecutive elements (element index idx, VZ-aligned when VEC) and
// convert to the compute type. Read-only arrays go through the non-coherent
// path; arrays that the same kernel also writes must use NC=false.
template <class T, int VZ, bool NC, class CT>
__device__ __forceinline__ void load_vec(const T* __restrict__ p, long long idx, CT (&out)[VZ]) {
  constexpr int BYTES = VZ * (int)sizeof(T);
  const T* q = p + idx;
  if constexpr (std::is_same<T, bf16>::value && std::is_same<CT, float>::value && BYTES % 16 == 0) {
#pragma unroll
    for (int c = 0; c < BYTES / 16; ++c) {
      const uint4 u = NC ? __ldg(reinterpret_cast<const uint4*>(q) + c) : __ldcg(reinterpret_cast<const uint4*>(q) + c);
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
      uint4 u = NC ? __ldg(reinterpret_cast<const uint4*>(q) + c)
                   : __ldcg(reinterpret_cast<const uint4*>(q) + c);
      const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
      for (int j = 0; j < PER; ++j) out[c * PER + j] = cvt_in<CT>(e[j]);
    }
  } else if constexpr (BYTES == 8) {
    uint2 u = NC ? __ldg(reinterpret_cast<const uint2*>(q)) : __ldcg(reinterpret_cast<const uint2*>(q));
    const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int j = 0; j < VZ; ++j) out[j] = cvt_in<CT>(e[j]);
  } else if constexpr (BYTES == 4) {
    unsigned int u = NC ? __ldg(reinterpret_cast<const unsigned int*>(q))
                        : __ldcg(reinterpret_cast<const unsigned int*>(q));
    const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int j = 0; j < VZ; ++j) out[j] = cvt_in<CT>(e[j]);
  } else {
#pragma unroll
    for (int j = 0; j < VZ; ++j) out[j] = cvt_in<CT>(q[j]);
  }
}

// Masked scalar variant: element j is loaded when j < nvalid, else zero.
template <class T, int VZ, class CT>
__device__ __forceinline__ void load_vec_masked(const T* __restrict__ p, long long idx, int nvalid,
                                                CT (&out)[VZ]) {
#pragma unroll
  for (int j = 0; j < VZ; ++j) out[j] = (j < nvalid) ? cvt_in<CT>(p[idx + j]) : CT(0);
}

// `vec` is uniform over the grid (nz % VZ == 0 and 16-byte aligned bases).
template <class T, int VZ, bool NC, class CT>
__device__ __forceinline__ void load_any(const T* __restrict__ p, long long idx, int nvalid, CT (&out)[VZ],
                                         bool vec) {
  if (vec && nvalid >= VZ) {
    load_vec<T, VZ, NC>(p, idx, out);
  } else {
    load_vec_masked<T, VZ>(p, idx, nvalid, out);
  }
}

// Store VZ compute-type values rounded onto the storage grid of T.
template <class T, int VZ, class CT>
__device__ __forceinline__ void store_any(T* __restrict__ p, long long idx, int nvalid, const CT (&v)[VZ],
                                          bool vec) {
  constexpr int BYTES = VZ * (int)sizeof(T);
  T tmp[VZ];
  if constexpr (std::is_same<CT, float>::value && std::is_same<T, bf16>::value && VZ % 2 == 0) {
#pragma unroll
    for (int j = 0; j < VZ; j += 2)
      *reinterpret_cast<__nv_bfloat162*>(&tmp[j]) = __floats2bfloat162_rn(v[j], v[j + 1]);
  } else if constexpr (std::is_same<CT, float>::value && std::is_same<T, fp16>::value && VZ % 2 == 0) {
#pragma unroll
    for (int j = 0; j < VZ; j += 2) *reinterpret_cast<__half2*>(&tmp[j]) = __floats2half2_rn(v[j], v[j + 1]);
  } else {
#pragma unroll
    for (int j = 0; j < VZ; ++j) tmp[j] = Store<T>::from(v[j]);
  }
  if (vec && nvalid >= VZ) {
    if constexpr (BYTES % 16 == 0) {
#pragma unroll
      for (int c = 0; c < BYTES / 16; ++c)
        reinterpret_cast<uint4*>(p + idx)[c] = reinterpret_cast<const uint4*>(tmp)[c];
    } else if constexpr (BYTES == 8) {
      *reinterpret_cast<uint2*>(p + idx) = *reinterpret_cast<const uint2*>(tmp);
    } else if constexpr (BYTES == 4) {
      *reinterpret_cast<unsigned int*>(p + idx) = *reinterpret_cast<const unsigned int*>(tmp);
    } else {
#pragma unroll
      for (int j = 0; j < VZ; ++j) p[idx + j] = tmp[j];
    }
  } else {
#pragma unroll
    for (int j = 0; j < VZ; ++j)
      if (j < nvalid) p[idx + j] = tmp[j];
  }
}

// GADI_EXACT_PACK = 1 packs already-rounded bf16 values with PRMT instead of
// F2FP: measured neutral to slightly worse (HcgB 257 -> 261 us,
// profiles/ab_pack_zpad_r2.jsonl) -- off
#ifndef GADI_EXACT_PACK
#define GADI_EXACT_PACK 0
#endif
// Store VZ compute-type values that are already exact values of T (rounded
// earlier in the pass): for bf16 the pair is packed by a byte permute of the
// fp32 patterns' top halves (one PRMT on the integer pipe) instead of a
// rounding conversion (F2FP); identical bits.  Other types as store_any.
template <class T, int VZ, class CT>
__device__ __forceinline__ void store_exact(T* __restrict__ p, long long idx, int nvalid, const CT (&v)[VZ], bool vec) {
  if constexpr (GADI_EXACT_PACK && std::is_same<CT, float>::value && std::is_same<T, bf16>::value && VZ % 2 == 0) {
    constexpr int BYTES = VZ * 2;
    if (vec && nvalid >= VZ && BYTES % 16 == 0) {
      unsigned w[VZ / 2];
#pragma unroll
      for (int j = 0; j < VZ; j += 2) {
        unsigned d;
        asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(d) : "r"(__float_as_uint(v[j])), "r"(__float_as_uint(v[j + 1])));
        w[j / 2] = d;
      }
#pragma unroll
      for (int c = 0; c < BYTES / 16; ++c)
        reinterpret_cast<uint4*>(p + idx)[c] = make_uint4(w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
      return;
    }
  }
  store_any<T, VZ>(p, idx, nvalid, v, vec);
}

// ------------------------------------------------------------ reductions
enum RedOp { RED_SUM = 0, RED_MAX = 1 };

// MAX propagates NaN like numpy's np.max (gadimp/gadi.py:151).
__device__ __forceinline__ double red_combine(int op, double a, double b) {
  if (op == RED_MAX) return (a > b || a != a) ? a : b;
  return a + b;
}

// Deterministic block reduction of NR doubles (fixed xor-shuffle tree, then
// warp partials summed in warp order by warp 0). Result valid in thread 0.
template <int NR, int NT>
__device__ __forceinline__ void block_reduce(double (&v)[NR], const int (&ops)[NR]) {
  constexpr int NW = NT / 32;
  __shared__ double sred[NR][NW];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int s = 0; s < NR; ++s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[s] = red_combine(ops[s], v[s], __shfl_xor_sync(0xffffffffu, v[s], o));
  }
  __syncthreads();  // sred may be reused by a previous call
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < NR; ++s) sred[s][w] = v[s];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NR; ++s) {
      double a = sred[s][0];
      for (int i = 1; i < NW; ++i) a = red_combine(ops[s], a, sred[s][i]);
      v[s] = a;
    }
  }
}

// Cross-block finish: every block deposits its partials, the last block to
// arrive (ticket) reduces them in block order and returns true in all of its
// threads with the totals in thread 0's `tot`. The ticket is reset for the
// next launch. Deterministic for a fixed grid.
template <int NR, int NT>
__device__ __forceinline__ bool grid_finish(double (&v)[NR], const int (&ops)[NR], double* __restrict__ partials,
                                            int pstride, unsigned int* ticket, double (&tot)[NR]) {
  __shared__ bool am_last;
  block_reduce<NR, NT>(v, ops);
  const int nb = gridDim.x;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NR; ++s) partials[(size_t)s * pstride + blockIdx.x] = v[s];
    __threadfence();
    unsigned int t = atomicAdd(ticket, 1u);
    am_last = (t == (unsigned)(nb - 1));
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  double acc[NR];
#pragma unroll
  for (int s = 0; s < NR; ++s) acc[s] = 0.0;
  bool any[NR];
#pragma unroll
  for (int s = 0; s < NR; ++s) any[s] = false;
  for (int i = threadIdx.x; i < nb; i += NT) {
#pragma unroll
    for (int s = 0; s < NR; ++s) {
      double x = __ldcg(partials + (size_t)s * pstride + i);
      acc[s] = any[s] ? red_combine(ops[s], acc[s], x) : x;
      any[s] = true;
    }
  }
  block_reduce<NR, NT>(acc, ops);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < NR; ++s) tot[s] = acc[s];
    *ticket = 0u;
  }
  return true;
}

}  // namespace gadi
