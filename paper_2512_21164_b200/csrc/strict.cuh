// Reference rounding inside the fused passes (gadi_solve(..., rounding=
// "reference")): the reference's round-after-every-operation emulation
// (gadimp/precision.py:176-220, sparsemat.py:178-199, inner.py:39-143)
// restated in the same streaming kernels as the storage model, at the same
// HBM traffic.
//
//  * SpMV: y_i = fl(...fl(fl(a_i,c0 x_c0) + fl(a_i,c1 x_c1)) ...), ascending
//    column order (lo_x, lo_y, lo_z, d, up_z, up_y, up_x), every product and
//    partial sum rounded to u_s.  bf16 / fp16 run as packed bf16x2 / f16x2
//    multiplies and adds (SASS HFMA2.BF16_V2 with a -0 addend, HADD2): each is
//    the exact result rounded once to u_s (RN, subnormals kept), which is the
//    reference's fp64-op-then-quantize (double rounding through fp32 is
//    innocuous at 8 / 11 significand bits).  fp32: mul.rn / add.rn.
//  * axpy: x <- fl(x + fl(alpha p)) (inner.py:74-75, 85, 127-128, 139).
//  * fl_dot(x, y, dfmt) (precision.py:189-220): products rounded to dfmt,
//    summed by the reference's pairwise tree (fl_sum), dfmt = u_s, or fp32
//    when strict_model = False and u_s is below fp32 (inner.py:39-44).  The
//    tree is split at aligned power-of-two blocks: a lane sums its own
//    VZ-element vector, a warp butterfly (xor 1, 2, ...) combines the lanes
//    of one aligned block of G elements, and the kernel writes one leaf per
//    block; tree_finish_kernel then sums the n/G leaves with the same tree
//    and runs the pass's scalar recurrence.  Zero padding of the last block
//    equals fl_sum's carried odd element (fl(a + 0) = a).
//  * alpha, beta = fl_op("div", ...) rounded to u_s (inner.py:73, 84, 126, 138).
#pragma once
#include "sweep.cuh"

namespace gadi {

// fl_dot accumulation format (the reference's `dfmt`)
enum DotKind { DK_F32 = 0, DK_BF16 = 1, DK_F16 = 2 };

__device__ __forceinline__ float dround(float v, int dk) {
  if (dk == DK_BF16) return __bfloat162float(__float2bfloat16_rn(v));
  if (dk == DK_F16) return __half2float(__float2half_rn(v));
  return v;
}
__device__ __forceinline__ float dadd(float a, float b, int dk) { return dround(__fadd_rn(a, b), dk); }

// pairwise tree of one lane's VZ values (an aligned block of the fl_sum tree)
template <int VZ>
__device__ __forceinline__ float vtree(float (&v)[VZ], int dk) {
#pragma unroll
  for (int w = 1; w < VZ; w *= 2)
#pragma unroll
    for (int k = 0; k + w < VZ; k += 2 * w) v[k] = dadd(v[k], v[k + w], dk);
  return v[0];
}

template <int V> struct Log2 { static constexpr int value = 1 + Log2<V / 2>::value; };
template <> struct Log2<1> { static constexpr int value = 0; };

// Scalars of the reference rounding: fl_op("div", a, b, u_s)
__device__ __forceinline__ double sround(double v, int us) {
  switch (us) {
    case 1: return (double)__bfloat162float(__float2bfloat16_rn(__double2float_rn(v)));  // precision.py:113-125
    case 2: return (double)__half2float(__double2half(v));
    case 3: return (double)__double2float_rn(v);
    default: return v;
  }
}
template <class ST> struct RndCode { static constexpr int value = 0; };
template <> struct RndCode<bf16> { static constexpr int value = 1; };
template <> struct RndCode<fp16> { static constexpr int value = 2; };
template <> struct RndCode<float> { static constexpr int value = 3; };

// ------------------------------------------------------------ packed u_s words
__device__ __forceinline__ unsigned bmul2(unsigned a, unsigned b) {
  unsigned d;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ unsigned badd2(unsigned a, unsigned b) {
  unsigned d;
  asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ unsigned hmul2(unsigned a, unsigned b) {
  unsigned d;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ unsigned hadd2(unsigned a, unsigned b) {
  unsigned d;
  asm("add.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// Two floats that are exact u_s values <-> one packed word (element k low).
template <class ST> struct Pk;
template <> struct Pk<bf16> {
  static __device__ __forceinline__ unsigned pack(float a, float b) {
    unsigned d;  // the top halves of two fp32 patterns (exact: a, b are bf16 values)
    asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(d) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)));
    return d;
  }
  static __device__ __forceinline__ void unpack(unsigned w, float& a, float& b) {
    a = bf_lo(w);
    b = bf_hi(w);
  }
  static __device__ __forceinline__ unsigned mul(unsigned a, unsigned b) { return bmul2(a, b); }
  static __device__ __forceinline__ unsigned add(unsigned a, unsigned b) { return badd2(a, b); }
};
template <> struct Pk<fp16> {
  static __device__ __forceinline__ unsigned pack(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);  // exact: a, b are fp16 values
    return *reinterpret_cast<const unsigned*>(&h);
  }
  static __device__ __forceinline__ void unpack(unsigned w, float& a, float& b) {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w));
    a = f.x;
    b = f.y;
  }
  static __device__ __forceinline__ unsigned mul(unsigned a, unsigned b) { return hmul2(a, b); }
  static __device__ __forceinline__ unsigned add(unsigned a, unsigned b) { return hadd2(a, b); }
};

// ------------------------------------------------------------ SpMV, axpy
// One lane's vector of the reference-rounded stencil (see top).  ST is the
// storage type; CT = float for bf16 / fp16 / fp32, double for fp64 (the
// ordered scipy form, apply_stencil<true>).
template <class ST, bool HASY, int VZ, int ZS, class CT>
__device__ __forceinline__ void stencil_vec_ref(const CoefT<CT>& c, const CT (&xm)[VZ], const CT (&ym)[VZ],
                                                const CT (&ce)[VZ], const CT (&lf)[ZS], const CT (&rt)[ZS],
                                                const CT (&yp)[VZ], const CT (&xp)[VZ], CT (&out)[VZ]) {
  CT zm[VZ], zp[VZ];
#pragma unroll
  for (int k = 0; k < VZ; ++k) {
    zm[k] = (k >= ZS) ? ce[k - ZS] : lf[k];
    zp[k] = (k + ZS < VZ) ? ce[k + ZS] : rt[k + ZS - VZ];
  }
  if constexpr (std::is_same<ST, bf16>::value || std::is_same<ST, fp16>::value) {
    static_assert(VZ % 2 == 0, "packed pairs");
    using K = Pk<ST>;
    const unsigned cx0 = K::pack(c.lo[0], c.lo[0]), cy0 = K::pack(c.lo[1], c.lo[1]);
    const unsigned cz0 = K::pack(c.lo[2], c.lo[2]), cd = K::pack(c.d, c.d);
    const unsigned cz1 = K::pack(c.up[2], c.up[2]), cy1 = K::pack(c.up[1], c.up[1]);
    const unsigned cx1 = K::pack(c.up[0], c.up[0]);
#pragma unroll
    for (int k = 0; k < VZ; k += 2) {
      unsigned a = K::mul(cx0, K::pack(xm[k], xm[k + 1]));
      if constexpr (HASY) a = K::add(a, K::mul(cy0, K::pack(ym[k], ym[k + 1])));
      a = K::add(a, K::mul(cz0, K::pack(zm[k], zm[k + 1])));
      a = K::add(a, K::mul(cd, K::pack(ce[k], ce[k + 1])));
      a = K::add(a, K::mul(cz1, K::pack(zp[k], zp[k + 1])));
      if constexpr (HASY) a = K::add(a, K::mul(cy1, K::pack(yp[k], yp[k + 1])));
      a = K::add(a, K::mul(cx1, K::pack(xp[k], xp[k + 1])));
      K::unpack(a, out[k], out[k + 1]);
    }
  } else if constexpr (std::is_same<ST, float>::value) {
#pragma unroll
    for (int k = 0; k < VZ; ++k) {
      float a = __fmul_rn(c.lo[0], xm[k]);
      if constexpr (HASY) a = __fadd_rn(a, __fmul_rn(c.lo[1], ym[k]));
      a = __fadd_rn(a, __fmul_rn(c.lo[2], zm[k]));
      a = __fadd_rn(a, __fmul_rn(c.d, ce[k]));
      a = __fadd_rn(a, __fmul_rn(c.up[2], zp[k]));
      if constexpr (HASY) a = __fadd_rn(a, __fmul_rn(c.up[1], yp[k]));
      out[k] = __fadd_rn(a, __fmul_rn(c.up[0], xp[k]));
    }
  } else {
#pragma unroll
    for (int k = 0; k < VZ; ++k) out[k] = apply_stencil<true>(c, CT(0), xm[k], ym[k], zm[k], ce[k], zp[k], yp[k], xp[k]);
  }
}

// scalar form (register-path / f-plane consumers): same operations per element
template <class ST, class CT>
__device__ __forceinline__ CT stencil_ref1(const CoefT<CT>& c, const Nb<CT>& n) {
  if constexpr (std::is_same<ST, double>::value) {
    return apply_stencil<true>(c, CT(0), n);
  } else {
    auto m = [](CT a, CT b) { return round_to<ST>(mul_rn(a, b)); };
    auto s = [](CT a, CT b) { return round_to<ST>(add_rn(a, b)); };
    CT a = m(c.lo[0], n.xm);
    a = s(a, m(c.lo[1], n.ym));
    a = s(a, m(c.lo[2], n.zm));
    a = s(a, m(c.d, n.ce));
    a = s(a, m(c.up[2], n.zp));
    a = s(a, m(c.up[1], n.yp));
    return s(a, m(c.up[0], n.xp));
  }
}

// y = fl(c + fl(s a)) on a whole vector
template <class ST, int VZ, class CT>
__device__ __forceinline__ void axpy_ref(CT s, const CT (&a)[VZ], const CT (&c)[VZ], CT (&y)[VZ]) {
  if constexpr (std::is_same<ST, bf16>::value || std::is_same<ST, fp16>::value) {
    using K = Pk<ST>;
    const unsigned s2 = K::pack(s, s);
#pragma unroll
    for (int k = 0; k < VZ; k += 2) {
      const unsigned w = K::add(K::pack(c[k], c[k + 1]), K::mul(s2, K::pack(a[k], a[k + 1])));
      K::unpack(w, y[k], y[k + 1]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < VZ; ++k) y[k] = add_rn(c[k], mul_rn(s, a[k]));
  }
}
template <class ST, class CT>
__device__ __forceinline__ CT axpy_ref1(CT s, CT a, CT c) {
  return round_to<ST>(add_rn(c, round_to<ST>(mul_rn(s, a))));
}

// ------------------------------------------------------------ fl_dot leaves
// Leaf output of a reference-rounding dot in a pass (fields of PassBase /
// PwBase): tree == nullptr in the storage model.
//
// Complex (crd) vectors are interleaved (re, im) on the device but the
// reference's vector is the block [re(0..m); im(0..m)] (problems.py:116), and
// fl_sum's tree runs over that block order.  A lane's VZ-vector then holds
// VZ/2 consecutive real parts and the matching imaginary parts: each half is
// an aligned block of its own half of the tree, so the lane (and the warp
// butterfly) keeps two partial sums -- packed as the two 32-bit halves of the
// pass's fp64 reduction slot -- and writes two leaves, one in each half of the
// leaf array.  One leaf per element: the element's block-layout position.
struct TreeOut {
  float* tree;    // leaves
  int tlog;       // log2(device elements per leaf block); -1: one leaf per element
  int dk;         // DotKind
  double* aux;    // the pass's other (fp64) totals, handed to the finisher
  long long cm;   // complex points m (interleaved crd vectors), 0 for real vectors
};

__device__ __forceinline__ double pack2f(float re, float im) {
  return __hiloint2double(__float_as_int(im), __float_as_int(re));
}
__device__ __forceinline__ float2 unpack2f(double v) {
  return make_float2(__int_as_float(__double2loint(v)), __int_as_float(__double2hiint(v)));
}

// Products of one lane's vector rounded to dfmt; either written as leaves
// (tlog < 0) or summed into the lane's aligned block(s) and returned (real:
// the sum; complex: the packed (re, im) sums).  CX: 0 real, 1 complex,
// 2 decided at run time by t.cm.
template <int VZ, int CX = 0>
__device__ __forceinline__ double dot_leaf(const TreeOut& t, long long i, int nv, const float (&a)[VZ],
                                           const float (&b)[VZ]) {
  float pr[VZ];
#pragma unroll
  for (int k = 0; k < VZ; ++k) pr[k] = (k < nv) ? dround(__fmul_rn(a[k], b[k]), t.dk) : 0.f;
  const bool cplx = CX == 1 || (CX == 2 && t.cm > 0);
  if (t.tlog < 0) {
#pragma unroll
    for (int k = 0; k < VZ; ++k)
      if (k < nv) {
        const long long j = i + k;
        t.tree[cplx ? ((j & 1) ? t.cm : 0) + (j >> 1) : j] = pr[k];
      }
    return 0.0;
  }
  if constexpr (CX != 0 && VZ >= 2) {
    if (cplx) {
      float re[VZ / 2], im[VZ / 2];
#pragma unroll
      for (int k = 0; k < VZ / 2; ++k) {
        re[k] = pr[2 * k];
        im[k] = pr[2 * k + 1];
      }
      return pack2f(vtree<VZ / 2>(re, t.dk), vtree<VZ / 2>(im, t.dk));
    }
  }
  return (double)vtree<VZ>(pr, t.dk);
}

// Warp step: combine the lanes of each aligned G-block (G = 2^tlog >= VZ)
// and write its leaf (two leaves for complex vectors).  Called by all 32
// lanes with t.tlog >= 0; `own` lanes hold valid data.
template <int VZ, int CX = 0>
__device__ __forceinline__ void tree_emit(const TreeOut& t, long long i, bool own, int lane, double v) {
  const int lv = t.tlog - Log2<VZ>::value;
  const bool cplx = CX == 1 || (CX == 2 && t.cm > 0);
  if (CX != 0 && cplx) {
    float2 s = unpack2f(v);
    for (int l = 0; l < lv; ++l) {
      s.x = dadd(s.x, __shfl_xor_sync(0xffffffffu, s.x, 1 << l), t.dk);
      s.y = dadd(s.y, __shfl_xor_sync(0xffffffffu, s.y, 1 << l), t.dk);
    }
    if (own && (lane & ((1 << lv) - 1)) == 0) {
      const long long leaf = (i >> 1) >> (t.tlog - 1);
      t.tree[leaf] = s.x;
      t.tree[(t.cm >> (t.tlog - 1)) + leaf] = s.y;
    }
    return;
  }
  float s = (float)v;
  for (int l = 0; l < lv; ++l) s = dadd(s, __shfl_xor_sync(0xffffffffu, s, 1 << l), t.dk);
  if (own && (lane & ((1 << lv) - 1)) == 0) t.tree[i >> t.tlog] = s;
}

// ------------------------------------------------------------ finisher
constexpr int TF_NT = 256, TF_PER = 16, TF_BLK = TF_NT * TF_PER;

// fl_sum tree of the aligned block src[0 .. TF_BLK) (zeros past cnt); the
// result is valid in thread 0.
__device__ __forceinline__ float block_tree(const float* __restrict__ src, long long cnt, int dk) {
  __shared__ float sw[TF_NT / 32];
  float v[TF_PER];
  const long long o = (long long)threadIdx.x * TF_PER;
  if (o + TF_PER <= cnt) {
#pragma unroll
    for (int k = 0; k < TF_PER; k += 4) {
      const float4 q = __ldcg(reinterpret_cast<const float4*>(src + o + k));
      v[k] = q.x;
      v[k + 1] = q.y;
      v[k + 2] = q.z;
      v[k + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < TF_PER; ++k) v[k] = (o + k < cnt) ? __ldcg(src + o + k) : 0.f;
  }
  float s = vtree<TF_PER>(v, dk);
#pragma unroll
  for (int l = 1; l < 32; l <<= 1) s = dadd(s, __shfl_xor_sync(0xffffffffu, s, l), dk);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float w[TF_NT / 32];
#pragma unroll
    for (int k = 0; k < TF_NT / 32; ++k) w[k] = sw[k];
    s = vtree<TF_NT / 32>(w, dk);
  }
  return s;
}

// Sum the m leaves (block b of TF_BLK leaves per CTA, then the last CTA sums
// the per-block values, in further rounds of TF_BLK while more than one
// remains) and run the pass's recurrence with the tree total in slot P::TS.
// lvl holds >= 2 * ceil(m / TF_BLK) + 2 floats.
// Slab decomposition (slot >= 0): the leaves are this rank's aligned subtree
// of the global tree; the total goes into this rank's gather row (slot
// `slot`; slot P::TS also carries the pass's fp64 totals) and
// tree_combine_kernel finishes the tree across ranks.
template <class P>
__global__ void __launch_bounds__(TF_NT) tree_finish_kernel(P p, const float* __restrict__ leaves, long long m,
                                                            float* __restrict__ lvl, unsigned int* __restrict__ ticket,
                                                            int slot) {
  __shared__ bool last;
  if (!p.prepare()) return;
  const TreeOut& t = p.tout;
  const long long base = (long long)blockIdx.x * TF_BLK;
  const float v = block_tree(leaves + base, m - base, t.dk);
  if (threadIdx.x == 0) {
    lvl[blockIdx.x] = v;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  float* src = lvl;
  long long cnt = gridDim.x;
  float* dst = lvl + ((cnt + 3) & ~3LL);  // 16-byte aligned for block_tree's vector loads
  while (cnt > 1) {
    const long long nblk = (cnt + TF_BLK - 1) / TF_BLK;
    for (long long b = 0; b < nblk; ++b) {
      const float s = block_tree(src + b * TF_BLK, cnt - b * TF_BLK, t.dk);
      if (threadIdx.x == 0) dst[b] = s;
      __syncthreads();
    }
    src = dst;
    dst = dst + ((nblk + 3) & ~3LL);
    cnt = nblk;
  }
  if (threadIdx.x == 0) {
    double tot[P::NR];
#pragma unroll
    for (int s = 0; s < P::NR; ++s) tot[s] = t.aux ? t.aux[s] : 0.0;
    tot[P::TS] = (double)__ldcg(src);
    if (slot < 0) {
      p.finalize(tot);
    } else {
      if (slot == P::TS)
#pragma unroll
        for (int s = 0; s < P::NR; ++s) p.defer[s] = tot[s];
      else
        p.defer[slot] = tot[P::TS];
    }
    *ticket = 0u;
  }
}

// Across ranks (P = 2^k equal aligned slabs): every rank's subtree total is a
// node of the global fl_sum tree at the same level, in rank order, so the
// rest of the tree is the pairwise tree over the gathered totals -- for a
// complex vector over the real halves and the imaginary halves separately
// (block order [re; im]), then one add.  The fp64 slots sum in rank order
// as finalize_kernel does.  Every rank computes the same value.
template <class P>
__global__ void tree_combine_kernel(P p, const double* __restrict__ gbuf, int nranks, int row, int cplx) {
  if (!p.prepare()) return;
  const TreeOut& t = p.tout;
  double tot[P::NR];
#pragma unroll
  for (int s = 0; s < P::NR; ++s) {
    tot[s] = gbuf[s];
    if (s != P::TS)
      for (int r = 1; r < nranks; ++r) tot[s] = red_combine(P::op(s), tot[s], gbuf[(size_t)r * row + s]);
  }
  float a[64], b[64];
  for (int r = 0; r < nranks; ++r) {
    a[r] = (float)gbuf[(size_t)r * row + P::TS];
    b[r] = cplx ? (float)gbuf[(size_t)r * row + P::NR] : 0.f;
  }
  for (int w = 1; w < nranks; w *= 2)
    for (int r = 0; r + w < nranks; r += 2 * w) {
      a[r] = dadd(a[r], a[r + w], t.dk);
      if (cplx) b[r] = dadd(b[r], b[r + w], t.dk);
    }
  tot[P::TS] = (double)(cplx ? dadd(a[0], b[0], t.dk) : a[0]);
  p.finalize(tot);
}

}  // namespace gadi
