// General-CSR operators (kernel K6): the same inner
// solvers, outer pass and power iteration as the stencil passes, for a
// `SparseMatrix` A that is not a recognised stencil (the reference's graded /
// mixed test families, Matrix Market inputs).  Splitting matrices H_low,
// S_low, S_low_T arrive as CSR with u_s values (REF/splitting.py:38-55).
//
// One thread per row; a row sums its entries in ascending column order
// (REF/sparsemat.py:192-198, scipy's csr_matvec for fp64): ordered
// non-contracted fp64 for A, compute-type FMAs for the u_s operators (storage
// model).  CG needs p at neighbouring rows before H p, so the fused stencil
// pass splits in two: p <- r + beta p (pointwise), then q = H p with the dot
// (gather).  All scalar logic is the stencil passes' (fin_* helpers).
#pragma once
#include "pointwise.cuh"

namespace gadi {

// device CSR: int64 row offsets, int32 columns, values of type VT
template <class VT>
struct CsrT {
  const long long* rp;
  const int* ci;
  const VT* v;
};

// sum_j a_ij x_j in ascending column order; XF maps the column value
template <bool ORD, class CT, class VT, class XF>
__device__ __forceinline__ CT csr_row(const CsrT<VT>& m, long long i, XF xf) {
  CT acc = CT(0);
  const long long e = m.rp[i + 1];
  for (long long k = m.rp[i]; k < e; ++k) acc = madd<ORD>((CT)m.v[k], xf(m.ci[k]), acc);
  return acc;
}

struct CsrBase : PwBase {
  static constexpr int VZ = 1;
};

// p <- (first ? f : round(f + beta p))   (inner.py:86 / 140; f = r or rbar)
template <class ST>
struct CsrDir : PwBase {
  typedef typename CTOf<ST>::type CT;
  static constexpr int VZ = (int)(16 / sizeof(ST)) >= 2 ? (int)(16 / sizeof(ST)) : 2, NR = 1;
  static constexpr bool HAS_RED = false;
  static constexpr int KID = K_HCG_A;
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  InnerState* st;
  const ST* f;
  ST* p;
  int first;
  CT beta;
  __device__ bool prepare() {
    if (st->done) return false;
    beta = (CT)st->beta;
    return true;
  }
  __device__ void apply(long long i, int nv, double (&)[1]) const {
    CT a[VZ], o[VZ];
    load_any<ST, VZ, true>(f, i, nv, a, true);
    if (first) {
#pragma unroll
      for (int k = 0; k < VZ; ++k) o[k] = a[k];
    } else {
      CT b[VZ];
      load_any<ST, VZ, false>(p, i, nv, b, true);
#pragma unroll
      for (int k = 0; k < VZ; ++k) o[k] = round_to<ST>(fma_rn(beta, b[k], a[k]));
    }
    store_any<ST, VZ>(p, i, nv, o, true);
  }
  __device__ void finalize(const double (&)[1]) const {}
};

// q = round(Op x) row by row, with the reduction of the solver step:
//   MODE 0  CG     Sum p.q          -> alpha   (inner.py:68-73)
//   MODE 1  CGNR   Sum w.w          -> alpha   (inner.py:121-126)
//   MODE 2  CGNR   rbar = S^T r, Sum rbar^2 -> beta (inner.py:134-138)
//   MODE 3  CGNR init: rbar = S^T rhs2, Sum rbar^2, Sum rhs2^2 (inner.py:108-116)
template <class ST, int MODE>
struct CsrSpmv : CsrBase {
  typedef typename CTOf<ST>::type CT;
  static constexpr int NR = MODE == 3 ? 2 : 1;
  static constexpr bool HAS_RED = true, ORD = std::is_same<ST, double>::value;
  static constexpr int KID = MODE == 0 ? K_HCG_A : (MODE == 1 ? K_CGNR_P1 : (MODE == 2 ? K_CGNR_P3 : K_CGNR_INIT));
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  InnerState* st;
  CsrT<ST> m;
  const ST* x;
  ST* q;
  double tol;
  int maxit;
  __device__ bool prepare() { return MODE == 3 ? true : !st->done; }
  __device__ void apply(long long i, int, double (&red)[NR]) const {
    const ST* xx = x;
    const CT y = round_to<ST>(csr_row<ORD, CT>(m, i, [xx](int j) { return cvt_in<CT>(xx[j]); }));
    q[i] = Store<ST>::from(y);
    if constexpr (MODE == 0) {
      red[0] += (double)(cvt_in<CT>(x[i]) * y);
    } else if constexpr (MODE == 3) {
      red[0] += (double)(y * y);
      const double f = (double)cvt_in<CT>(x[i]);
      red[1] += f * f;
    } else {
      red[0] += (double)(y * y);
    }
  }
  __device__ void finalize(const double (&t)[NR]) const {
    if constexpr (MODE == 0) fin_cg_alpha(st, t[0]);
    if constexpr (MODE == 1) fin_cgnr_alpha(st, t[0]);
    if constexpr (MODE == 2) fin_cgnr_beta(st, t[0]);
    if constexpr (MODE == 3) fin_cgnr_init(st, t[0], t[NR - 1], tol, maxit);
  }
};

// u += alpha p ; r -= alpha q ; Sum r^2
//   MODE 0 CG (fp32 products, inner.py:74-86)   MODE 1 CGNR (fp64 ||r||, inner.py:127-133)
template <class ST, int MODE>
struct CsrUpdate : PwBase {
  typedef typename CTOf<ST>::type CT;
  static constexpr int VZ = (int)(16 / sizeof(ST)) >= 2 ? (int)(16 / sizeof(ST)) : 2, NR = 1;
  static constexpr bool HAS_RED = true;
  static constexpr int KID = MODE == 0 ? K_HCG_B : K_CGNR_P2;
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  InnerState* st;
  const ST* p;
  const ST* q;
  ST* u;
  ST* r;
  CT alpha;
  __device__ bool prepare() {
    if (st->done) return false;
    alpha = (CT)st->alpha;
    return true;
  }
  __device__ void apply(long long i, int nv, double (&red)[1]) const {
    CT pp[VZ], qq[VZ], uu[VZ], rr[VZ], un[VZ], rn[VZ];
    load_any<ST, VZ, true>(p, i, nv, pp, true);
    load_any<ST, VZ, true>(q, i, nv, qq, true);
    load_any<ST, VZ, false>(u, i, nv, uu, true);
    load_any<ST, VZ, false>(r, i, nv, rr, true);
#pragma unroll
    for (int k = 0; k < VZ; ++k) {
      un[k] = round_to<ST>(fma_rn(alpha, pp[k], uu[k]));
      rn[k] = round_to<ST>(fma_rn(-alpha, qq[k], rr[k]));
      if (k < nv) red[0] += MODE == 0 ? (double)(rn[k] * rn[k]) : (double)rn[k] * (double)rn[k];
    }
    store_any<ST, VZ>(u, i, nv, un, true);
    store_any<ST, VZ>(r, i, nv, rn, true);
  }
  __device__ void finalize(const double (&t)[1]) const {
    if constexpr (MODE == 0) fin_cg_beta(st, t[0]);
    else fin_cgnr_relres(st, t[0]);
  }
};

// rhs2 = round(coeff z) -> r ; y = 0   (gadi.py:158, inner.py:108-112)
template <class ST>
struct CsrCgnrRhs : PwBase {
  typedef typename CTOf<ST>::type CT;
  static constexpr int VZ = (int)(16 / sizeof(ST)) >= 2 ? (int)(16 / sizeof(ST)) : 2, NR = 1;
  static constexpr bool HAS_RED = false;
  static constexpr int KID = K_CGNR_INIT;
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  const ST* z;
  ST* r;
  ST* y;
  CT coeff;
  __device__ bool prepare() { return true; }
  __device__ void apply(long long i, int nv, double (&)[1]) const {
    CT zz[VZ], f[VZ], zero[VZ];
    load_any<ST, VZ, true>(z, i, nv, zz, true);
#pragma unroll
    for (int k = 0; k < VZ; ++k) {
      f[k] = round_to<ST>(coeff * zz[k]);
      zero[k] = CT(0);
    }
    store_any<ST, VZ>(r, i, nv, f, true);
    store_any<ST, VZ>(y, i, nv, zero, true);
  }
  __device__ void finalize(const double (&)[1]) const {}
};

// x_new = round_u(x + y / scale)   (gadi.py:163)
template <class SU>
struct CsrOuterX : PwBase {
  static constexpr int VZ = 2, NR = 1;
  static constexpr bool HAS_RED = false;
  static constexpr int KID = K_OUTER;
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  const double* x;
  const SU* y;
  double* xout;
  double scale, inv_scale;
  int u32;
  __device__ bool prepare() { return true; }
  __device__ void apply(long long i, int nv, double (&)[1]) const {
#pragma unroll
    for (int k = 0; k < VZ; ++k)
      if (k < nv) {
        const double t = add_rn(x[i + k], mul_rn(cvt_in<double>(y[i + k]), inv_scale));  // scale = 2^k
        xout[i + k] = u32 ? (double)__double2float_rn(t) : t;
      }
  }
  __device__ void finalize(const double (&)[1]) const {}
};

// r = b - A x_new (u_r), the fp64 monitor residual and the monitor sums
// (gadi.py:147, 166-176; see the stencil Outer pass for the UR variants)
template <int UR, bool HAS_E>
struct CsrOuterR : CsrBase {
  static constexpr int NR = 6;
  static constexpr bool HAS_RED = true;
  static constexpr int KID = K_OUTER;
  static __device__ __forceinline__ int op(int s) { return s == 1 ? RED_MAX : RED_SUM; }
  CsrT<double> A;
  const double* x;   // x_new
  const double* xs;  // exact solution (unless ones)
  const double* b;
  double* r;
  OuterSums* out;
  int ones;
  __device__ bool prepare() { return true; }
  __device__ void apply(long long i, int, double (&red)[6]) const {
    const double* xx = x;
    const double ax = csr_row<true, double>(A, i, [xx](int j) { return xx[j]; });
    const double rmon = sub_rn(b[i], ax);  // gadi.py:166
    double ralg = rmon;
    if constexpr (UR == 1) {  // fp32 emulated: quantize(b - spmv(a32, x, fp32)) (sparsemat.py:234)
      float acc = 0.f;
      bool any = false;
      for (long long k = A.rp[i]; k < A.rp[i + 1]; ++k) {
        const float pr = __fmul_rn(__double2float_rn(A.v[k]), (float)x[A.ci[k]]);
        acc = any ? __fadd_rn(acc, pr) : pr;
        any = true;
      }
      ralg = (double)__fsub_rn(__double2float_rn(b[i]), acc);
    }
    if constexpr (UR == 2) {  // compensated (sparsemat.py:202-212)
      double s = b[i], c = 0.0;
      for (long long k = A.rp[i]; k < A.rp[i + 1]; ++k) {
        const double xxv = -x[A.ci[k]];
        const double pr = mul_rn(A.v[k], xxv);
        const double ep = fma_rn(A.v[k], xxv, -pr);
        const double sn = add_rn(s, pr);
        const double bb = sub_rn(sn, s);
        const double er = add_rn(sub_rn(s, sub_rn(sn, bb)), sub_rn(pr, bb));
        s = sn;
        c = add_rn(c, add_rn(er, ep));
      }
      ralg = add_rn(s, c);
    }
    r[i] = ralg;
    red[0] += rmon * rmon;
    const double ar = fabs(ralg);
    red[1] = (ar > red[1] || ar != ar) ? ar : red[1];
    red[2] += ralg * ralg;
    red[3] += x[i] * x[i];
    if constexpr (HAS_E) {
      const double* s = xs;
      const int o = ones;
      const double e = sub_rn(o ? 1.0 : xs[i], x[i]);
      const double ae = csr_row<true, double>(A, i, [xx, s, o](int j) { return sub_rn(o ? 1.0 : s[j], xx[j]); });
      red[4] += e * e;
      red[5] += ae * ae;
    }
  }
  __device__ void finalize(const double (&t)[6]) const {
#pragma unroll
    for (int s = 0; s < 6; ++s) out->v[s] = t[s];
  }
};

// power iteration (analysis.py:58-66): TRANS=false t = A (w / nw);
// TRANS=true w = A^T t, Sum w^2 -> sigma update
template <bool TRANS>
struct CsrNorm : CsrBase {
  static constexpr int NR = 1;
  static constexpr bool HAS_RED = TRANS;
  static constexpr int KID = TRANS ? K_NORM_B : K_NORM_A;
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  NormState* ns;
  CsrT<double> M;  // A or A^T
  const double* in;
  double* outv;
  double rnw;
  __device__ bool prepare() {
    if (ns->done) return false;
    rnw = 1.0 / ns->nw;
    return true;
  }
  __device__ void apply(long long i, int, double (&red)[1]) const {
    const double* xx = in;
    const double sc = rnw;
    const double y = TRANS ? csr_row<true, double>(M, i, [xx](int j) { return xx[j]; })
                           : csr_row<true, double>(M, i, [xx, sc](int j) { return xx[j] * sc; });
    outv[i] = y;
    if (TRANS) red[0] += y * y;
  }
  __device__ void finalize(const double (&t)[1]) const { fin_norm(ns, t[0]); }
};

// y = Op x on fp64 arrays of u_s images (sparsemat.spmv on a CSR operator);
// STRICT rounds every product and partial sum to u_s (REF/sparsemat.py:188-199)
template <class ST, bool STRICT>
struct CsrApply : CsrBase {
  typedef typename CTOf<ST>::type CT;
  static constexpr int NR = 1;
  static constexpr bool HAS_RED = false, ORD = std::is_same<ST, double>::value;
  static constexpr int KID = K_APPLY;
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  CsrT<double> m;  // fp64 images of the operator's u_s values
  const double* in;
  double* outv;
  __device__ bool prepare() { return true; }
  __device__ void apply(long long i, int, double (&)[1]) const {
    CT acc = CT(0);
    bool any = false;
    for (long long k = m.rp[i]; k < m.rp[i + 1]; ++k) {
      const CT a = (CT)m.v[k], xv = (CT)in[m.ci[k]];
      if constexpr (STRICT) {
        const CT pr = round_to<ST>(mul_rn(a, xv));
        acc = any ? round_to<ST>(add_rn(acc, pr)) : pr;
      } else {
        acc = madd<ORD>(a, xv, acc);
      }
      any = true;
    }
    outv[i] = (double)(STRICT ? acc : round_to<ST>(acc));
  }
  __device__ void finalize(const double (&)[1]) const {}
};

}  // namespace gadi
