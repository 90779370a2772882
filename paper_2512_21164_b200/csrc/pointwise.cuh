// Pointwise (halo-free) passes: the u_r -> u_s cast that opens every H-solve,
// the complex reaction-diffusion CGNR (S = alpha I + i V is diagonal in the
// interleaved complex layout, so S, S^T and S^T S need no neighbours), and
// small utilities (b = A 1, block <-> interleaved permutations).
#pragma once
#include "passes.cuh"

namespace gadi {

constexpr int PW_NT = 256;

template <class P>
__global__ void __launch_bounds__(PW_NT) pointwise_kernel(P p) {
  if (!p.prepare()) return;
  constexpr int VZ = P::VZ, NR = P::NR;
  double red[NR];
#pragma unroll
  for (int s = 0; s < NR; ++s) red[s] = 0.0;
  const long long n = p.n;
  const long long step = (long long)gridDim.x * PW_NT * VZ;
  if constexpr (TreeSlot<P>::value >= 0) {
    // reference rounding: warp-uniform trips, one fl_dot leaf per warp vector
    // block of 32 VZ elements (tout.tlog = log2(32 VZ), strict.cuh)
    const int lane = threadIdx.x & 31;
    for (long long w0 = ((long long)blockIdx.x * PW_NT + (threadIdx.x & ~31)) * VZ; w0 < n; w0 += step) {
      const long long i = w0 + (long long)lane * VZ;
      const int nv = (int)((n - i) < VZ ? ((n - i) > 0 ? (n - i) : 0) : VZ);
      if (nv > 0) p.apply(i, nv, red);
      if (p.tout.tlog >= 0) tree_emit<VZ, 2>(p.tout, i, nv > 0, lane, red[TreeSlot<P>::value]);
      red[TreeSlot<P>::value] = 0.0;
    }
  } else {
    for (long long i = ((long long)blockIdx.x * PW_NT + threadIdx.x) * VZ; i < n; i += step) {
      const int nv = (int)((n - i) < VZ ? (n - i) : VZ);
      p.apply(i, nv, red);
    }
  }
  if constexpr (P::HAS_RED) {
    double tot[NR];
    int ops[NR];
#pragma unroll
    for (int s = 0; s < NR; ++s) ops[s] = P::op(s);
    if (grid_finish<NR, PW_NT>(red, ops, p.partials, p.pstride, p.ticket, tot)) {
      if (threadIdx.x == 0) finish_pass(p, tot);
    }
  }
}

struct PwBase {
  long long n;
  double* defer;  // slab decomposition: this rank's row of the gather buffer
  double* partials;
  unsigned int* ticket;
  int pstride;
  TreeOut tout;   // reference rounding: fl_dot leaves (strict.cuh)
};

__device__ __forceinline__ void init_state(InnerState* st, double tol, int maxit) {
  st->tol = tol;
  st->maxit = maxit;
  st->it = 0;
  st->breakdown = 0;
  st->converged = 0;
  st->done = 0;
  st->beta = 0.0;
  st->relres = 1.0;
}

// r_s = RNE_{u_s}(scale * r) (gadi.py:151-153); z = 0; rs = r_s.r_s;
// nrhs = ||r_s||_2 (fp64; inner.py:56-63) and the zero-rhs short cut.
template <class ST, bool RF = false>
struct HcgInit : PwBase {
  typedef typename CTOf<ST>::type CT;
  static constexpr int VZ = (int)(16 / sizeof(ST)) >= 2 ? (int)(16 / sizeof(ST)) : 2;
  static constexpr int NR = 2;
  static constexpr int TS = (RF && !std::is_same<ST, double>::value) ? 0 : -1;
  static constexpr bool HAS_RED = true;
  static constexpr int KID = K_HCG_INIT;
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  const double* r64;
  ST* rs;
  ST* z;
  InnerState* st;
  double scale, tol;
  int maxit;
  __device__ bool prepare() { return true; }
  __device__ void apply(long long i, int nv, double (&red)[2]) const {
    double rr[VZ];
    load_any<double, VZ, true>(r64, i, nv, rr, true);
    CT f[VZ], zero[VZ];
#pragma unroll
    for (int k = 0; k < VZ; ++k) {
      f[k] = cvt_in<CT>(Store<ST>::from(scale * rr[k]));
      zero[k] = CT(0);
      if (k < nv) {
        if constexpr (TS < 0) red[0] += (double)(f[k] * f[k]);
        red[1] += (double)f[k] * (double)f[k];
      }
    }
    if constexpr (TS >= 0) red[0] = dot_leaf<VZ, 2>(tout, i, nv, f, f);  // inner.py:63 fl_dot(r, r)
    store_any<ST, VZ>(rs, i, nv, f, true);
    store_any<ST, VZ>(z, i, nv, zero, true);
  }
  __device__ void finalize(const double (&t)[2]) const {
    init_state(st, tol, maxit);
    const double nrhs = sqrt(t[1]);
    st->nrhs = nrhs;
    st->rs = t[0];
    if (nrhs == 0.0) {  // inner.py:58-59
      st->converged = 1;
      st->relres = 0.0;
      st->done = 1;
    } else if (maxit <= 0) {
      st->done = 1;
    }
  }
};

// Z-lag (GADI_ZLAG, passes.cuh HcgA): the last CG iteration's z += alpha p
// (inner.py:74), after the loop.  The iteration count and the breakdown flag
// select it: K = it - 1 iterations ran their HcgB (p_K in P[it & 1]); a
// breakdown in HcgA(K) returns before the update (inner.py:70-72), as does a
// loop that never started.
template <class ST, bool RF = false>
struct HcgZFinal : PwBase {
  typedef typename CTOf<ST>::type CT;
  static constexpr int VZ = (int)(16 / sizeof(ST)) >= 2 ? (int)(16 / sizeof(ST)) : 2;
  static constexpr int NR = 1;
  static constexpr int TS = -1;
  static constexpr bool HAS_RED = false;
  static constexpr int KID = K_HCG_Z;
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  const InnerState* st;
  const ST* P0;
  const ST* P1;
  ST* z;
  const ST* p;
  CT alpha;
  __device__ bool prepare() {
    if (st->breakdown || st->it <= 0) return false;
    alpha = (CT)st->alpha;
    p = (st->it & 1) ? P1 : P0;
    return true;
  }
  __device__ void apply(long long i, int nv, double (&)[1]) const {
    CT pv[VZ], zv[VZ], zn[VZ];
    load_any<ST, VZ, true>(p, i, nv, pv, true);
    load_any<ST, VZ, false>(z, i, nv, zv, true);
    axpy_m<ST, RF>(alpha, pv, zv, zn);
    store_exact<ST, VZ>(z, i, nv, zn, true);
  }
  __device__ void finalize(const double (&)[1]) const {}
};

// ---------------------------------------------------------------- complex S
// Interleaved pairs (re, im).  S (a + ib) = (alpha a - v b) + i (v a + alpha b),
// S^T = alpha I - N flips the sign of v.  Accumulation order follows the CSR
// rows of S = [[aI, -V], [V, aI]]: real row  alpha*a then (-v)*b ;
// imaginary row v*a then alpha*b.
template <bool ORD, class CT>
__device__ __forceinline__ void cmul_s(CT al, CT v, CT a, CT b, CT& re, CT& im) {
  if (ORD) {
    re = add_rn(mul_rn(al, a), mul_rn(-v, b));
    im = add_rn(mul_rn(v, a), mul_rn(al, b));
  } else {
    re = fma_rn(-v, b, al * a);
    im = fma_rn(al, b, v * a);
  }
}

template <class ST>
struct CplxBase : PwBase {
  typedef typename CTOf<ST>::type CT;
  static constexpr int VZ = (int)(16 / sizeof(ST)) >= 2 ? (int)(16 / sizeof(ST)) : 2;
  static constexpr bool ORD = std::is_same<ST, double>::value;
  const ST* vs;  // u_s image of v (one per complex point)
  CT al;         // u_s image of alpha
  __device__ void loadv(long long i, int nv, CT (&vv)[VZ]) const {
    if (nv == VZ) {
      // VZ / 2 consecutive potentials, one vector load (i is a multiple of VZ)
      CT t[VZ / 2];
      load_vec<ST, VZ / 2, true>(vs, i >> 1, t);
#pragma unroll
      for (int k = 0; k < VZ; k += 2) vv[k] = vv[k + 1] = t[k / 2];
      return;
    }
#pragma unroll
    for (int k = 0; k < VZ; k += 2) {
      const CT t = (k < nv) ? cvt_in<CT>(vs[(i + k) >> 1]) : CT(0);
      vv[k] = t;
      vv[k + 1] = t;
    }
  }
  // out = round(S^T a) for the pairs in a
  __device__ void st_apply(const CT (&a)[VZ], const CT (&vv)[VZ], CT (&o)[VZ]) const {
#pragma unroll
    for (int k = 0; k < VZ; k += 2) {
      CT re, im;
      cmul_s<ORD>(al, -vv[k], a[k], a[k + 1], re, im);
      o[k] = round_to<ST>(re);
      o[k + 1] = round_to<ST>(im);
    }
  }
  // out = round(S a): w is a u_s vector of the storage model (see round_vec)
  __device__ void s_apply(const CT (&a)[VZ], const CT (&vv)[VZ], CT (&o)[VZ]) const {
#pragma unroll
    for (int k = 0; k < VZ; k += 2) {
      CT re, im;
      cmul_s<ORD>(al, vv[k], a[k], a[k + 1], re, im);
      o[k] = round_to<ST>(re);
      o[k + 1] = round_to<ST>(im);
    }
  }
  // reference rounding of S (sgn = 1) or S^T (sgn = -1), CSR row order:
  // real row fl(fl(alpha a) + fl((-v) b)), imaginary row fl(fl(v a) + fl(alpha b))
  __device__ void apply_ref(CT sgn, const CT (&a)[VZ], const CT (&vv)[VZ], CT (&o)[VZ]) const {
#pragma unroll
    for (int k = 0; k < VZ; k += 2) {
      const CT v = sgn * vv[k];
      o[k] = round_to<ST>(add_rn(round_to<ST>(mul_rn(al, a[k])), round_to<ST>(mul_rn(-v, a[k + 1]))));
      o[k + 1] = round_to<ST>(add_rn(round_to<ST>(mul_rn(v, a[k])), round_to<ST>(mul_rn(al, a[k + 1]))));
    }
  }
};

// rhs2 = round(coeff z) ; r = rhs2 ; y = 0 ; rs = |round(S^T rhs2)|^2 ; nrhs
template <class ST, bool RF = false>
struct CInit : CplxBase<ST> {
  typedef CplxBase<ST> B;
  typedef typename B::CT CT;
  static constexpr int VZ = B::VZ, NR = 2;
  static constexpr int TS = (RF && !B::ORD) ? 0 : -1;
  static constexpr bool HAS_RED = true;
  static constexpr int KID = K_C_INIT;
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  const ST* z;
  ST* r;
  ST* y;
  InnerState* st;
  CT coeff;
  double tol;
  int maxit;
  __device__ bool prepare() { return true; }
  __device__ void apply(long long i, int nv, double (&red)[2]) const {
    CT zz[VZ], vv[VZ], f[VZ], rb[VZ], zero[VZ];
    load_any<ST, VZ, true>(z, i, nv, zz, true);
    this->loadv(i, nv, vv);
#pragma unroll
    for (int k = 0; k < VZ; ++k) {
      f[k] = round_to<ST>(mul_rn(coeff, zz[k]));
      zero[k] = CT(0);
    }
    if constexpr (RF) this->apply_ref(CT(-1), f, vv, rb);
    else this->st_apply(f, vv, rb);
#pragma unroll
    for (int k = 0; k < VZ; ++k)
      if (k < nv) {
        if constexpr (TS < 0) red[0] += (double)(rb[k] * rb[k]);
        red[1] += (double)f[k] * (double)f[k];
      }
    if constexpr (TS >= 0) red[0] = dot_leaf<VZ, 1>(this->tout, i, nv, rb, rb);
    store_any<ST, VZ>(r, i, nv, f, true);
    store_any<ST, VZ>(y, i, nv, zero, true);
  }
  __device__ void finalize(const double (&t)[2]) const {
    init_state(st, tol, maxit);
    const double nrhs = sqrt(t[1]);
    st->nrhs = nrhs;
    st->rs = t[0];
    if (nrhs == 0.0) {
      st->converged = 1;
      st->relres = 0.0;
      st->done = 1;
    } else if (maxit <= 0) {
      st->done = 1;
    }
  }
};

// p <- rbar (+ beta p), rbar = round(S^T r) recomputed pointwise ; w = S p ; |w|^2
template <class ST, bool RF = false>
struct CP1 : CplxBase<ST> {
  typedef CplxBase<ST> B;
  typedef typename B::CT CT;
  static constexpr int VZ = B::VZ, NR = 1;
  static constexpr int TS = (RF && !B::ORD) ? 0 : -1;
  static constexpr bool HAS_RED = true;
  static constexpr int KID = K_C_P1;
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  const ST* r;
  ST* p;
  InnerState* st;
  CT beta;
  bool first;
  __device__ bool prepare() {
    if (st->done) return false;
    first = (st->it == 0);
    beta = (CT)st->beta;
    return true;
  }
  __device__ void apply(long long i, int nv, double (&red)[1]) const {
    CT rr[VZ], vv[VZ], rb[VZ], pp[VZ], w[VZ];
    load_any<ST, VZ, true>(r, i, nv, rr, true);
    this->loadv(i, nv, vv);
    if constexpr (RF) this->apply_ref(CT(-1), rr, vv, rb);
    else this->st_apply(rr, vv, rb);
    if (!first) {
      load_any<ST, VZ, false>(p, i, nv, pp, true);
#pragma unroll
      for (int k = 0; k < VZ; ++k) pp[k] = RF ? axpy_ref1<ST>(beta, pp[k], rb[k]) : round_to<ST>(fma_rn(beta, pp[k], rb[k]));
    } else {
#pragma unroll
      for (int k = 0; k < VZ; ++k) pp[k] = rb[k];
    }
    if constexpr (RF) this->apply_ref(CT(1), pp, vv, w);
    else this->s_apply(pp, vv, w);
    if constexpr (TS >= 0) {
      red[0] = dot_leaf<VZ, 1>(this->tout, i, nv, w, w);
    } else {
#pragma unroll
      for (int k = 0; k < VZ; ++k)
        if (k < nv) red[0] += (double)(w[k] * w[k]);
    }
    store_any<ST, VZ>(p, i, nv, pp, true);
  }
  __device__ void finalize(const double (&t)[1]) const {
    if (t[0] <= 0.0) {
      st->breakdown = 1;
      st->done = 1;
      return;
    }
    st->alpha = sround(st->rs / t[0], ScalarRnd<ST, RF>::value);
  }
};

// y += alpha p ; r -= alpha S p ; fp64 |r|^2 ; rs_new = |round(S^T r)|^2 ; beta
template <class ST, bool RF = false>
struct CP2 : CplxBase<ST> {
  typedef CplxBase<ST> B;
  typedef typename B::CT CT;
  static constexpr int VZ = B::VZ, NR = 2;
  static constexpr int TS = (RF && !B::ORD) ? 1 : -1;
  static constexpr bool HAS_RED = true;
  static constexpr int KID = K_C_P2;
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  const ST* p;
  ST* y;
  ST* r;
  InnerState* st;
  CT alpha;
  __device__ bool prepare() {
    if (st->done) return false;
    alpha = (CT)st->alpha;
    return true;
  }
  __device__ void apply(long long i, int nv, double (&red)[2]) const {
    CT pp[VZ], vv[VZ], w[VZ], yy[VZ], rr[VZ], rb[VZ];
    load_any<ST, VZ, true>(p, i, nv, pp, true);
    load_any<ST, VZ, false>(y, i, nv, yy, true);
    load_any<ST, VZ, false>(r, i, nv, rr, true);
    this->loadv(i, nv, vv);
    if constexpr (RF) this->apply_ref(CT(1), pp, vv, w);
    else this->s_apply(pp, vv, w);
#pragma unroll
    for (int k = 0; k < VZ; ++k) {
      yy[k] = RF ? axpy_ref1<ST>(alpha, pp[k], yy[k]) : round_to<ST>(fma_rn(alpha, pp[k], yy[k]));
      rr[k] = RF ? axpy_ref1<ST>(-alpha, w[k], rr[k]) : round_to<ST>(fma_rn(-alpha, w[k], rr[k]));
    }
    if constexpr (RF) this->apply_ref(CT(-1), rr, vv, rb);
    else this->st_apply(rr, vv, rb);
#pragma unroll
    for (int k = 0; k < VZ; ++k)
      if (k < nv) {
        red[0] += (double)rr[k] * (double)rr[k];
        if constexpr (TS < 0) red[1] += (double)(rb[k] * rb[k]);
      }
    if constexpr (TS >= 0) red[1] = dot_leaf<VZ, 1>(this->tout, i, nv, rb, rb);
    store_any<ST, VZ>(y, i, nv, yy, true);
    store_any<ST, VZ>(r, i, nv, rr, true);
  }
  __device__ void finalize(const double (&t)[2]) const {
    const int it = st->it + 1;
    st->it = it;
    const double relres = sqrt(t[0]) / st->nrhs;  // inner.py:130
    st->relres = relres;
    if (relres <= st->tol) {
      st->converged = 1;
      st->done = 1;
      return;
    }
    if (it >= st->maxit) {
      st->done = 1;
      return;
    }
    const double rs_new = t[1];
    if (rs_new <= 0.0) {  // inner.py:136-137
      st->done = 1;
      return;
    }
    st->beta = sround(rs_new / st->rs, ScalarRnd<ST, RF>::value);
    st->rs = rs_new;
  }
};

// y = S x or S^T x for the crd family (interleaved), fp64 arrays of u_s images.
template <class ST, bool TRANS, bool STRICT>
struct CApply : CplxBase<ST> {
  typedef CplxBase<ST> B;
  typedef typename B::CT CT;
  static constexpr int VZ = B::VZ, NR = 1;
  static constexpr bool HAS_RED = false;
  static constexpr int KID = K_APPLY;
  static __device__ __forceinline__ int op(int) { return RED_SUM; }
  const double* in;
  double* outv;
  __device__ bool prepare() { return true; }
  __device__ void apply(long long i, int nv, double (&)[1]) const {
    double a[VZ], o[VZ];
    CT vv[VZ];
    load_any<double, VZ, true>(in, i, nv, a, true);
    this->loadv(i, nv, vv);
#pragma unroll
    for (int k = 0; k < VZ; k += 2) {
      const CT v = TRANS ? -vv[k] : vv[k];
      const CT xa = (CT)a[k], xb = (CT)a[k + 1];
      CT re, im;
      if (STRICT) {
        // real row: alpha*a then (-v)*b ; imaginary row: v*a then alpha*b
        re = round_to<ST>(add_rn(round_to<ST>(mul_rn(this->al, xa)), round_to<ST>(mul_rn(-v, xb))));
        im = round_to<ST>(add_rn(round_to<ST>(mul_rn(v, xa)), round_to<ST>(mul_rn(this->al, xb))));
      } else {
        cmul_s<B::ORD>(this->al, v, xa, xb, re, im);
      }
      o[k] = (double)re;
      o[k + 1] = (double)im;
    }
    store_any<double, VZ>(outv, i, nv, o, true);
  }
  __device__ void finalize(const double (&)[1]) const {}
};

// ---------------------------------------------------------------- utilities
// b = A 1 in the reference's CSR row order (problems.py:42-45): each present
// coefficient is added as 1.0 * c, ascending by column.
struct RhsOnes {
  int nx, ny, nz, zs;  // zs = 2 for the crd interleaved layout; nx = global planes
  int x0;              // global index of this slab's first plane
  long long plane;
  CoefT<double> A;
  const double* v;  // crd potential (may be null)
  double* b;
};

static __global__ void rhs_ones_kernel(RhsOnes p, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long x = p.x0 + i / p.plane, rem = i % p.plane;
    const int y = (int)(rem / p.nz), z = (int)(rem % p.nz);
    const int zc = z / p.zs;         // grid column
    const int ncol = p.nz / p.zs;
    double acc = 0.0;
    const bool cplx = p.zs == 2;
    if (cplx && (z & 1)) acc = add_rn(0.0, mul_rn(p.v[i >> 1], 1.0));
    const CoefT<double>& c = p.A;
    if (c.lo[0] != 0.0 && x > 0) acc = add_rn(acc, mul_rn(c.lo[0], 1.0));
    if (c.lo[1] != 0.0 && y > 0) acc = add_rn(acc, mul_rn(c.lo[1], 1.0));
    if (c.lo[2] != 0.0 && zc > 0) acc = add_rn(acc, mul_rn(c.lo[2], 1.0));
    if (c.d != 0.0) acc = add_rn(acc, mul_rn(c.d, 1.0));
    if (c.up[2] != 0.0 && zc < ncol - 1) acc = add_rn(acc, mul_rn(c.up[2], 1.0));
    if (c.up[1] != 0.0 && y < p.ny - 1) acc = add_rn(acc, mul_rn(c.up[1], 1.0));
    if (c.up[0] != 0.0 && x < p.nx - 1) acc = add_rn(acc, mul_rn(c.up[0], 1.0));
    if (cplx && !(z & 1)) acc = add_rn(acc, mul_rn(-p.v[i >> 1], 1.0));
    p.b[i] = acc;
  }
}

// block [re(0..m); im(0..m)] <-> interleaved (re, im) pairs, m = n/2
static __global__ void interleave_kernel(const double* __restrict__ blk, double* __restrict__ il, long long m) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    il[2 * i] = blk[i];
    il[2 * i + 1] = blk[m + i];
  }
}
static __global__ void deinterleave_kernel(const double* __restrict__ il, double* __restrict__ blk, long long m) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    blk[i] = il[2 * i];
    blk[m + i] = il[2 * i + 1];
  }
}

template <class ST>
__global__ void quantize_kernel(const double* __restrict__ in, ST* __restrict__ out, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = Store<ST>::from(in[i]);
}

template <class ST>
__global__ void widen_kernel(const ST* __restrict__ in, double* __restrict__ out, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = cvt_in<double>(in[i]);
}

// Philox-free deterministic start vector for the power iteration when no
// host vector is supplied: splitmix64 -> Box-Muller normals.
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// element i of this slab is global element i0 + i (the vector is the same
// for any slab decomposition)
static __global__ void randn_kernel(double* __restrict__ v, long long n, unsigned long long seed, long long i0) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long gi = (unsigned long long)(i0 + i);
    const unsigned long long a = splitmix64(seed ^ (2ull * gi));
    const unsigned long long b = splitmix64(seed ^ (2ull * gi + 1ull));
    const double u1 = ((a >> 11) + 1.0) * (1.0 / 9007199254740993.0);
    const double u2 = (b >> 11) * (1.0 / 9007199254740992.0);
    v[i] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
  }
}

// v <- v / ||v|| after a sum-of-squares reduction (analysis.py:57)
static __global__ void sumsq_kernel(const double* __restrict__ v, long long n, double* __restrict__ partials) {
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    s += v[i] * v[i];
  double a[1] = {s};
  const int ops[1] = {RED_SUM};
  block_reduce<1, 256>(a, ops);
  if (threadIdx.x == 0) partials[blockIdx.x] = a[0];
}
// sum the per-block partials in block order into this rank's gather row
static __global__ void partials_total_kernel(const double* __restrict__ partials, int nparts, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nparts; ++i) s += partials[i];
    out[0] = s;
  }
}
// v <- v / sqrt(sum of the gathered rows, in rank order)
static __global__ void scale_by_norm_kernel(double* __restrict__ v, long long n, const double* __restrict__ rows,
                                            int nranks, int row) {
  __shared__ double nrm;
  if (threadIdx.x == 0) {
    double s = rows[0];
    for (int r = 1; r < nranks; ++r) s += rows[(size_t)r * row];
    nrm = sqrt(s);
  }
  __syncthreads();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    v[i] = v[i] / nrm;
}

static __global__ void norm_state_init(NormState* ns, double tol, int maxit) {
  ns->nw = 1.0;  // first NormA pass divides the (already normalised) start vector by 1
  ns->sigma = 0.0;
  ns->tol = tol;
  ns->it = 0;
  ns->maxit = maxit;
  ns->done = maxit <= 0 ? 1 : 0;
}

}  // namespace gadi
