// Reference-rounding mode of the inner solvers (gadi_set_rounding(ctx, 1, …)).
//
// The reference emulates every low-precision operation as "exact fp64
// result, then one RNE rounding to the format" (gadimp/precision.py:136-186,
// sparsemat.py:178-199, inner.py:47-143), with dot products summed by a
// pairwise tree that rounds after every level (precision.py:189-220).  This
// file restates that arithmetic on the device literally: vectors are fp64
// arrays holding u_s images, every product / sum / axpy is an fp64 op followed
// by q(., fmt), and fl_dot is the same adjacent-pair tree (one launch per
// level).  The iterates are therefore bitwise the reference's; the only
// unpinned quantities are the fp64 BLAS norms (||rhs||, the CGNR ||r||) whose
// summation order numpy does not fix.
//
// This is the parity mode (host-driven, one synchronisation per reduction);
// the benchmark path is the fused storage-model engine (engine.cuh).
#include <cmath>
#include <vector>
#include "engine.cuh"

namespace gadi {

namespace {

constexpr int XT = 256;

__host__ __device__ inline double qf(double v, int f) {
  switch (f) {
    case GADI_BF16: return (double)__bfloat162float(__float2bfloat16_rn((float)v));  // via fp32, precision.py:113-125
    case GADI_FP16: return (double)__half2float(__double2half(v));
    case GADI_FP32: return (double)(float)v;
    default: return v;
  }
}

// Operator of the exact SpMV: a real constant-coefficient stencil on (nx, ny,
// nz), or the crd family on the interleaved layout (nz = 2 n_g, component
// stride 2): op 1 = H = alpha I + L on each component, 2 = S = alpha + iV,
// 3 = S^T = alpha - iV (problems.py:96-120, block form [[aI, -V], [V, aI]]).
struct XOp {
  CoefT<double> c;
  int nx, ny, nz;
  int cplx, which;  // which: 1 H, 2 S, 3 S^T (crd only)
  double alpha;     // u_s image of alpha (crd S diagonal)
  const double* v;  // crd potential (fp64, per grid point)
  // general CSR operator (kind GADI_CSR): values are the u_s images
  const long long* rp;
  const int* ci;
  const double* cv;
};

// Row sum in ascending column order: first product, then q(acc + prod)
// (sparsemat.py:192-198); zero coefficients are absent from the CSR.
struct RowAcc {
  double acc;
  bool any;
  int f;
  __device__ void add(double coef, double x) {
    const double pr = qf(coef * x, f);
    acc = any ? qf(acc + pr, f) : pr;
    any = true;
  }
};

__global__ void xspmv_kernel(XOp op, const double* __restrict__ in, double* __restrict__ out, long long n, int f) {
  for (long long i = (long long)blockIdx.x * XT + threadIdx.x; i < n; i += (long long)gridDim.x * XT) {
    RowAcc r{0.0, false, f};
    if (op.rp) {
      for (long long k = op.rp[i]; k < op.rp[i + 1]; ++k) r.add(op.cv[k], in[op.ci[k]]);
    } else if (!op.cplx) {
      const long long plane = (long long)op.ny * op.nz;
      const long long x = i / plane, rem = i % plane;
      const int y = (int)(rem / op.nz), z = (int)(rem % op.nz);
      const CoefT<double>& c = op.c;
      if (c.lo[0] != 0.0 && x > 0) r.add(c.lo[0], in[i - plane]);
      if (c.lo[1] != 0.0 && y > 0) r.add(c.lo[1], in[i - op.nz]);
      if (c.lo[2] != 0.0 && z > 0) r.add(c.lo[2], in[i - 1]);
      if (c.d != 0.0) r.add(c.d, in[i]);
      if (c.up[2] != 0.0 && z < op.nz - 1) r.add(c.up[2], in[i + 1]);
      if (c.up[1] != 0.0 && y < op.ny - 1) r.add(c.up[1], in[i + op.nz]);
      if (c.up[0] != 0.0 && x < op.nx - 1) r.add(c.up[0], in[i + plane]);
    } else {
      const long long g = i >> 1;  // grid point
      const int comp = (int)(i & 1);
      const int ng = op.nz / 2;
      if (op.which == 1) {
        const long long gplane = (long long)op.ny * ng;  // grid points per x-plane
        const long long gx = g / gplane, grem = g % gplane;
        const int gy = (int)(grem / ng), gz = (int)(grem % ng);
        const CoefT<double>& c = op.c;
        if (c.lo[0] != 0.0 && gx > 0) r.add(c.lo[0], in[i - 2LL * gplane]);
        if (c.lo[1] != 0.0 && gy > 0) r.add(c.lo[1], in[i - 2LL * ng]);
        if (c.lo[2] != 0.0 && gz > 0) r.add(c.lo[2], in[i - 2]);
        if (c.d != 0.0) r.add(c.d, in[i]);
        if (c.up[2] != 0.0 && gz < ng - 1) r.add(c.up[2], in[i + 2]);
        if (c.up[1] != 0.0 && gy < op.ny - 1) r.add(c.up[1], in[i + 2LL * ng]);
        if (c.up[0] != 0.0 && gx < op.nx - 1) r.add(c.up[0], in[i + 2LL * gplane]);
      } else {
        // S:   re row: a x_re, then -v x_im ; im row: v x_re, then a x_im
        // S^T: re row: a x_re, then +v x_im ; im row: -v x_re, then a x_im
        const double vq = qf(op.v[g], f);
        const double sgn = op.which == 2 ? 1.0 : -1.0;
        if (comp == 0) {
          r.add(op.alpha, in[i]);
          if (vq != 0.0) r.add(-sgn * vq, in[i + 1]);
        } else {
          if (vq != 0.0) r.add(sgn * vq, in[i - 1]);
          r.add(op.alpha, in[i]);
        }
      }
    }
    out[i] = r.any ? r.acc : 0.0;
  }
}

// out = q(s * in)
__global__ void xscale_kernel(double* __restrict__ out, const double* __restrict__ in, double s, long long n, int f) {
  for (long long i = (long long)blockIdx.x * XT + threadIdx.x; i < n; i += (long long)gridDim.x * XT)
    out[i] = qf(s * in[i], f);
}

// out = q(y + sgn * q(a * x))   (inner.py:74-75, 85, 127-128, 139)
__global__ void xaxpy_kernel(double* out, const double* y, double a, const double* x, double sgn, long long n, int f) {
  for (long long i = (long long)blockIdx.x * XT + threadIdx.x; i < n; i += (long long)gridDim.x * XT) {
    const double t = qf(a * x[i], f);
    out[i] = qf(sgn > 0 ? y[i] + t : y[i] - t, f);
  }
}

// T[pos(i)] = q(a_i * b_i) with pos the reference (block) index of i
__global__ void xprod_kernel(double* __restrict__ T, const double* __restrict__ a, const double* __restrict__ b,
                             long long n, int f, int cplx) {
  const long long m = n / 2;
  for (long long i = (long long)blockIdx.x * XT + threadIdx.x; i < n; i += (long long)gridDim.x * XT) {
    const long long j = cplx ? ((i & 1) ? m + (i >> 1) : (i >> 1)) : i;
    T[j] = qf(a[i] * b[i], f);
  }
}

// one level of fl_sum (precision.py:202-206): out[k] = q(in[2k] + in[2k+1]);
// an odd tail element is carried unchanged
__global__ void xtree_kernel(double* __restrict__ out, const double* __restrict__ in, long long size, int f) {
  const long long m = size / 2;
  for (long long k = (long long)blockIdx.x * XT + threadIdx.x; k < m; k += (long long)gridDim.x * XT)
    out[k] = qf(in[2 * k] + in[2 * k + 1], f);
  if ((size & 1) && blockIdx.x == 0 && threadIdx.x == 0) out[m] = in[size - 1];
}

// per-block fp64 sums of squares (fixed order within a block)
__global__ void xsumsq_kernel(const double* __restrict__ v, long long n, double* __restrict__ partials) {
  double s = 0.0;
  for (long long i = (long long)blockIdx.x * XT + threadIdx.x; i < n; i += (long long)gridDim.x * XT) s += v[i] * v[i];
  double a[1] = {s};
  const int ops[1] = {RED_SUM};
  block_reduce<1, XT>(a, ops);
  if (threadIdx.x == 0) partials[blockIdx.x] = a[0];
}

int blocks_for(const Ctx* c, long long n) {
  return (int)std::max<long long>(1, std::min<long long>((n + XT - 1) / XT, (long long)c->sms * 8));
}

struct X {
  Ctx* c;
  long long n;
  int f, df;
  double* t[2];  // tree ping-pong

  int launched() {
    c->launches++;
    GADI_CUDA(cudaGetLastError());
    return 0;
  }
  int spmv(const XOp& op, const double* in, double* out) {
    xspmv_kernel<<<blocks_for(c, n), XT, 0, c->stream>>>(op, in, out, n, f);
    return launched();
  }
  int scale(double* out, const double* in, double s) {
    xscale_kernel<<<blocks_for(c, n), XT, 0, c->stream>>>(out, in, s, n, f);
    return launched();
  }
  int axpy(double* out, const double* y, double a, const double* x, double sgn) {
    xaxpy_kernel<<<blocks_for(c, n), XT, 0, c->stream>>>(out, y, a, x, sgn, n, f);
    return launched();
  }
  // fl_dot(a, b, dfmt) (precision.py:209-220) -> host
  int dot(const double* a, const double* b, double* out) {
    xprod_kernel<<<blocks_for(c, n), XT, 0, c->stream>>>(t[0], a, b, n, df, c->kind == GADI_COMPLEX);
    GADI_TRY(launched());
    long long size = n;
    int cur = 0;
    while (size > 1) {
      const long long m = size / 2 + (size & 1);
      xtree_kernel<<<blocks_for(c, size / 2 + 1), XT, 0, c->stream>>>(t[cur ^ 1], t[cur], size, df);
      GADI_TRY(launched());
      cur ^= 1;
      size = m;
    }
    GADI_CUDA(cudaMemcpyAsync(out, t[cur], sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    GADI_CUDA(cudaStreamSynchronize(c->stream));
    return 0;
  }
  // fp64 2-norm (np.linalg.norm; BLAS summation order is not pinned)
  int norm(const double* v, double* out) {
    const int nb = blocks_for(c, n);
    xsumsq_kernel<<<nb, XT, 0, c->stream>>>(v, n, c->partials);
    GADI_TRY(launched());
    std::vector<double> h(nb);
    GADI_CUDA(cudaMemcpyAsync(h.data(), c->partials, sizeof(double) * nb, cudaMemcpyDeviceToHost, c->stream));
    GADI_CUDA(cudaStreamSynchronize(c->stream));
    double s = 0.0;
    for (double p : h) s += p;
    *out = std::sqrt(s);
    return 0;
  }
};

XOp make_op(const Ctx* c, int which) {
  XOp o;
  o.c = which == 1 ? c->H : (which == 2 ? c->S : c->ST);
  o.nx = c->nx;
  o.ny = c->ny;
  o.nz = c->nz;
  o.cplx = c->kind == GADI_COMPLEX;
  o.which = which;
  o.alpha = c->d.alpha_s;
  o.v = c->v64;
  o.rp = nullptr;
  o.ci = nullptr;
  o.cv = nullptr;
  if (c->kind == GADI_CSR) {
    const CsrDev& m = c->csr[which == 1 ? CS_H : (which == 2 ? CS_S : CS_ST)];
    o.rp = m.rp;
    o.ci = m.ci;
    o.cv = m.v64;
  }
  return o;
}

void set_stats(InnerState* s, int it, double relres, bool conv, bool brk) {
  s->it = it;
  s->relres = relres;
  s->converged = conv ? 1 : 0;
  s->breakdown = brk ? 1 : 0;
  s->done = 1;
}

}  // namespace

int exact_alloc(Ctx* c) {
  if (c->ex[0]) return 0;
  for (int k = 0; k < EX_N; ++k) GADI_CUDA(cudaMalloc((void**)&c->ex[k], sizeof(double) * (size_t)c->n));
  return 0;
}

void exact_free(Ctx* c) {
  for (int k = 0; k < EX_N; ++k)
    if (c->ex[k]) {
      cudaFree(c->ex[k]);
      c->ex[k] = nullptr;
    }
}

// cg_spd(H_low, q(scale r64), tol, maxit, u_s, strict_model) (inner.py:47-89);
// the solution is left in ex[EX_Z].
int exact_h_solve(Ctx* c, const double* r64, double scale, double tol, int maxit) {
  GADI_TRY(exact_alloc(c));
  X k{c, c->n, c->us, c->dot_fmt, {c->ex[EX_T0], c->ex[EX_T1]}};
  double* x = c->ex[EX_Z];
  double* r = c->ex[EX_R];
  double* p = c->ex[EX_P];
  double* hp = c->ex[EX_Q];
  const XOp H = make_op(c, 1);
  GADI_TRY(k.scale(r, r64, scale));  // gadi.py:153 r_s = q(scale r)
  GADI_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * (size_t)c->n, c->stream));
  double nrhs;
  GADI_TRY(k.norm(r, &nrhs));
  if (nrhs == 0.0) {
    set_stats(c->h_hst, 0, 0.0, true, false);
    return 0;
  }
  GADI_CUDA(cudaMemcpyAsync(p, r, sizeof(double) * (size_t)c->n, cudaMemcpyDeviceToDevice, c->stream));
  double rs;
  GADI_TRY(k.dot(r, r, &rs));
  double relres = 1.0;
  bool conv = false, brk = false;
  int it = 0;
  while (it < maxit) {
    GADI_TRY(k.spmv(H, p, hp));
    double php;
    GADI_TRY(k.dot(p, hp, &php));
    if (php <= 0.0) {
      brk = true;
      break;
    }
    const double alpha = qf(rs / php, c->us);
    GADI_TRY(k.axpy(x, x, alpha, p, 1.0));
    GADI_TRY(k.axpy(r, r, alpha, hp, -1.0));
    double rs_new;
    GADI_TRY(k.dot(r, r, &rs_new));
    ++it;
    relres = std::sqrt(std::max(rs_new, 0.0)) / nrhs;
    if (relres <= tol) {
      conv = true;
      break;
    }
    if (rs_new <= 0.0) break;
    const double beta = qf(rs_new / rs, c->us);
    GADI_TRY(k.axpy(p, r, beta, p, 1.0));
    rs = rs_new;
  }
  set_stats(c->h_hst, it, relres, conv, brk);
  return 0;
}

// cg_normal_skew(S_low, q(coeff z), tol, maxit, u_s, strict_model, S_low_T)
// (gadi.py:158, inner.py:92-143); the solution is left in ex[EX_Y].
int exact_s_solve(Ctx* c, const double* z, double coeff, double tol, int maxit) {
  GADI_TRY(exact_alloc(c));
  X k{c, c->n, c->us, c->dot_fmt, {c->ex[EX_T0], c->ex[EX_T1]}};
  double* y = c->ex[EX_Y];
  double* r = c->ex[EX_R];
  double* p = c->ex[EX_P];
  double* w = c->ex[EX_Q];
  double* rb = c->ex[EX_RB];
  const XOp S = make_op(c, 2), ST = make_op(c, 3);
  GADI_TRY(k.scale(r, z, coeff));
  GADI_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * (size_t)c->n, c->stream));
  double nrhs;
  GADI_TRY(k.norm(r, &nrhs));
  if (nrhs == 0.0) {
    set_stats(c->h_sst, 0, 0.0, true, false);
    return 0;
  }
  GADI_TRY(k.spmv(ST, r, rb));
  GADI_CUDA(cudaMemcpyAsync(p, rb, sizeof(double) * (size_t)c->n, cudaMemcpyDeviceToDevice, c->stream));
  double rs;
  GADI_TRY(k.dot(rb, rb, &rs));
  double relres = 1.0;
  bool conv = false, brk = false;
  int it = 0;
  while (it < maxit) {
    GADI_TRY(k.spmv(S, p, w));
    double denom;
    GADI_TRY(k.dot(w, w, &denom));
    if (denom <= 0.0) {
      brk = true;
      break;
    }
    const double alpha = qf(rs / denom, c->us);
    GADI_TRY(k.axpy(y, y, alpha, p, 1.0));
    GADI_TRY(k.axpy(r, r, alpha, w, -1.0));
    ++it;
    double nr;
    GADI_TRY(k.norm(r, &nr));
    relres = nr / nrhs;
    if (relres <= tol) {
      conv = true;
      break;
    }
    GADI_TRY(k.spmv(ST, r, rb));
    double rs_new;
    GADI_TRY(k.dot(rb, rb, &rs_new));
    if (rs_new <= 0.0) break;
    const double beta = qf(rs_new / rs, c->us);
    GADI_TRY(k.axpy(p, rb, beta, p, 1.0));
    rs = rs_new;
  }
  set_stats(c->h_sst, it, relres, conv, brk);
  return 0;
}

}  // namespace gadi
