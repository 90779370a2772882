/*
 * gadi_b200 — C ABI of the B200-native mixed-precision GADI hot path.
 *
 * The reference (gadimp 0.1.0, arXiv 2512.21164) is a pure-Python package;
 * its hot path is the Python call
 *     gadimp.gadi.gadi_solve(problem, splitting, cfg, keep_iterates)
 *         (/root/reference/pkg/src/gadimp/gadi.py:115-209)
 * and the functions it calls per outer step:
 *     sparsemat.residual  (sparsemat.py:219-234)  -> gadi_outer_step (fused)
 *     inner.cg_spd        (inner.py:47-89)        -> gadi_outer_step / gadi_h_solve
 *     inner.cg_normal_skew(inner.py:92-143)       -> gadi_outer_step / gadi_s_solve
 *     analysis.matrix_norm_2 (analysis.py:51-70)  -> gadi_norm2
 *     sparsemat.spmv      (sparsemat.py:178-199)  -> gadi_spmv
 * There is no reference FFI; this header is the boundary a gadimp
 * maintainer binds with ctypes.
 *
 * Conventions: plain C types only; every function returns 0 on success or a
 * GADI_ERR_* code (message via gadi_last_error()).  Host pointers are
 * borrowed for the duration of the call.  A context owns all of its device
 * memory and one CUDA stream; it is not thread-safe (one context per solve,
 * as SPEC.md:369 "one solve = one isolated context").  Vectors cross the ABI
 * in the reference's layout (lexicographic grid order; the complex
 * reaction-diffusion family in block form [re; im], problems.py:116).
 */
#ifndef GADI_B200_H
#define GADI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GADI_OK 0
#define GADI_ERR_CUDA 1
#define GADI_ERR_ARG 2
#define GADI_ERR_OOM 3
#define GADI_ERR_UNSUPPORTED 4

/* precision formats, precision.py:80-88 */
enum gadi_fmt { GADI_BF16 = 0, GADI_FP16 = 1, GADI_FP32 = 2, GADI_FP64 = 3, GADI_FP64X2 = 4 };

/* operator families */
enum gadi_kind {
  GADI_STENCIL = 0, /* real constant-coefficient 5-point (2-D) / 7-point (3-D) */
  GADI_COMPLEX = 1, /* crd: A = [[L, -V], [V, L]], L 2-D 5-point (problems.py:96-120) */
  GADI_CSR = 2      /* general sparse matrices (sparsemat.SparseMatrix) */
};

/* constant stencil: axis 0 = slowest (x), 2 = fastest (z); lo multiplies the
 * neighbour with the smaller linear index.  Appendix A of SURVEY.md. */
typedef struct {
  double d;
  double lo[3];
  double up[3];
} gadi_coef;

/* CSR matrix in the reference's SparseMatrix layout (sparsemat.py:35-60). */
typedef struct {
  int64_t nrows;
  int64_t nnz;
  const int64_t* row_offsets; /* nrows + 1 */
  const int64_t* col_indices; /* nnz, ascending within each row */
  const double* values;       /* nnz */
} gadi_csr;

typedef struct {
  int kind;        /* enum gadi_kind */
  int ndim;        /* 2 or 3 (stencil kinds) */
  int64_t dims[3]; /* grid extents (x, y, z); 2-D uses (n_g, 1, n_g) */
  int64_t n;       /* number of real unknowns */
  gadi_coef A;     /* fp64 coefficients of A (crd: of L) */
  gadi_coef H;     /* u_s images of H = alpha I + M (crd: alpha I + L) */
  gadi_coef S;     /* u_s images of S = alpha I + N (real stencils) */
  double alpha_s;  /* u_s image of alpha (crd S diagonal) */
  const double* v; /* crd potential V diagonal, n/2 values (fp64) */
  gadi_csr csr_A, csr_H, csr_S, csr_ST; /* kind == GADI_CSR */
  int u, u_r, u_s; /* enum gadi_fmt */
} gadi_problem_desc;

typedef struct gadi_ctx gadi_ctx;
typedef struct gadi_comm gadi_comm;

/* per outer step scalars (gadi.py:166-176 inputs) */
typedef struct {
  double sum_r2;     /* ||b - A x||^2, fp64 monitor residual */
  double max_r;      /* max |r_alg| (u_r residual; drives the power-of-two scale) */
  double sum_ralg2;  /* ||r_alg||^2 (IterationRecord.residual_norm of the next step) */
  double sum_x2;     /* ||x||^2 */
  double sum_e2;     /* ||x* - x||^2 (0 when no exact solution) */
  double sum_ae2;    /* ||A (x* - x)||^2 */
} gadi_outer_scalars;

/* inner solve outcome, inner.py:30-36 InnerSolveStats */
typedef struct {
  int iterations;
  int converged;
  int breakdown;
  int pad;
  double final_relative_residual;
} gadi_inner_stats;

/* device time of the phases of one outer step (ms), gadi.py:142-183 timers */
typedef struct {
  double residual, inner_h, inner_s, update, monitor;
} gadi_phase_times;

typedef struct {
  double scale;       /* 2^-ceil(log2 max|r|), gadi.py:151-152 */
  double coeff;       /* RNE_{u_s}((2 - omega) alpha), gadi.py:135 */
  double inner_tol;
  int maxit_h, maxit_s;
  int use_graph;      /* replay the step as a CUDA graph when possible */
} gadi_step_args;

const char* gadi_last_error(void);
int gadi_device_count(int* count);
/* library build identification (kernels compiled for sm_100a) */
const char* gadi_build_info(void);

int gadi_ctx_create(const gadi_problem_desc* desc, int device, gadi_ctx** out);
int gadi_ctx_destroy(gadi_ctx* ctx);

/* ---- slab decomposition across ranks (one process per GPU).
 * The slowest grid axis (x planes; rows for 2-D and crd) is split into
 * contiguous slabs.  A slab context owns global planes [x0, x1) of the
 * problem described by `desc` (global dims; crd: desc->v is the whole
 * potential) and exchanges one halo plane with each neighbour before every
 * stencil pass; every Krylov / monitor reduction gathers the per-rank sums
 * and reduces them in rank order on the device, so all ranks take identical
 * decisions.  Vectors crossing the ABI of a slab context are the slab's rows.
 * There is no reference counterpart (the reference is single-process). */
/* NCCL: rank 0 creates the id, the caller broadcasts it (torch.distributed). */
int gadi_comm_nccl_unique_id(unsigned char* id128);
int gadi_comm_create_nccl(const unsigned char* id128, int nranks, int rank, int device, gadi_comm** out);
/* In-process group of `nranks` slabs on one device, one host thread per rank
 * (single-GPU test harness of the decomposition); `key` names the group. */
int gadi_comm_create_local(int key, int nranks, int rank, gadi_comm** out);
/* As above; peer = 1: slab contexts built on it switch to the device-signalled
 * peer transport (the same kernels as one process per GPU; see below). */
int gadi_comm_create_local2(int key, int nranks, int rank, int peer, gadi_comm** out);
int gadi_comm_destroy(gadi_comm* comm);
/* Peer transport (csrc/peer.cu).  A slab context whose communicator asks for
 * it (NCCL: unless GADI_COMM=nccl; local2: peer = 1) maps its neighbours'
 * halo'd vectors, gather rows and epoch flags at creation (CUDA IPC handles
 * exchanged over the base communicator; plain pointers within one process)
 * and runs every halo exchange / scalar all-gather as kernels that write the
 * peers' memory and synchronise on system-scope release/acquire flags -- no
 * host in the loop, so the inner solves run as CUDA-graph WHILE loops.  If
 * any rank cannot map its peers, every rank keeps the base transport.
 * gadi_ctx_comm_kind reports the context's transport ("peer", "nccl", "local"). */
const char* gadi_ctx_comm_kind(gadi_ctx* ctx);
/* The same transport with the blob exchange done by the caller (one process
 * per GPU with any host collective, e.g. torch.distributed over gloo): a
 * transport-less communicator, then per slab context export this rank's blob
 * (CUDA IPC handles + layout), gather every rank's blob in rank order and
 * attach.  blob_len = the length gadi_ctx_peer_export reports. */
int gadi_comm_create_host(int nranks, int rank, gadi_comm** out);
int gadi_ctx_peer_export(gadi_ctx* ctx, void* blob, size_t cap, size_t* len);
int gadi_ctx_peer_attach(gadi_ctx* ctx, const void* blobs, size_t blob_len);
int gadi_comm_info(gadi_comm* comm, int* rank, int* nranks);
int gadi_ctx_create_slab(const gadi_problem_desc* desc, int device, gadi_comm* comm, int64_t x0, int64_t x1,
                         gadi_ctx** out);
int gadi_ctx_slab(gadi_ctx* ctx, int64_t* x0, int64_t* x1, int64_t* n_local);

/* b (block layout, n values) -> device */
int gadi_set_rhs(gadi_ctx* ctx, const double* b);
/* b = A 1 generated on the device (problems.py:42-45) */
int gadi_gen_rhs_ones(gadi_ctx* ctx);
/* b device -> host */
int gadi_get_rhs(gadi_ctx* ctx, double* b);
/* exact solution: xs == NULL with all_ones = 1 means x* = 1; xs == NULL and
 * all_ones = 0 means "no exact solution" (ferr, mu are None). */
int gadi_set_exact(gadi_ctx* ctx, const double* xs, int all_ones);

/* ||A||_2 by power iteration on A^T A (analysis.py:51-70).  v0: host start
 * vector already normalised (NULL: device generator with `seed`). */
int gadi_norm2(gadi_ctx* ctx, const double* v0, uint64_t seed, double tol, int maxit, double* sigma,
               int* iterations);

/* x = 0, r = b - A 0: fills the scalars of the initial residual */
int gadi_outer_begin(gadi_ctx* ctx, gadi_outer_scalars* out);
/* One outer step (gadi.py:147-176): H-solve (CG) of the scaled, cast
 * residual; rhs2 = coeff z; S-solve (CGNR); x += y/scale; new residual and
 * monitor sums.  The residual of step k+1 is produced by step k. */
int gadi_outer_step(gadi_ctx* ctx, const gadi_step_args* args, gadi_outer_scalars* out, gadi_inner_stats* h,
                    gadi_inner_stats* s, gadi_phase_times* t);
/* x device -> host (block layout) */
int gadi_get_x(gadi_ctx* ctx, double* x);

/* Standalone inner solvers on the context's operators, x0 = 0.
 * rhs and x are u_s images in fp64 (n values, block layout). */
int gadi_h_solve(gadi_ctx* ctx, const double* rhs, double tol, int maxit, double* x, gadi_inner_stats* st);
int gadi_s_solve(gadi_ctx* ctx, const double* rhs, double tol, int maxit, double* x, gadi_inner_stats* st);

/* Inner-solver arithmetic.  mode 0 (default): the storage model -- u_s
 * storage, fp32 arithmetic, fp64 dot accumulation (the paper's cublas*Ex
 * design).  mode 1: the reference's round-after-every-op
 * emulation (precision.py:136-220, inner.py:47-143) with dot products summed
 * by the pairwise tree in `dot_fmt` (inner.py:39-44 _dot_format: u_s when
 * strict_model, fp32 otherwise): iterates bitwise the reference's.  Mode 1 is
 * a parity mode (one host synchronisation per reduction). */
int gadi_set_rounding(gadi_ctx* ctx, int mode, int dot_fmt);

/* y = Op x with Op in {0: A (fp64, ordered), 1: H, 2: S, 3: S^T (u_s storage)}.
 * strict = 1 rounds every product and partial sum to u_s in ascending column
 * order (bitwise sparsemat.spmv on the u_s copies, sparsemat.py:188-199);
 * strict = 0 is the solver's storage model (compute-type accumulation). */
int gadi_spmv(gadi_ctx* ctx, int op, int strict, const double* x, double* y);

/* r = fl(b - A x) in the context's u_r (fp64 / fp32 emulated / fp64x2
 * compensated) with the rhs set by gadi_set_rhs; sparsemat.residual
 * (sparsemat.py:219-234).  Clobbers the solver iterate. */
int gadi_residual(gadi_ctx* ctx, const double* x, double* r);

/* Live per-kernel device timers (CUDA events on the context stream around
 * every launch while enabled).  kid: 0 H-CG init, 1 H-CG pass A, 2 H-CG
 * pass B, 3 CGNR init, 4-6 CGNR passes 1-3, 7-9 crd CGNR init/P1/P2,
 * 10 outer pass, 11-12 ||A||_2 passes, 13 operator apply.  Enabling resets. */
int gadi_prof_enable(gadi_ctx* ctx, int on);
int gadi_prof_read(gadi_ctx* ctx, int kid, double* total_ms, int64_t* launches);
/* device time between two points on the context stream */
int gadi_timer_start(gadi_ctx* ctx);
int gadi_timer_stop(gadi_ctx* ctx, double* ms);

/* elapsed device ms of the last gadi_norm2 call */
double gadi_last_norm_ms(gadi_ctx* ctx);
/* number of device kernels this context has launched */
int64_t gadi_kernel_launches(gadi_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
