/*
 * ciq.h -- C ABI of the B200-native msMINRES-CIQ library (libciq.so).
 *
 * Computes K^{1/2} B and K^{-1/2} B for a symmetric positive-definite kernel matrix K and a block
 * B of T right-hand sides with Contour Integral Quadrature + multi-shift MINRES (Pleiss et al.,
 * arXiv 2006.11267; "P:n" = line n of the paper text PAPER.md):
 *
 *     K^{-1/2} b ~ sum_q w_q (t_q I + K)^{-1} b,   K^{1/2} b ~ K sum_q w_q (t_q I + K)^{-1} b
 *                                                   (eq. contour_integral_quad)
 *
 * with the Hale-Higham-Trefethen shifts/weights (eq. quad_points_and_locations)
 * built from a Lanczos estimate of lambda_min/lambda_max, the shifted solves by
 * msMINRES (App. C), and the preconditioned rotated variants R b, R' b of App. A
 * (eqs. precond_sqrt / precond_sqrt_inverse).
 *
 * Conventions (apply to every entry point):
 *  - Matrices are row-major float32 with an explicit leading dimension (elements).  B and out are
 *    N x T ("column c is right-hand side b_c"), X is N x d, a dense K is N x N.
 *  - Pointers may be HOST or DEVICE memory (detected with cudaPointerGetAttributes).  Host inputs
 *    are copied to device workspace inside the call; host outputs are written back before the
 *    call returns.  Device inputs are read in place on the ctx stream.
 *  - Ownership: the caller owns every buffer it passes.  Operator / preconditioner arrays passed
 *    to ciq_init must stay valid until ciq_free if they are device pointers (host arrays are
 *    copied at init).  The ctx owns its workspace (grown lazily per T) and its NCCL communicator.
 *  - Stream ordering: device work runs on a private non-blocking stream of the ctx, ordered after
 *    everything already enqueued on the stream given to ciq_init (event join).  ciq_apply /
 *    ciq_matvec return after the result has been written (the lambda estimate and the
 *    convergence poll are host decisions), so the caller may use the output immediately.
 *  - Errors: status codes only, never exceptions across the ABI; ciq_last_error() gives text.
 *    A non-converged solve is NOT an error: the result is written and CIQ_NOT_CONVERGED returned
 *    (S:284).
 *  - Thread safety: one ctx per host thread; contexts are independent.
 *  - Determinism: every reduction is fixed-order (no float atomics); the same inputs on the same
 *    launch configuration give bitwise-identical outputs.
 */
#ifndef CIQ_H_
#define CIQ_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CIQ_MAX_Q 64

typedef enum {
  CIQ_OK = 0,
  CIQ_NOT_CONVERGED = 1,     /* result written, max_q,c |phibar|/||b_c|| > tol after max_iters, */
                             /* or a NaN / inf residual (also at tol = 0; info.max_rel_residual */
                             /* = inf, the solve stops at that iteration)                       */
  CIQ_ERR_INVALID_ARG = -1,  /* null pointer, Q out of [1, CIQ_MAX_Q], tol < 0, max_iters < 1, ... */
  CIQ_ERR_DIM = -2,          /* n <= 0, T <= 0, d < 1, leading dimension too small            */
  CIQ_ERR_NOT_PD = -3,       /* lambda_min estimate <= 0 (operator not positive definite)     */
  CIQ_ERR_ELLIPTIC = -4,     /* quadrature rule not finite (elliptic function failure)        */
  CIQ_ERR_CUDA = -5,         /* CUDA runtime / launch error, or no CUDA device                */
  CIQ_ERR_NCCL = -6,         /* NCCL could not be loaded or a collective failed               */
  CIQ_ERR_OOM = -7           /* device allocation failed                                     */
} ciq_status;

typedef enum {
  CIQ_OP_DENSE = 0,     /* K = A + diag*I for a given dense symmetric A                   */
  CIQ_OP_RBF = 1,       /* k = o^2 exp(-r^2/2)                                (reading G11)        */
  CIQ_OP_MATERN52 = 2,  /* k = o^2 (1 + sqrt5 r + 5 r^2/3) exp(-sqrt5 r)                           */
  CIQ_OP_MATERN32 = 3,  /* k = o^2 (1 + sqrt3 r) exp(-sqrt3 r);  r = ||(x - x')/l||, K += diag*I   */
  CIQ_OP_SPARSE = 4     /* a given sparse symmetric matrix in CSR form (e.g. the stencil precision */
                        /* Lambda = g_obs A^T A + g_prior L^T L of the Gibbs sampler),  */
                        /* K = A + diag*I; fp32 SIMT SpMM                    */
} ciq_op_kind;

typedef enum {
  CIQ_MODE_SQRT = 0,     /* K^{1/2} B (R B with a preconditioner)       -- one extra MVM */
  CIQ_MODE_INVSQRT = 1,  /* K^{-1/2} B (R' B with a preconditioner)                               */
  CIQ_MODE_WHITEN = 2    /* same as INVSQRT (reading G9)                                          */
} ciq_mode;

typedef enum {
  CIQ_MVM_AUTO = 0,      /* tensor-core path where implemented, else SIMT fp32                  */
  CIQ_MVM_SIMT = 1,      /* fp32 CUDA-core tiles (reference kernel)                             */
  CIQ_MVM_TC = 2,        /* tcgen05 split-fp16 tensor-core kernel, full tiles (fails if unavailable) */
  CIQ_MVM_TC_SYM = 3,    /* tcgen05 symmetric-tile kernel: each k(x_i, x_j), i < j, evaluated once
                            and applied to both rows (single GPU, RBF / Matern, d <= 8, RHS chunk of
                            16 or 32 columns; fails if unavailable).  CIQ_MVM_AUTO picks it where
                            DESIGN.md section 8 measures it faster (RHS chunk of 16)              */
  CIQ_MVM_FP64_TC = 4    /* reported only (ciq_info.mvm_impl_used): the fp64 route's materialised-M
                            MVM on the FP64 tensor pipe (DMMA; params.fp64 / preconditioned)      */
} ciq_mvm_impl;

/* The operator K (touched only through MVMs, P:397 / P:1161-1162). */
typedef struct {
  int32_t kind;               /* ciq_op_kind                                                    */
  int64_t n;                  /* global N                                                       */
  const float* K;             /* DENSE: N x N row-major, leading dimension ldk (>= N)            */
  int64_t ldk;
  const float* X;             /* kernels: N x d points, leading dimension ldx (>= d), replicated */
  int64_t d;                  /*          on every rank                                         */
  int64_t ldx;
  const float* lengthscale;   /* host pointer: d values if ard != 0, else 1 value (> 0)         */
  int32_t ard;
  float outputscale;          /* o^2 (> 0)                                                      */
  float diag;                 /* sigma^2 >= 0 added to the diagonal (noise / jitter, G12); also  */
                              /* the rigorous lower bound on lambda_min used by the estimator (G6) */
  const int64_t* csr_indptr;  /* SPARSE: this rank's row block (all N rows on one GPU) in CSR:   */
  const int32_t* csr_indices; /*   indptr[rows + 1] (indptr[0] = 0), global column indices and    */
  const float* csr_values;    /*   values of the nnz = indptr[rows] entries (host or device; the */
  int64_t nnz;                /*   ctx keeps a device copy).  The matrix must be symmetric.       */
} ciq_operator;

/* Preconditioner P = L L^T + sigma2 I, L = N x rank row-major (ld >= rank; with row
 * sharding: this rank's row block of L, like B -- the matrix-free route then all-reduces the
 * rank x T products L^T W / U^T W per application).  When L comes
 * from a partial pivoted Cholesky of the kernel part of K and sigma2 = op.diag, lambda_min of
 * P^{-1/2} K P^{-1/2} is >= 1 (reading G6) and the estimator uses that bound. */
typedef struct {
  const float* L;
  int64_t rank;
  int64_t ldl;
  float sigma2;               /* > 0                                                    */
  int32_t matrix_free;        /* 0 (default): the fp64 route -- M = P^{-1/2} K P^{-1/2} is formed */
                              /*   once in fp64 (N^2 doubles) and the solve runs on fp64 vectors  */
                              /*   (precond64.cu; needed for 1e-4 parity of R'B at kappa(K)~1e6,  */
                              /*   DESIGN.md section 5); used whenever M fits in device memory.   */
                              /* 1: apply M matrix-free per iteration (K MVM + two Woodbury       */
                              /*   P^{-1/2} applications, fp32 vectors): O(N) memory, accuracy    */
                              /*   limited by the fp32 sensitivity of R'B.  */
  int32_t kind;               /* 0 (default): P = L L^T + sigma2 I as above.                     */
                              /* 1: block-Jacobi P = blockdiag of (K + diag I)'s own diagonal     */
                              /*   blocks of size `block` (L, rank, sigma2, matrix_free ignored): */
                              /*   a P without a closed-form square root -- P^{1/2} B is computed */
                              /*   by CIQ on P ("nested CIQ") and the solve uses the P^{-1}- */
                              /*   only recurrence on x_q = (K + t_q P)^{-1} c; */
                              /*   fp64 throughout (K materialised: N^2 doubles), single GPU.     */
  int64_t block;              /* kind 1: block size (>= 1; the last block is ragged)             */
} ciq_precond;

/* Row sharding across GPUs (one process per GPU).  NULL comm = single GPU; a comm
 * with world = 1 runs the sharded code path (collectives included) on one rank.  Rank r
 * owns rows ciq_shard_rows(n, r, world); per iteration the ranks all-gather the next Lanczos
 * block and the T-sized alpha / beta^2 partial sums (summed in rank order: bit-identical scalar
 * state on every rank). */
typedef struct {
  int32_t rank;
  int32_t world;
  const void* nccl_unique_id; /* 128 bytes from ciq_nccl_unique_id() on rank 0, broadcast by the
                                 caller (e.g. torch.distributed)                                */
  void* loopback_group;       /* non-NULL: in-process loopback transport instead of NCCL (ranks are
                                 threads sharing one GPU; from ciq_loopback_group_create)      */
} ciq_comm;

typedef struct {
  int32_t Q;                  /* quadrature points, 1..CIQ_MAX_Q (default 8)             */
  int32_t max_iters;          /* J_max >= 1 (default 400)                                 */
  double tol;                 /* stop when max_{q,c} |phibar|/||b_c|| <= tol (G3); 0 = exactly   */
                              /* max_iters iterations (fixed J).  Default 1e-4          */
  int32_t lanczos_iters;      /* lambda-estimation Lanczos steps (default 10)            */
  int32_t lanczos_cols;       /* start columns pooled by the estimator (default 16, G5)          */
  double lambda_min;          /* > 0 together with lambda_max > 0: skip the estimation           */
  double lambda_max;
  const double* t;            /* optional explicit rule (host, Q values each): skips estimation  */
  const double* w;            /*   and the HHT construction (parity tests)                      */
  const float* lanczos_start; /* optional start block (host or device), lanczos_cols columns:   */
                              /*   THIS RANK's rows [row_begin, row_end) of the N x lanczos_cols */
                              /*   block, like B (all N rows on one GPU); NULL = counter-based   */
  int64_t ld_start;           /*   N(0,1) draw from `seed` (same on every rank count)            */
  uint64_t seed;
  int32_t mode;               /* ciq_mode                                                       */
  int32_t mvm_impl;           /* ciq_mvm_impl                                                   */
  int32_t poll_every;         /* iterations per captured CUDA graph / convergence poll (def. 6)  */
  double breakdown_tol;       /* Lanczos invariant-subspace threshold, relative (default 1e-6)   */
  int32_t profile_kernels;    /* 1: bracket every MVM / update launch with CUDA events and report */
                              /*    their device time in ciq_info (small overhead; default 0)     */
  int32_t lanczos_reuse;      /* 1: estimate lambda_min / lambda_max from the first 12 Lanczos     */
                              /*    steps of the solve itself (Lanczos started at b, as App. D     */
                              /*    P:1494 describes it), then replay the shifted updates of those */
                              /*    steps: no separate ~10-MVM estimation run.  Ignored with a     */
                              /*    preconditioner, an explicit rule/spectrum, or max_iters <= 24. */
                              /*    Default 0 (separate estimation from lanczos_start, G5).       */
  int32_t keep_shift_solutions; /* 1: also return the Q shifted solves x_q = (t_q I + K)^{-1} b   */
  float* shift_solutions;     /*    (the forward solves the backward pass reuses) into     */
                              /*    shift_solutions, Q x rows x T floats (row-major per shift,     */
                              /*    ld = T; host or device).  Not with a preconditioner.           */
  int32_t fp64;               /* 1: accuracy mode for kernel operators without a preconditioner: */
                              /*    K + sigma^2 I is materialised in fp64 (N^2 doubles; OOM error  */
                              /*    if it does not fit), MVMs on the FP64 pipe, fp64 Lanczos /     */
                              /*    msMINRES vectors (the preconditioned fp64 route, precond64.cu, */
                              /*    with P = I).  ~30x slower than the tensor-core path; removes   */
                              /*    the fp32 floor kappa(K) * ~1e-7 of the default. */
                              /*    lanczos_reuse / keep_shift_solutions are ignored.  Default 0.  */
  int32_t stored_basis;       /* 1: keep the Lanczos basis W_1..W_J (O(J N T) memory, falls back  */
                              /*    to the streaming recurrence if it does not fit) and form        */
                              /*    Y = W_J z once at the end: ~5 vectors of HBM      */
                              /*    traffic per iteration instead of 3Q + 6.  Not  */
                              /*    with a preconditioner or keep_shift_solutions.  Default 0.     */
  int32_t mvm_relax;          /* 1: relaxed inexact Krylov (Simoncini & Szyld): the MVM error may  */
                              /*    grow as 1 / ||r_j|| without moving the result, so once the max */
                              /*    relative residual is <= 0.1 the full-tile tensor-core MVM runs */
                              /*    with 4x longer TMEM accumulation chains (fewer column splits), */
                              /*    and from 0.01 with kernel entries rounded to fp16 (dense K: the */
                              /*    K_hi planes only).  DESIGN.md section 5; ciq_info.relaxed_from / */
                              /*    relaxed2_from report the switch steps.  Single GPU, no          */
                              /*    preconditioner.  Default 1; 0 = every MVM accurate.            */
} ciq_params;

typedef struct {
  int32_t iters;              /* J: msMINRES iterations applied                                 */
  int32_t mvms;               /* MVMs with K: lambda-estimation + J (+1 in SQRT mode)           */
  int32_t converged;
  int32_t rotated;            /* 1 if a preconditioner was used (result is R B / R' B)           */
  int32_t breakdown_cols;     /* columns frozen on an invariant subspace                        */
  int32_t Q;
  double lambda_min, lambda_max;  /* used for the rule (after safety margins)                   */
  double ritz_min, ritz_max;      /* raw Ritz extremes (NaN if estimation skipped)              */
  double max_rel_residual;        /* max_{q,c} |phibar|/||b_c|| at exit                         */
  double t[CIQ_MAX_Q], w[CIQ_MAX_Q];
  float ms_total, ms_lambda, ms_loop, ms_final;
  int64_t kernel_launches;    /* kernels launched by this call (graph nodes counted per launch) */
  float ms_mvm;               /* profile_kernels: summed device time of the msMINRES-loop MVMs   */
  int32_t mvm_timed;          /*   number of loop MVMs timed (= iters)                          */
  float ms_update;            /* profile_kernels: summed device time of the streaming updates    */
  int32_t update_timed;
  int32_t mvm_impl_used;      /* ciq_mvm_impl of the loop MVMs: SIMT, TC, TC_SYM or FP64_TC      */
  int32_t mvm_splits;         /* column splits of the tensor-core MVM grid (1 = none)            */
  int32_t fp64_route;         /* 1: solve on fp64 vectors (precond64.cu / params.fp64 / nested)   */
  int32_t nested_p_mvms;      /* nested CIQ (block-Jacobi P): MVMs with P spent on P^{1/2} b     */
  int32_t nested_iters;       /*   and the inner msMINRES iterations                             */
  int32_t overlap;            /* row-sharded: 1 if the Lanczos-block all-gather ran next to the
                                 local diagonal block's MVM */
  int32_t relaxed_from;       /* params.mvm_relax: first msMINRES step run with the relaxed MVM  */
                              /*   (longer accumulation chains); 0 if none                      */
  int32_t relaxed2_from;      /*   ... and with kernel entries rounded to fp16 (second level)      */
} ciq_info;

typedef struct ciq_ctx ciq_ctx;

/* Fill *p with the defaults listed above. */
void ciq_params_default(ciq_params* p);

/* Create a context for operator `op` (and optional preconditioner `pc`, optional row-sharding
 * `comm`) on CUDA stream `stream` (a cudaStream_t; NULL = the legacy default stream).  Validates
 * the operator, allocates the operator workspace, prepares the scaled points / dense K copy. */
ciq_status ciq_init(ciq_ctx** ctx, const ciq_operator* op, const ciq_precond* pc,
                    const ciq_comm* comm, void* stream);

/* out (N x T, ldo) <- K^{1/2} B or K^{-1/2} B (R B / R' B with a preconditioner) for B (N x T,
 * ldb).  With row sharding, B and out hold this rank's row block [row_begin, row_end) (see
 * ciq_shard_rows).  `info` may be NULL. */
ciq_status ciq_apply(ciq_ctx* ctx, const float* B, int64_t ldb, int64_t T, float* out, int64_t ldo,
                     const ciq_params* p, ciq_info* info);

/* One application of the operator: out <- K V (+ diag*V), the MVM of P:1155-1161 as used by the
 * solver (same kernel, same precision path selected by mvm_impl).  V: N x T (full); out: this
 * rank's rows. */
ciq_status ciq_matvec(ciq_ctx* ctx, const float* V, int64_t ldv, int64_t T, float* out, int64_t ldo,
                      int32_t mvm_impl);

/* Partial pivoted Cholesky of the kernel part of K (Harbrecht et al.): rank
 * greedy steps, each picking the largest remaining diagonal residual (lowest index on ties),
 * appending the normalised residual column.  L (N x rank, ldl >= rank, host or device) receives
 * the factor; use it as ciq_precond.L with sigma2 = op.diag for the App. A preconditioner. */
ciq_status ciq_pivoted_cholesky(ciq_ctx* ctx, int32_t rank, float* L, int64_t ldl);

/* Backward pass of K^{-1/2} B (App. B "Efficient Vector-Jacobi Products for Backpropagation",
 * eq. ciq_deriv): with the back-propagated gradient V (rows x T, same layout as B),
 *     G = sum_c -1/2 sum_q w_q ( x_q(v_c) x_q(b_c)^T + x_q(b_c) x_q(v_c)^T ),
 *     x_q(u) = (t_q I + K)^{-1} u,
 * i.e. dL/dK for L(K^{-1/2} B) with dL/d(K^{-1/2} B) = V.  Two msMINRES solves (b with the
 * estimated or given rule, then v with the SAME rule), then the rank-2QT product on the GPU.
 * G: N x N floats (ld = ldg >= N, host or device).  params->mode is ignored (the derivative is of
 * K^{-1/2} b); keep_shift_solutions / shift_solutions are ignored.  Single GPU, no preconditioner
 * (CIQ_ERR_INVALID_ARG otherwise).  info (nullable): the forward solve's info, mvms = both solves. */
ciq_status ciq_vjp(ciq_ctx* ctx, const float* B, int64_t ldb, const float* V, int64_t ldv, int64_t T,
                   const ciq_params* params, float* G, int64_t ldg, ciq_info* info);

/* Hyper-parameter gradient through the CIQ backward pass (eq. ciq_deriv; SURVEY
 * §8(f) row f1): for L = sum_c v_c^T (K^{-1/2} b_c) with K = o^2 k(X, X; l) + sigma^2 I,
 *     grad[0] = dL/dl,  grad[1] = dL/d(o^2),  grad[2] = dL/d(sigma^2)
 * as  dL/dtheta = sum_ij G_ij dK_ij/dtheta = -sum_q w_q sum_c x_q(v_c)^T (dK/dtheta) x_q(b_c)
 * with the shifted solves x_q(u) = (t_q I + K)^{-1} u of the forward solve and of a second solve on
 * V with the same rule (G is never formed: O(J mvm(K)) time, O(Q N T) memory).  The
 * bilinear forms use one matrix-free dK/dl MVM (tensor-core epilogue with the derivative of the
 * kernel form) and one K MVM per shift, fp64 reductions.
 *   B, V: N x T (ld >= T, host or device).  grad: 3 doubles (host).
 * Single GPU, kernel operators with an isotropic lengthscale, no preconditioner / posterior:
 * CIQ_ERR_INVALID_ARG otherwise.  info (nullable): the forward solve's info, mvms = all MVMs. */
ciq_status ciq_hyper_grad(ciq_ctx* ctx, const float* B, int64_t ldb, const float* V, int64_t ldv, int64_t T,
                          const ciq_params* params, double* grad, ciq_info* info);

/* Thompson sampling (SS5.2, eq. thompson_sample).
 * ciq_set_posterior turns a matrix-free kernel context built on the candidate set X* (ciq_init
 * with op.X = X*, op.diag = the jitter) into the GP posterior covariance operator at X*,
 *     COV* + jitter I = K** + jitter I - K*x (Kxx + noise I)^{-1} Kx*,
 * with posterior mean mu* = K*x (Kxx + noise I)^{-1} y ("posterior mean and covariance of the
 * Gaussian process at the candidate set").  Every later ciq_apply / ciq_matvec /
 * ciq_thompson on ctx uses this operator (lambda_min lower bound: the jitter, COV* being PSD).
 *   Xt: m x d training inputs (row-major, ldxt >= d, host or device; same kernel and
 *       lengthscale as the ctx), y: m training targets (host or device; NULL = zero mean),
 *   noise > 0: the training-data noise.  1 <= m <= 4096.
 * The training block is factorised once on the host in fp64 (Cholesky of Kxx + noise I and L^{-1});
 * U = K*x L^{-T} (N x m, fp64) and mu* are built on the device.  Call again to replace the data.
 * With a preconditioner (ciq_init's pc, sigma2 = the jitter) the solve runs on
 * P^{-1/2} (COV* + jitter I) P^{-1/2} (App. A); ciq_pivoted_cholesky on a posterior ctx factors
 * COV* (the Hartmann-posterior preconditioning of P:914-915).
 * Single GPU, kernel operators: CIQ_ERR_INVALID_ARG otherwise;
 * CIQ_ERR_NOT_PD if Kxx + noise I is not positive definite in fp64. */
ciq_status ciq_set_posterior(ciq_ctx* ctx, const float* Xt, int64_t ldxt, int64_t m, const float* y, double noise);

/* One Thompson-sampling step (eq. thompson_sample): for each column c of eps (N x T, ld =
 * ld_eps >= T, host or device; each column one standard-normal draw)
 *     f_c = mu* + COV*^{1/2} eps_c  (msMINRES-CIQ, sqrt mode; params->mode ignored),
 *     idx[c] = argmin_j f_c[j]  (lowest j among equal minima; int64, host or device).
 * samples (nullable): receives f (N x T, ld = ld_samples >= T, host or device).
 * Requires ciq_set_posterior first (CIQ_ERR_INVALID_ARG otherwise).  info as for ciq_apply. */
ciq_status ciq_thompson(ciq_ctx* ctx, const float* eps, int64_t ld_eps, int64_t T, const ciq_params* params,
                        int64_t* idx, float* samples, int64_t ld_samples, ciq_info* info);

void ciq_free(ciq_ctx* ctx);

const char* ciq_status_string(ciq_status s);
/* sha256 prefix (16 hex digits) of the sources this library was compiled from (build.py
 * source_hash()); lets a caller check the binary matches the committed sources. */
const char* ciq_source_hash(void);
const char* ciq_last_error(const ciq_ctx* ctx);   /* NULL ctx: last error of ciq_init on this thread */

/* Row block [*row_begin, *row_end) owned by `rank` of `world` for a global N (multiples of 128). */
void ciq_shard_rows(int64_t n, int32_t rank, int32_t world, int64_t* row_begin, int64_t* row_end);

/* Host-only helpers (no GPU needed) -- the host steps a2/a3 of the hot path, exported for tests.
 * ciq_quadrature_rule: the HHT rule t_q, w_q from lambda_min < lambda_max, in
 *   real arithmetic via the Jacobi imaginary transform (G10); returns CIQ_ERR_INVALID_ARG /
 *   CIQ_ERR_ELLIPTIC on bad input / non-finite output.
 * ciq_tridiag_extremes: smallest and largest eigenvalue of the symmetric tridiagonal matrix with
 *   diagonal alpha[0..m-1] and off-diagonal beta[0..m-2] (fp64 Sturm bisection).
 * ciq_nccl_unique_id: 128-byte ncclUniqueId (loads NCCL; CIQ_ERR_NCCL if unavailable). */
ciq_status ciq_quadrature_rule(double lambda_min, double lambda_max, int32_t Q, double* t, double* w);
ciq_status ciq_tridiag_extremes(const double* alpha, const double* beta, int32_t m,
                                double* eig_min, double* eig_max);
ciq_status ciq_nccl_unique_id(void* out128);

/* In-process loopback transport for `world` ranks (threads of one process, any device): used to
 * exercise the row-sharded path without NCCL.  Destroy after every ctx using it is freed. */
void* ciq_loopback_group_create(int32_t world);
void ciq_loopback_group_destroy(void* group);

#ifdef __cplusplus
}
#endif
#endif /* CIQ_H_ */
