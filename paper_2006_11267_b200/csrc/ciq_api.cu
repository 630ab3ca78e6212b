// ciq_api.cu -- the C ABI (include/ciq.h) and the host orchestration of one msMINRES-CIQ call
// (SURVEY §3.2): RHS normalisation -> lambda estimation (Lanczos, fp64 Sturm bisection on the
// host) -> host HHT rule -> J iterations of [MVM, alpha, streaming update, Givens] with a device
// convergence flag polled every `poll_every` iterations -> last pending update -> (SQRT) one more
// MVM -> output.  Every step of the path runs in this library's kernels.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <functional>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ciq.h"
#include "host_math.h"
#include "internal.h"
#include "comm.h"
#include "nccl_dl.h"

using namespace ciq;

namespace {

thread_local std::string g_init_error;

struct Workspace {
  int tp = 0, nq = 0;
  int esz = 4;             // bytes per element of W / P / D / Y: 4 (fp32) or 8 (fp64 route)
  int64_t rows = 0;
  float* w[3] = {nullptr, nullptr, nullptr};
  float* p = nullptr;
  float* d = nullptr;      // [2 slots][nq][rows][tp]
  float* y = nullptr;
  float* xq = nullptr;     // [nq][rows][tp] kept per-shift solutions (keep_shift_solutions)
  size_t xq_elems = 0;
  double* apart = nullptr; // [mvm blocks][tp]
  double* bpart = nullptr; // [stream blocks][tp]
  double* colsq = nullptr; // [tp]
  char* scal_mem = nullptr;
  Scal sc{};
};

struct LambdaWork {
  int tpl = 0, nb = 0;
  int64_t rows = 0;
  float* basis = nullptr;  // [nb][rows][tpl]
  float* p = nullptr;
  double* part = nullptr;
  double* h1 = nullptr;
  double* h2 = nullptr;
  double* bsq = nullptr;
  double* alphas = nullptr;
  double* betas = nullptr;
  double* inv = nullptr;
  int* len = nullptr;
};

}  // namespace

// Low-rank-plus-diagonal preconditioner on the device (precond.cu): U (n x r2, orthonormal),
// per-power gains g_p = (s^2 + sigma2)^p - sigma2^p and scalars a_p = sigma2^p for p = -1, 1/2, -1/2.
struct PrecondDev {
  bool on = false;
  int rank = 0, r2 = 0;
  double sigma2 = 0.0;
  float* l = nullptr;       // n x rank (owned copy)
  double* u = nullptr;      // n x r2 (fp64: see precond.cu)
  double* g[3] = {nullptr, nullptr, nullptr};
  float a[3] = {0.f, 0.f, 0.f};
  double ad[3] = {0.0, 0.0, 0.0};   // the same scalars in fp64 (fp64 route)
  // fp64 route (precond64.cu): M = P^{-1/2} K P^{-1/2} materialised in fp64, rows x ldm
  bool matrix_free = false;         // ciq_precond.matrix_free: never materialise
  bool m64_ready = false, m64_failed = false;
  double* m64 = nullptr;
  int64_t ldm = 0;
  // work
  double* part = nullptr;   size_t part_cap = 0;   // utv partials  [splits][r2][tp]
  double* h = nullptr;      size_t h_cap = 0;      // U^T v         [r2][tp]
  double* bpart = nullptr;  size_t bpart_cap = 0;  // dot partials  [blocks][tp]
  float* t1 = nullptr; size_t t_cap = 0;  // [2][n][tp] scratch of M v = P^-1/2 K P^-1/2 v
};
enum { PW_INV = 0, PW_HALF = 1, PW_MHALF = 2 };

// GP posterior covariance operator at the candidates (posterior.cu; ciq_set_posterior):
// COV* + jitter I = (K** + jitter I) - U U^T with U = K*x L^{-T} (n x m, fp64).
struct PostDev {
  bool on = false;
  bool inner = false;       // run_mvm re-entered for the K** part
  int m = 0;
  double* u = nullptr;      // n x m (fp64: the mean)
  float* uf = nullptr;      // n x m (fp32: the per-MVM downdate)
  float* mu = nullptr;      // n, posterior mean mu*
  float* part = nullptr;    size_t part_cap = 0;   // U^T v partials [splits][m][tp]
  float* h = nullptr;       size_t h_cap = 0;      // U^T v [m][tp]
  double* bpart = nullptr;  size_t bpart_cap = 0;  // alpha partials [blocks][tp]
  float* t = nullptr;       size_t t_cap = 0;      // K** v (rows x tp)
  float* f = nullptr;       size_t f_cap = 0;      // thompson samples staging (n x T)
  float* am_v = nullptr;    size_t am_v_cap = 0;   // argmin partials
  int64_t* am_i = nullptr;  size_t am_i_cap = 0;
  int64_t* idx = nullptr;   size_t idx_cap = 0;
};

// Nested-CIQ route (App. A, precond_nested.cu): block-Jacobi P = blockdiag of K's own
// diagonal blocks; K + sigma^2 I materialised in fp64, P^{-1} blocks inverted on the host in fp64.
struct NestedDev {
  bool on = false;
  int64_t block = 0;
  std::vector<int64_t> b0;    // block starts, nb + 1 entries (b0[nb] = n)
  bool ready = false;
  double* k64 = nullptr;      // n x ldk: K + sigma^2 I (fp64)
  int64_t ldk = 0;
  double* pinv = nullptr;     // block b (size m_b) at offset b0[b] * block, row-major, ld = m_b
  double* work = nullptr;     // fp64 vectors of pmsminres
  size_t work_cap = 0;
};

struct ciq_ctx {
  ciq_operator op{};
  PrecondDev pc;
  NestedDev nest;
  PostDev post;
  std::vector<double> ls;     // per-coordinate lengthscales of a kernel operator (copied at init)
  OpDev dev{};
  cudaStream_t stream = nullptr;       // private non-blocking work stream (graph-capturable)
  cudaStream_t user_stream = nullptr;  // the caller's stream given to ciq_init
  cudaEvent_t join_ev = nullptr;
  int rank = 0, world = 1;
  bool sharded = false;       // a ciq_comm was given: the row-sharded code path (also for world = 1)
  bool deriv = false;         // MVMs apply dK/dl instead of K (ciq_hyper_grad only)
  bool fp64_active = false;   // the current ciq_apply runs the fp64 route (precond64.cu)
  int64_t row0 = 0, row1 = 0;
  int64_t per = 0;            // rows per shard (multiple of 128; last shard may be shorter)
  int64_t nfull = 0;          // rows of the replicated (all-gathered) vectors = world * per >= n
  Comm* comm = nullptr;
  // row-sharded overlap: the MVM's local column block runs on s2 while the
  // Lanczos block's planes are all-gathered on `stream`; run_mvm applies mvm_win when on
  struct MvmWinArgs {
    bool on = false;
    int lo = 0, hi = 0, skip_lo = 0, skip_hi = 0, no_diag = 0, grid_cap = 0;
    int p_split_off = 0;       // first partial-product slot written
    int64_t ap_row_off = 0;    // first alpha-partial row written
  } mvm_win;
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // relaxed MVM schedule (params.mvm_relax): the next run_mvm launches the full-tile kernel with
  // `nsplit` column splits, or `nsplit_alt` once ctrl->relaxed (chosen by the kernel at launch)
  struct MvmGate {
    bool on = false;
    int nsplit = 0, nsplit_alt = 0;
  } mvm_gate;
  double* gsum = nullptr;     // [world][m] allgather buffer of cross-rank partial sums
  size_t gsum_cap = 0;
  double* tsum = nullptr;     // [tp] local sums
  size_t tsum_cap = 0;
  float* xs = nullptr;        // owned scaled points
  double* xs64 = nullptr;     // owned scaled points in fp64 (exact quotients of the fp32 inputs)
  float* kcopy = nullptr;     // owned dense copy (host-provided K)
  float* basis = nullptr;     // stored-basis variant: W_1 .. W_{J_max+1}, this rank's rows
  size_t basis_elems = 0;
  double* bhist = nullptr;    // stored-basis scalars [4][J_max + 1][tp] + nrm_1 / frozen_0 [2][tp]
  size_t bhist_elems = 0;
  float* bcoef = nullptr;     // combination coefficients [J][tp]
  size_t bcoef_elems = 0;
  int64_t* csr_rp = nullptr;  // owned device copy of the sparse operator's local CSR block
  int32_t* csr_ci = nullptr;
  float* csr_cv = nullptr;
  Workspace ws;
  LambdaWork lw;
  float* staging = nullptr;   // host-pointer staging (rows x tp)
  // tensor-core MVM operands
  bool tc_ok = false;
  int64_t npad = 0;
  int kf = 32;                // feature contraction of the tensor-core MVM (3 (d + 2) <= kf)
  __half* kplanes = nullptr;  // dense path (or a materialised kernel operator): split K planes [hi | lo]
  bool mat_ready = false;     // kernel operator: kplanes hold the materialised K (mvm_materialize)
  int64_t kplane_elems = 0;
  float kscale = 1.f;
  __half* feat_a = nullptr;   // [npad/8][4][8][8]
  __half* feat_b = nullptr;
  __half* planes = nullptr;   // split V planes, grown on demand
  size_t planes_elems = 0;
  float* inv_scale = nullptr;
  int inv_scale_n = 0;
  float* psplit = nullptr;    // nsplit x rows x tp partial products
  size_t psplit_elems = 0;
  float* stash = nullptr;     // lanczos_reuse: W_1..W_R of the warm-up steps (full height)
  // ciq_vjp work buffers (kept across calls: no cudaMalloc / cudaFree per call)
  float* vjp_xb = nullptr;  size_t vjp_xb_cap = 0;
  float* vjp_xv = nullptr;  size_t vjp_xv_cap = 0;
  float* vjp_y = nullptr;   size_t vjp_y_cap = 0;
  float* vjp_g = nullptr;   size_t vjp_g_cap = 0;
  double* vjp_w = nullptr;  size_t vjp_w_cap = 0;
  size_t stash_elems = 0;
  double* hist = nullptr;     // lanczos_reuse: per-step scalar history [7][R][tp]
  size_t hist_elems = 0;
  double* apart_tc = nullptr;
  size_t apart_tc_elems = 0;
  // fused alpha of the full-tile kernel (TcArgs::alpha_out): set by the recurrence around its MVM
  const Scal* alpha_fuse = nullptr;
  bool alpha_fused = false;        // the last run_mvm computed alpha itself
  double* cta_part = nullptr;      // [SMs][tp]
  size_t cta_part_elems = 0;
  unsigned* ticket = nullptr;      // zero between launches
  int last_nsplit = 1;
  int mvm_kind_used = 0;      // 1 simt, 2 tc, 3 symmetric-tile tc (of the last loop MVM)
  int last_kind = 0;          // mvm_kind_used of the captured iteration graph
  // symmetric-tile MVM (mvm_sym.cu): unit table, partial-slot prefix sums, fp32 partial products
  int2* sym_units = nullptr;
  int* sym_base = nullptr;
  float* sym_part = nullptr;
  size_t sym_part_elems = 0;
  int64_t sym_n = -1;
  int sym_tn = 0, sym_nb = 0, sym_ng = 0, sym_slots = 0, sym_nunits = 0;
  // CUDA graph of `poll_every` msMINRES iterations (period-6 buffer rotation => replayable)
  uint64_t buf_gen = 0;       // bumped on every device re-allocation (invalidates the graph)
  cudaGraphExec_t gexec = nullptr;
  uint64_t gkey[6] = {0, 0, 0, 0, 0, 0};
  int64_t graph_nodes = 0;
  Ctrl* ctrl_host = nullptr;  // pinned poll slots [2]
  int64_t staging_elems = 0;
  std::string err;
  int64_t launches = 0;
  // profile_kernels: (start, stop, iteration, kind 0=mvm 1=update)
  struct Timed { cudaEvent_t a, b; int j, kind; };
  std::vector<Timed> timed;
  std::vector<cudaEvent_t> event_pool;
  bool profiling = false;
  bool has_precond = false;
};

namespace {

bool is_device_ptr(const void* p) {
  if (p == nullptr) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

ciq_status set_err(ciq_ctx* c, ciq_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) c->err = buf; else g_init_error = buf;
  return s;
}

#define CUDA_TRY(ctx, expr)                                                                       \
  do {                                                                                            \
    cudaError_t e_ = (expr);                                                                      \
    if (e_ != cudaSuccess)                                                                        \
      return set_err(ctx, e_ == cudaErrorMemoryAllocation ? CIQ_ERR_OOM : CIQ_ERR_CUDA,           \
                     "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__);        \
  } while (0)

#define LAUNCH(ctx, expr)  \
  do {                     \
    ++(ctx)->launches;     \
    CUDA_TRY(ctx, expr);   \
  } while (0)

template <class T>
cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(count, 1) * sizeof(T));
}
template <class T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

int round16(int64_t t) { return (int)((t + 15) / 16 * 16); }

void free_workspace(Workspace& ws) {
  for (auto& b : ws.w) dfree(b);
  dfree(ws.p); dfree(ws.d); dfree(ws.y); dfree(ws.apart); dfree(ws.bpart); dfree(ws.colsq); dfree(ws.xq);
  ws.xq_elems = 0;
  dfree(ws.scal_mem);
  ws.tp = ws.nq = 0;
}

void free_lambda(LambdaWork& lw) {
  dfree(lw.basis); dfree(lw.p); dfree(lw.part); dfree(lw.h1); dfree(lw.h2); dfree(lw.bsq);
  dfree(lw.alphas); dfree(lw.betas); dfree(lw.inv); dfree(lw.len);
  lw.tpl = lw.nb = 0;
}

ciq_status ensure_workspace(ciq_ctx* c, int tp, int nq, int esz = 4) {
  Workspace& ws = c->ws;
  const int64_t rows = c->row1 - c->row0;
  const int64_t n = c->op.n;
  if (ws.tp == tp && ws.nq >= nq && ws.rows == rows && ws.esz == esz) return CIQ_OK;
  ++c->buf_gen;
  free_workspace(ws);
  ws.tp = tp;
  ws.nq = nq;
  ws.rows = rows;
  ws.esz = esz;
  // W buffers hold all N rows (the MVM input; world * per >= N with zero padding); the local
  // block is rows [row0, row1).  The fp64 route stores the same buffers as doubles (esz = 8: the
  // float* handles then address twice as many floats).
  (void)n;
  const size_t f = (size_t)esz / 4;
  for (auto& b : ws.w) CUDA_TRY(c, dalloc(&b, f * c->nfull * tp));
  CUDA_TRY(c, dalloc(&ws.p, f * rows * tp));
  CUDA_TRY(c, dalloc(&ws.d, f * 2 * nq * rows * tp));
  CUDA_TRY(c, dalloc(&ws.y, f * rows * tp));
  CUDA_TRY(c, dalloc(&ws.apart, (size_t)std::max(mvm_simt_blocks(rows), mvm64_blocks(rows)) * tp + 64 * (size_t)tp));
  CUDA_TRY(c, dalloc(&ws.bpart, (size_t)rowblocks(std::max(rows, c->nfull), tp) * tp));
  CUDA_TRY(c, dalloc(&ws.colsq, (size_t)tp));
  // scalar block
  size_t nd = (size_t)tp * 6 + (size_t)nq * tp * 9 + 2 * (size_t)nq;
  size_t bytes = nd * 8 + (size_t)tp * 8 + (size_t)nq * tp * 4 * 5 + sizeof(Ctrl) + 256;
  CUDA_TRY(c, dalloc(&ws.scal_mem, bytes));
  char* m = ws.scal_mem;
  auto takeD = [&](size_t k) { double* r = reinterpret_cast<double*>(m); m += k * 8; return r; };
  Scal& sc = ws.sc;
  sc.beta1 = takeD(tp); sc.nrm_prev = takeD(tp); sc.nrm_cur = takeD(tp); sc.tb_cur = takeD(tp); sc.alpha = takeD(tp);
  sc.c1 = takeD((size_t)nq * tp); sc.s1 = takeD((size_t)nq * tp); sc.c2 = takeD((size_t)nq * tp);
  sc.s2 = takeD((size_t)nq * tp); sc.phibar = takeD((size_t)nq * tp);
  sc.shifts = takeD(nq); sc.weights = takeD(nq); sc.col_rel = takeD(tp);
  sc.da = takeD((size_t)nq * tp); sc.db = takeD((size_t)nq * tp); sc.de = takeD((size_t)nq * tp);
  sc.df = takeD((size_t)nq * tp);
  auto takeF = [&](size_t k) { float* r = reinterpret_cast<float*>(m); m += k * 4; return r; };
  sc.ca = takeF((size_t)nq * tp); sc.cb = takeF((size_t)nq * tp); sc.ce = takeF((size_t)nq * tp);
  sc.cf = takeF((size_t)nq * tp);
  sc.cphi = takeF((size_t)nq * tp);
  sc.frozen = reinterpret_cast<int*>(m); m += (size_t)tp * 4;
  sc.col_state = reinterpret_cast<int*>(m); m += (size_t)tp * 4;
  m = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(m) + 15) & ~uintptr_t(15));
  sc.ctrl = reinterpret_cast<Ctrl*>(m);
  return CIQ_OK;
}

ciq_status ensure_staging(ciq_ctx* c, int64_t elems) {
  if (c->staging_elems >= elems) return CIQ_OK;
  dfree(c->staging);
  CUDA_TRY(c, dalloc(&c->staging, (size_t)elems));
  c->staging_elems = elems;
  return CIQ_OK;
}

// dst (rows x tp, device, zero-padded) <- src (rows x cols, ld), src host or device.
ciq_status load_rows(ciq_ctx* c, const float* src, int64_t ld, int64_t rows, int cols, float* dst, int tp) {
  if (is_device_ptr(src)) {
    LAUNCH(c, launch_load_block(src, ld, rows, cols, dst, tp, c->stream));
  } else {
    CUDA_TRY(c, cudaMemsetAsync(dst, 0, (size_t)rows * tp * 4, c->stream));
    CUDA_TRY(c, cudaMemcpy2DAsync(dst, (size_t)tp * 4, src, (size_t)ld * 4, (size_t)cols * 4, (size_t)rows,
                                  cudaMemcpyHostToDevice, c->stream));
  }
  return CIQ_OK;
}

ciq_status store_rows(ciq_ctx* c, const float* src, int tp, int64_t rows, int cols, float* dst, int64_t ld) {
  if (is_device_ptr(dst)) {
    LAUNCH(c, launch_store_block(src, tp, rows, cols, dst, ld, c->stream));
  } else {
    CUDA_TRY(c, cudaMemcpy2DAsync(dst, (size_t)ld * 4, src, (size_t)tp * 4, (size_t)cols * 4, (size_t)rows,
                                  cudaMemcpyDeviceToHost, c->stream));
  }
  return CIQ_OK;
}

cudaEvent_t pool_event(ciq_ctx* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Bracket the next launch(es) with events when profiling (begin_timed / end_timed).
void begin_timed(ciq_ctx* c, int j, int kind) {
  if (!c->profiling) return;
  ciq_ctx::Timed t{pool_event(c), pool_event(c), j, kind};
  cudaEventRecord(t.a, c->stream);
  c->timed.push_back(t);
}
void end_timed(ciq_ctx* c) {
  if (!c->profiling) return;
  cudaEventRecord(c->timed.back().b, c->stream);
}

template <class T>
ciq_status grow(ciq_ctx* c, T** buf, size_t* cap, size_t need) {
  if (*cap >= need) return CIQ_OK;
  ++c->buf_gen;
  dfree(*buf);
  CUDA_TRY(c, dalloc(buf, need));
  *cap = need;
  return CIQ_OK;
}

bool is_kernel_op(const ciq_ctx* c) {
  return c->op.kind == CIQ_OP_RBF || c->op.kind == CIQ_OP_MATERN52 || c->op.kind == CIQ_OP_MATERN32;
}

// A/B switches for experiments: compiled in only with -DCIQ_EXPERIMENTS (scripts/build_variant.py);
// the shipped library ignores the environment.
bool experiment_env(const char* name) {
#ifdef CIQ_EXPERIMENTS
  return getenv(name) != nullptr;
#else
  (void)name;
  return false;
#endif
}

// The matrix-free tensor-core MVM (mvm_tc2.cu) needs >= 4 column tiles of 64 per unit
// (tc2_choose_nsplit), i.e. N >= 256; smaller kernel operators use the fp32 SIMT kernel.
constexpr int64_t kTcMinN = 256;

int sm_count() {
  int nsm = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return nsm;
}

bool use_tc3(const ciq_ctx* c, int tp);

// Tensor-core MVM for tp columns: available unless the SIMT kernel is requested, the features do
// not fit fp16 (build_tc_features), N < 256, or d > 8 (KF = 64) with a T chunk the pair kernel
// does not take.
bool use_tc(const ciq_ctx* c, int impl, int tp) {
  if (impl == CIQ_MVM_SIMT) return false;
  if (!c->tc_ok) return false;
  if (c->op.kind == CIQ_OP_DENSE) return true;
  return c->op.n >= kTcMinN && (c->kf == 32 || use_tc3(c, tp));
}

// Dense path: split the K stream (npad/64 tiles per row block) so that row tiles x chunks x splits
// fill whole waves, keeping >= 6 K tiles per CTA.
int choose_nsplit_dense(int64_t rows, int64_t npad, int chunks, int nsm) {
  const int64_t rt = (rows + 127) / 128;
  const int64_t nkt = npad / 64;
  // accuracy bound as tc2_choose_nsplit: at most kMaxChainDense 64-wide K tiles (12 MMAs each) feed
  // one fp32 TMEM accumulator (round-toward-zero accumulation)
  constexpr int64_t kMaxChainDense = 66;
  const int smin = (int)std::max<int64_t>(1, (nkt + kMaxChainDense - 1) / kMaxChainDense);
  int best = smin;
  double best_eff = 0.0;
  for (int s = smin; s <= std::max(64, smin); ++s) {
    if (nkt / s < 6 && s > smin) break;
    const int64_t units = rt * chunks * s;
    const int64_t waves = (units + nsm - 1) / nsm;
    const double eff = (double)units / (double)(waves * nsm) - 0.002 * waves;  // favour fewer waves
    if (eff > best_eff + 0.01) { best_eff = eff; best = s; }
  }
  return best;
}

// Small N, many right-hand sides (C4: N = 5000, T = 1024): the matrix-free kernel recomputes every
// kernel tile once per 64-column chunk of T (16x for T = 1024), while the N^2 entries fit easily in
// HBM.  Such calls materialise K once (fp32 on the CUDA cores, then the dense split-fp16 planes)
// and run the HBM-bound dense kernel instead (north_star: "a dense-K path runs as a bandwidth-bound
// batched GEMV/GEMM").  CIQ_NO_MATERIALIZE=1 disables it.
constexpr int kMatMinT = 256;
constexpr int64_t kMatMaxN = 20000;
bool use_mat(const ciq_ctx* c, int tp) {
  const bool off = experiment_env("CIQ_NO_MATERIALIZE");
  return !off && !c->deriv && c->op.kind != CIQ_OP_DENSE && c->tc_ok && tp >= kMatMinT && c->op.n <= kMatMaxN;
}

ciq_status ensure_mat_planes(ciq_ctx* c) {
  if (c->mat_ready) return CIQ_OK;
  const int64_t rows = c->row1 - c->row0, n = c->op.n;
  const int64_t npad = (n + 127) / 128 * 128;
  const int64_t rows_pad = (rows + 127) / 128 * 128;
  float* k = nullptr;
  CUDA_TRY(c, dalloc(&k, (size_t)rows * n));
  CUDA_TRY(c, launch_materialize(c->dev, c->row0, rows, k, c->stream));
  unsigned int* mx = nullptr;
  CUDA_TRY(c, dalloc(&mx, 1));
  CUDA_TRY(c, cudaMemsetAsync(mx, 0, 4, c->stream));
  CUDA_TRY(c, launch_absmax(k, n, rows, n, mx, c->stream));
  unsigned int hbits = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&hbits, mx, 4, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  float amax;
  std::memcpy(&amax, &hbits, 4);
  if (!(amax > 0) || !std::isfinite(amax)) amax = 1.f;
  c->kscale = std::ldexp(1.f, 14 - (int)std::ceil(std::log2(amax)));
  c->kplane_elems = rows_pad * npad;
  CUDA_TRY(c, dalloc(&c->kplanes, (size_t)2 * c->kplane_elems));   // [hi | lo] fp16 planes
  CUDA_TRY(c, launch_split_dense(k, n, rows, n, npad, c->kscale, c->kplanes, c->kplanes + c->kplane_elems, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  dfree(k);
  dfree(mx);
  c->mat_ready = true;
  return CIQ_OK;
}

// The matrix-free MVM on CTA pairs (mvm_tc3.cu): the tensor-core path for d > 8 (feature
// contraction KF = 64, which the one-CTA kernel mvm_tc2.cu does not take), for RHS chunks of 32 / 64
// columns with enough column tiles per unit.  For d <= 8 the one-CTA kernel is faster (DESIGN.md
// §8) and is used; CIQ_TC3=1 (experiment builds only) selects the pair kernel for A/B runs.
bool use_tc3(const ciq_ctx* c, int tp) {
  if (c->op.kind == CIQ_OP_DENSE || use_mat(c, tp)) return false;
  if (c->kf == 32 && !experiment_env("CIQ_TC3")) return false;
  const int tn = tc_chunk_cols(tp);
  const int64_t rows = c->row1 - c->row0;
  const int nsm = sm_count();
  const int nsplit = tc2_choose_nsplit(rows, c->op.n, tp / tn, nsm / 2, tc3_min_tiles());
  return tc3_supported(tn, c->op.n, nsplit);
}

// Column width of one chunk of the split V planes: the pair kernel loads half of each 64-column
// MMA chunk per CTA, so its planes are laid out in TN/2-wide chunks.
int plane_cols(const ciq_ctx* c, int tp) {
  const int tn = tc_chunk_cols(tp);
  return use_tc3(c, tp) ? tn / 2 : tn;
}

// Row-sharded overlap of the Lanczos-block all-gather with the local diagonal block's MVM (the
// full-tile kernel on this rank's own column tiles, whose planes the streaming pass just wrote):
// kernel operators on the tensor-core path, no preconditioner / posterior / derivative.
bool use_overlap(const ciq_ctx* c, int impl, int tp) {
  if (!c->sharded || !use_tc(c, impl, tp) || !is_kernel_op(c) || use_mat(c, tp) || use_tc3(c, tp)) return false;
  return !c->pc.on && !c->post.on && !c->deriv && !experiment_env("CIQ_NO_OVERLAP");
}

// The symmetric-tile MVM (mvm_sym.cu): every k(x_i, x_j), i < j, evaluated once
// and applied to rows i and j.  Single GPU (it needs the whole square), RBF / Matern with d <= 8,
// RHS chunks of 16 or 32 columns.  CIQ_MVM_AUTO takes it for 16-column chunks, where the MVM is
// epilogue-bound with little tensor work per kernel value (C5 and T <= 16),
// and only where the full-tile kernel's TMEM accumulation chains are at least as long as the
// symmetric kernel's (<= 384 MMAs): the tensor core accumulates with a round-toward-zero bias of
// ~1.1e-8 per MMA, so at small N, where mvm_tc2.cu splits the columns into
// short chains, the full-tile kernel is the more accurate one (and the MVM is cheap either way).
constexpr int64_t kSymMinN = 1024;
constexpr int64_t kSymChainMmas = 384;   // mvm_sym.cu: A_ROWS = 16 tiles x 24 MMAs
bool use_sym(const ciq_ctx* c, int impl, int tp) {
  if (impl != CIQ_MVM_AUTO && impl != CIQ_MVM_TC_SYM) return false;
  if (!c->tc_ok || c->sharded || c->deriv || c->kf != 32 || !is_kernel_op(c)) return false;
  if (c->op.n < kSymMinN || c->row0 != 0 || c->row1 != c->op.n || use_mat(c, tp)) return false;
  const int tn = tc_chunk_cols(tp);
  if (!sym_supported(tn)) return false;
  if (impl == CIQ_MVM_AUTO) {
    if (tn != 16 || experiment_env("CIQ_NO_SYM")) return false;
    const int64_t ntiles = (c->op.n + 63) / 64;
    const int nsplit = tc2_choose_nsplit(c->op.n, c->op.n, tp / tn, sm_count());
    if ((ntiles + nsplit - 1) / nsplit * 12 < kSymChainMmas) return false;
  }
  return true;
}

// Unit table, slot prefix sums and partial buffer of the symmetric-tile MVM for tp columns
// (uploaded once per N / chunk width; grown before any graph capture).
ciq_status ensure_sym(ciq_ctx* c, int tp) {
  const int tn = tc_chunk_cols(tp);
  if (c->sym_n != c->op.n || c->sym_tn != tn) {
    std::vector<int2> units;
    std::vector<int> base;
    int ng = 0, slots = 0;
    sym_geometry(c->op.n, tn, &units, &base, &ng, &slots);
    ++c->buf_gen;
    dfree(c->sym_units);
    dfree(c->sym_base);
    c->sym_units = nullptr;
    c->sym_base = nullptr;
    CUDA_TRY(c, dalloc(&c->sym_units, units.size()));
    CUDA_TRY(c, dalloc(&c->sym_base, base.size()));
    CUDA_TRY(c, cudaMemcpy(c->sym_units, units.data(), units.size() * sizeof(int2), cudaMemcpyHostToDevice));
    CUDA_TRY(c, cudaMemcpy(c->sym_base, base.data(), base.size() * sizeof(int), cudaMemcpyHostToDevice));
    c->sym_n = c->op.n;
    c->sym_tn = tn;
    c->sym_nb = (int)base.size() - 1;
    c->sym_ng = ng;
    c->sym_slots = slots;
    c->sym_nunits = (int)units.size();
  }
  return grow(c, &c->sym_part, &c->sym_part_elems, (size_t)(tp / tn) * c->sym_slots * 128 * tn);
}

// Rows of the split V planes: npad, or the all-gathered height world * per when row-sharded (the
// ranks all-gather their blocks of the planes in place).
int64_t vrows(const ciq_ctx* c) { return c->sharded ? std::max(c->npad, c->nfull) : c->npad; }

// Column splits and number of alpha-partial rows of the tensor-core MVM for tp columns.
void mvm_geometry(const ciq_ctx* c, int tp, int impl, int* nsplit, int64_t* nblk) {
  const int64_t rows = c->row1 - c->row0;
  const int chunks = tp / tc_chunk_cols(tp);
  const int nsm = sm_count();
  if (c->op.kind == CIQ_OP_DENSE || use_mat(c, tp)) {
    *nsplit = choose_nsplit_dense(rows, c->npad, chunks, nsm);
    *nblk = (rows + 127) / 128 * *nsplit * 4;
  } else if (use_sym(c, impl, tp)) {
    *nsplit = 1;
    *nblk = (rows + 127) / 128;
  } else {
    // the pair kernel (mvm_tc3.cu) balances units over nsm / 2 pairs, the one-CTA kernel over nsm CTAs
    const bool pair = use_tc3(c, tp);
    *nsplit = pair ? tc2_choose_nsplit(rows, c->op.n, chunks, nsm / 2, tc3_min_tiles())
                   : tc2_choose_nsplit(rows, c->op.n, chunks, nsm);
#ifdef CIQ_EXPERIMENTS
    static const int force = getenv("CIQ_TC_NSPLIT") ? atoi(getenv("CIQ_TC_NSPLIT")) : 0;
    if (force > 0) *nsplit = force;
#endif
    *nblk = (rows + 255) / 256 * *nsplit * 8;
  }
}

// Row-sharded overlap geometry (full-tile kernel only): this rank's rows [row0, row1) are also the
// column tiles [lo, hi) of K whose V planes exist before the all-gather.  The remote launch covers
// the other tiles ([0, lo) and [hi, ntiles)) with nsr splits / nbr alpha rows, the local launch the
// window with nsl / nbl; the consumer sums nsr + nsl partial products, alpha nbr + nbl rows.
struct OverlapGeo {
  int lo, hi, nsr, nsl;
  int64_t nbr, nbl;
};
constexpr int kOverlapReservedSMs = 16;   // SMs left to the concurrent all-gather (NCCL kernels)
bool use_overlap(const ciq_ctx* c, int impl, int tp);
OverlapGeo overlap_geometry(const ciq_ctx* c, int tp) {
  OverlapGeo g{};
  const int64_t rows = c->row1 - c->row0;
  const int chunks = tp / tc_chunk_cols(tp);
  const int nsm = sm_count();
  const int ntiles = (int)((c->op.n + 63) / 64);
  g.lo = (int)(c->row0 / 64);
  g.hi = (int)std::min<int64_t>(ntiles, (c->row1 + 63) / 64);
  const int nloc = g.hi - g.lo, nrem = ntiles - nloc;
  const int capl = std::max(1, nsm - kOverlapReservedSMs);
  g.nsl = tc2_choose_nsplit(rows, (int64_t)nloc * 64, chunks, capl);
  g.nsr = nrem > 0 ? tc2_choose_nsplit(rows, (int64_t)nrem * 64, chunks, nsm) : 0;
  g.nbl = (rows + 255) / 256 * g.nsl * 8;
  g.nbr = (rows + 255) / 256 * g.nsr * 8;
  return g;
}

// Allocate every buffer run_mvm(tp, allow_split) may need (so a CUDA-graph capture never
// allocates).
ciq_status post_buffers(ciq_ctx* c, int tp);

ciq_status prepare_mvm_buffers(ciq_ctx* c, int tp, int impl) {
  if (c->post.on) {
    ciq_status sp = post_buffers(c, tp);
    if (sp != CIQ_OK) return sp;
  }
  if (!use_tc(c, impl, tp)) return CIQ_OK;
  if (use_mat(c, tp)) {
    ciq_status sm = ensure_mat_planes(c);
    if (sm != CIQ_OK) return sm;
  }
  if (use_sym(c, impl, tp)) {
    ciq_status ss = ensure_sym(c, tp);
    if (ss != CIQ_OK) return ss;
  }
  const int64_t rows = c->row1 - c->row0;
  int nsplit = 1;
  int64_t nblk = 0;
  mvm_geometry(c, tp, impl, &nsplit, &nblk);
  ciq_status st = grow(c, &c->planes, &c->planes_elems, (size_t)2 * vrows(c) * tp);
  if (st != CIQ_OK) return st;
  if (c->inv_scale_n < tp) {
    ++c->buf_gen;
    dfree(c->inv_scale);
    CUDA_TRY(c, dalloc(&c->inv_scale, (size_t)tp));
    c->inv_scale_n = tp;
  }
  if (use_overlap(c, impl, tp)) {   // the two windowed launches' partial products / alpha rows
    const OverlapGeo og = overlap_geometry(c, tp);
    nsplit = std::max(nsplit, og.nsr + og.nsl);
    nblk = std::max<int64_t>(nblk, og.nbr + og.nbl);
    if (c->s2 == nullptr) {
      CUDA_TRY(c, cudaStreamCreateWithFlags(&c->s2, cudaStreamNonBlocking));
      CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
      CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    }
  }
  if (nsplit > 1) {
    st = grow(c, &c->psplit, &c->psplit_elems, (size_t)nsplit * rows * tp);
    if (st != CIQ_OK) return st;
  }
  st = grow(c, &c->cta_part, &c->cta_part_elems, (size_t)sm_count() * tp);
  if (st != CIQ_OK) return st;
  if (c->ticket == nullptr) {
    CUDA_TRY(c, cudaMalloc(&c->ticket, sizeof(unsigned)));
    CUDA_TRY(c, cudaMemset(c->ticket, 0, sizeof(unsigned)));
  }
  return grow(c, &c->apart_tc, &c->apart_tc_elems, (size_t)nblk * tp);
}

// P (+ alpha partials) <- K V.  With the tensor-core path the result may be split into
// `*nsplit_out` partial products (stride rows*tp) when allow_split; otherwise it is complete.
ciq_status run_post_mvm(ciq_ctx* c, const float* v, int tp, float* p, double* apart, const Ctrl* done, int impl,
                        const double* nrm, int* nsplit_out, double** apart_used, int* apart_nblk, bool skip_pack);

ciq_status run_mvm(ciq_ctx* c, const float* v, int tp, float* p, double* apart, const Ctrl* done, int impl,
                   const double* nrm = nullptr, bool allow_split = false, int* nsplit_out = nullptr,
                   double** apart_used = nullptr, int* apart_nblk = nullptr, bool skip_pack = false) {
  if (c->post.on && !c->post.inner)
    return run_post_mvm(c, v, tp, p, apart, done, impl, nrm, nsplit_out, apart_used, apart_nblk, skip_pack);
  const int64_t rows = c->row1 - c->row0;
  if (nsplit_out) *nsplit_out = 1;
  if (!use_tc(c, impl, tp)) {
    if (impl == CIQ_MVM_TC)
      return set_err(c, CIQ_ERR_INVALID_ARG,
                     "tensor-core MVM unavailable for this operator (N < 256, huge features, or d > 8 with an RHS chunk < 32)");
    OpDev od = c->dev;
    if (c->deriv) {   // dK/dl (ciq_hyper_grad): kernel kinds 4-6, o^2 / l, no sigma^2
      od.kind += 10;   // internal kinds 11-13 (mvm_*.cu: KIND templates 4-6)
      od.o2 = c->op.outputscale / c->ls[0];
      od.diag = 0.f;
    }
    LAUNCH(c, launch_mvm_simt(od, v, tp, c->row0, c->row1, p, tp, apart, done, c->stream));
    if (apart_used) *apart_used = apart;
    if (apart_nblk) *apart_nblk = mvm_simt_blocks(rows);
    c->mvm_kind_used = 1;
    return CIQ_OK;
  }
  const int tn = tc_chunk_cols(tp);
  const int chunks = tp / tn;
  const int nsm = sm_count();
  (void)allow_split;
  const bool mat = use_mat(c, tp);
  if (mat) {
    ciq_status sm = ensure_mat_planes(c);
    if (sm != CIQ_OK) return sm;
  }
  const bool dense = c->op.kind == CIQ_OP_DENSE || mat;
  const bool sym = !dense && use_sym(c, impl, tp);
  if (impl == CIQ_MVM_TC_SYM && !sym)
    return set_err(c, CIQ_ERR_INVALID_ARG,
                   "symmetric-tile MVM unavailable (needs one GPU, RBF / Matern, d <= 8, N >= 1024, RHS chunk 16 or 32)");
  if (sym) {
    ciq_status ss = ensure_sym(c, tp);
    if (ss != CIQ_OK) return ss;
  }
  int nsplit = 1;
  int64_t nblk = 0;
  mvm_geometry(c, tp, impl, &nsplit, &nblk);
  const bool win = c->mvm_win.on && !dense && !sym && !use_tc3(c, tp) && nsplit_out != nullptr;
  if (c->mvm_win.on && !win) return set_err(c, CIQ_ERR_INVALID_ARG, "internal: windowed MVM needs the full-tile kernel");
  if (win) {   // one column window of the row-sharded overlap (overlap_geometry)
    const ciq_ctx::MvmWinArgs& w = c->mvm_win;
    const int ntw = (w.hi - w.lo) - (w.skip_hi - w.skip_lo);
    const int capw = w.grid_cap > 0 ? std::min(w.grid_cap, nsm) : nsm;
    nsplit = tc2_choose_nsplit(rows, (int64_t)ntw * 64, chunks, capw);
    nblk = (rows + 255) / 256 * nsplit * 8;
  }
  const bool gated = c->mvm_gate.on && !dense && !sym && !win && !use_tc3(c, tp) && done != nullptr;
  const bool gated_dense = c->mvm_gate.on && dense && done != nullptr;   // level 2 only (K_hi planes)
  if (gated) {   // the relaxed schedule's accurate grid (buffers sized for it; the alternative is smaller)
    nsplit = c->mvm_gate.nsplit;
    nblk = (rows + 255) / 256 * nsplit * 8;
  }
  ciq_status st = grow(c, &c->planes, &c->planes_elems, (size_t)2 * vrows(c) * tp);
  if (st != CIQ_OK) return st;
  if (c->inv_scale_n < tp) {
    ++c->buf_gen;
    dfree(c->inv_scale);
    CUDA_TRY(c, dalloc(&c->inv_scale, (size_t)tp));
    c->inv_scale_n = tp;
  }
  float* pout = p;
  if (nsplit > 1 || win) {
    const size_t off = win ? (size_t)c->mvm_win.p_split_off : 0;
    st = grow(c, &c->psplit, &c->psplit_elems, (off + nsplit) * rows * tp);
    if (st != CIQ_OK) return st;
    pout = c->psplit + off * rows * tp;
  }
  double* ap = apart;
  if (apart != nullptr) {
    const size_t off = win ? (size_t)c->mvm_win.ap_row_off : 0;
    st = grow(c, &c->apart_tc, &c->apart_tc_elems, (off + nblk) * tp);
    if (st != CIQ_OK) return st;
    ap = c->apart_tc + off * tp;
  }
  // (skip_pack: the previous streaming pass already wrote v's split planes and inv_scale)
  if (!skip_pack)
    LAUNCH(c, launch_pack_v(v, c->op.n, vrows(c), tp, plane_cols(c, tp), nrm, c->planes, c->inv_scale, c->stream));
  TcArgs a{};
  a.kind = c->op.kind + (c->deriv ? 10 : 0);   // 11-13: dK/dl (ciq_hyper_grad; KIND templates 4-6)
  a.n = c->op.n;
  a.npad = c->npad;
  a.vrows = vrows(c);
  a.row0 = c->row0;
  a.row1 = c->row1;
  a.tp = tp;
  a.nsplit = nsplit;
  a.feat_a = c->feat_a;
  a.feat_b = c->feat_b;
  a.vplanes = c->planes;
  a.inv_scale = c->inv_scale;
  a.v = v;
  a.p = pout;
  a.p_split_stride = (size_t)rows * tp;
  a.apart = ap;
  a.o2 = c->deriv ? c->op.outputscale / c->ls[0] : c->op.outputscale;
  a.diag = c->deriv ? 0.f : c->op.diag;
  a.done = done;
  a.kplanes = c->kplanes;
  a.kplane_elems = c->kplane_elems;
  a.kscale_inv = 1.f / c->kscale;
  a.chunks = chunks;
  const bool pair = !dense && use_tc3(c, tp);
  a.kf = c->kf;
  a.nunits = dense ? (int)((rows + 127) / 128) * nsplit * chunks
                   : (pair ? tc3_units(rows, nsplit, chunks) : tc2_units(rows, nsplit, chunks));
  if (gated_dense) a.gate = &done->relaxed;
  if (gated) {
    a.gate = &done->relaxed;
    a.nsplit_alt = c->mvm_gate.nsplit_alt;
    a.nunits_alt = tc2_units(rows, c->mvm_gate.nsplit_alt, chunks);
  }
  if (win) {
    a.win_lo = c->mvm_win.lo;
    a.win_hi = c->mvm_win.hi;
    a.skip_lo = c->mvm_win.skip_lo;
    a.skip_hi = c->mvm_win.skip_hi;
    a.no_diag = c->mvm_win.no_diag;
    a.grid_cap = c->mvm_win.grid_cap;
  }
#ifdef CIQ_TC_TRACE
  a.dbg = getenv("CIQ_TC_DEBUG") ? atoi(getenv("CIQ_TC_DEBUG")) : 0;
  if ((a.dbg & 128) && !dense) {
    cudaMalloc(&a.dbg_clk, 32 * 256 * sizeof(long long));   // device memory: stamps must be cheap stores
    cudaMemset(a.dbg_clk, 0, 32 * 256 * sizeof(long long));
  }
#endif
  if (sym) {
    a.nunits = c->sym_nunits * chunks;
    a.sym_units = c->sym_units;
    a.sym_base = c->sym_base;
    a.sym_part = c->sym_part;
    a.sym_nb = c->sym_nb;
    a.sym_ng = c->sym_ng;
    a.sym_b = sym_group_blocks(tn);
    a.sym_slots = c->sym_slots;
  }
  c->alpha_fused = false;
#ifdef CIQ_NO_ALPHA_FUSE
  c->alpha_fuse = nullptr;   // experiments only: the separate alpha pass
#endif
  if (!dense && !sym && !pair && !win && ap != nullptr && c->alpha_fuse != nullptr && !c->sharded && !c->post.on &&
      !c->deriv && c->cta_part != nullptr &&
      c->cta_part_elems >= (size_t)nsm * tp && c->ticket != nullptr) {
    a.alpha_out = c->alpha_fuse->alpha;
    a.alpha_nrm = c->alpha_fuse->nrm_cur;
    a.alpha_frozen = c->alpha_fuse->frozen;
    a.cta_part = c->cta_part;
    a.ticket = c->ticket;
    c->alpha_fused = true;
  }
  if (dense) LAUNCH(c, launch_mvm_dense2(a, nsm, c->stream));
  else if (sym) LAUNCH(c, launch_mvm_sym(a, nsm, c->stream));
  else if (pair) LAUNCH(c, launch_mvm_tc3(a, nsm, c->stream));
  else LAUNCH(c, launch_mvm_tc2(a, nsm, c->stream));
#ifdef CIQ_TC_TRACE
  if (a.dbg_clk) {  // experiments only: the per-tile timeline of CTA 0 / pair 0 (slots: T2_STAMP / T3_STAMP)
    cudaStreamSynchronize(c->stream);
    std::vector<long long> h(32 * 256);
    cudaMemcpy(h.data(), a.dbg_clk, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
    long long t0 = h[0];
    for (int sl = 0; sl < 32; ++sl)
      if (h[sl * 256] != 0 && h[sl * 256] < t0) t0 = h[sl * 256];
    for (int j = 0; j < 256; ++j) {
      fprintf(stderr, "%4d", j);
      for (int sl = 0; sl < (j < 8 ? 32 : 14); ++sl) {
        const long long v = h[sl * 256 + j];
        fprintf(stderr, " %8lld", v ? v - t0 : -1LL);
      }
      fprintf(stderr, "\n");
    }
    cudaFree(a.dbg_clk);
  }
#endif
  if (nsplit > 1 && nsplit_out == nullptr)  // caller wants the complete product in p
    LAUNCH(c, launch_sum_splits(c->psplit, nsplit, (size_t)rows * tp, rows * tp, p, c->stream,
                                gated ? &done->relaxed : nullptr, gated ? c->mvm_gate.nsplit_alt : 0));
  if (nsplit_out) *nsplit_out = nsplit;
  if (apart_used) *apart_used = ap;
  if (apart_nblk) *apart_nblk = (int)nblk;
  c->mvm_kind_used = sym ? 3 : 2;
  return CIQ_OK;
}

// Work buffers of run_post_mvm at this tp (grown before any graph capture).
ciq_status post_buffers(ciq_ctx* c, int tp) {
  PostDev& Q = c->post;
  const int64_t rows = c->row1 - c->row0;
  ciq_status st = grow(c, &Q.part, &Q.part_cap, (size_t)post_splits(rows) * Q.m * tp);
  if (st == CIQ_OK) st = grow(c, &Q.h, &Q.h_cap, (size_t)Q.m * tp);
  if (st == CIQ_OK) st = grow(c, &Q.bpart, &Q.bpart_cap, (size_t)post_apply_blocks(rows) * tp);
  if (st == CIQ_OK) st = grow(c, &Q.t, &Q.t_cap, (size_t)rows * tp);
  return st;
}

// p <- (COV* + jitter I) v = (K** + jitter I) v - U (U^T v)  (eq. thompson_sample's COV*),
// with the fixed-order fp64 partials of p . v when the caller wants alpha partials.  K** v is the
// ordinary MVM (tcgen05 matrix-free kernel); the downdate is two skinny fp32 GEMMs (posterior.cu).
ciq_status run_post_mvm(ciq_ctx* c, const float* v, int tp, float* p, double* apart, const Ctrl* done, int impl,
                        const double* nrm, int* nsplit_out, double** apart_used, int* apart_nblk, bool skip_pack) {
  PostDev& Q = c->post;
  const int64_t rows = c->row1 - c->row0;
  ciq_status st = post_buffers(c, tp);
  if (st != CIQ_OK) return st;
  Q.inner = true;
  st = run_mvm(c, v, tp, Q.t, nullptr, done, impl, nrm, false, nullptr, nullptr, nullptr, skip_pack);
  Q.inner = false;
  if (st != CIQ_OK) return st;
  LAUNCH(c, launch_post_downdate(Q.uf, Q.m, v, Q.t, tp, rows, Q.part, Q.h, p, apart ? Q.bpart : nullptr, c->stream));
  if (nsplit_out) *nsplit_out = 1;
  if (apart_used) *apart_used = apart ? Q.bpart : nullptr;
  if (apart_nblk) *apart_nblk = post_apply_blocks(rows);
  return CIQ_OK;
}

// Dense path: split the (local rows of) K once into fp16 planes with a global power-of-two scale
// 2^(14 - ceil(log2 max|K|)) so both halves stay in the fp16 normal range.
bool build_dense_planes(ciq_ctx* c) {
  const int64_t rows = c->row1 - c->row0, n = c->op.n;
  const int64_t npad = (n + 127) / 128 * 128;
  const int64_t rows_pad = (rows + 127) / 128 * 128;
  unsigned int* mx = nullptr;
  if (cudaMalloc(&mx, 4) != cudaSuccess) return false;
  cudaMemset(mx, 0, 4);
  const float* kloc = c->dev.k + c->row0 * c->dev.ldk;
  launch_absmax(kloc, c->dev.ldk, rows, n, mx, c->stream);
  unsigned int hbits = 0;
  cudaMemcpy(&hbits, mx, 4, cudaMemcpyDeviceToHost);
  cudaFree(mx);
  float amax;
  std::memcpy(&amax, &hbits, 4);
  if (!(amax > 0) || !std::isfinite(amax)) amax = 1.f;
  c->kscale = std::ldexp(1.f, 14 - (int)std::ceil(std::log2(amax)));
  c->kplane_elems = rows_pad * npad;
  if (cudaMalloc(&c->kplanes, (size_t)2 * c->kplane_elems * 2) != cudaSuccess) return false;
  if (launch_split_dense(kloc, c->dev.ldk, rows, n, npad, c->kscale, c->kplanes, c->kplanes + c->kplane_elems,
                         c->stream) != cudaSuccess)
    return false;
  c->npad = npad;
  c->tc_ok = cudaStreamSynchronize(c->stream) == cudaSuccess;
  return c->tc_ok;
}

// Augmented split-fp16 features of the tensor-core MVM (mvm_tc.cu): with y = (x - mean)/l *
// sqrt(log2 e) and h = |y|^2/2, A_i = [y_i, -h_i, 1], B_j = [y_j, 1, -h_j] so that
// A_i.B_j = -(log2 e/2) |x_i - x_j|^2/l^2; rows [Ah | Al | Ah | 0], [Bh | Bh | Bl | 0] (K = 32),
// stored as K-major 8x8 core matrices [n/8][4][8][8].
bool build_tc_features(ciq_ctx* c, const std::vector<float>& xh) {
  const int64_t n = c->op.n;
  const int d = (int)c->op.d;
  const int d2 = d + 2;
  if (3 * d2 > 64) return false;
  const int kf = 3 * d2 > 32 ? 64 : 32;   // feature contraction (64: pair kernel only)
  const int64_t npad = (n + 127) / 128 * 128;
  std::vector<double> mean(d, 0.0);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) mean[k] += xh[i * d + k];
  for (int k = 0; k < d; ++k) mean[k] /= (double)n;
  const double sl = std::sqrt(1.4426950408889634);
  // (+256 zero rows: the 256-row units of mvm_tc2.cu may start at any 128-aligned row < npad)
  std::vector<__half> fa((size_t)(npad + 256) * kf, __float2half(0.f)), fb((size_t)(npad + 256) * kf, __float2half(0.f));
  std::vector<double> a(d2), b(d2);
  double hmax = 0.0;
  auto put = [&](std::vector<__half>& f, int64_t i, int kidx, double val, bool lo) {
    __half h = __float2half_rn((float)val);
    if (lo) h = __float2half_rn((float)(val - (double)__half2float(h)));
    const int64_t ng = i / 8, r = i % 8;
    const int kc = kidx / 8, kk = kidx % 8;
    f[(size_t)((ng * (kf / 8) + kc) * 64 + r * 8 + kk)] = h;
  };
  for (int64_t i = 0; i < n; ++i) {
    double hh = 0.0;
    for (int k = 0; k < d; ++k) {
      const double y = ((double)xh[i * d + k] - mean[k]) * sl;
      a[k] = b[k] = y;
      hh += 0.5 * y * y;
    }
    hmax = std::max(hmax, hh);
    a[d] = -hh; a[d + 1] = 1.0;
    b[d] = 1.0; b[d + 1] = -hh;
    for (int k = 0; k < d2; ++k) {
      put(fa, i, k, a[k], false);          // Ah
      put(fa, i, d2 + k, a[k], true);      // Al
      put(fa, i, 2 * d2 + k, a[k], false); // Ah
      put(fb, i, k, b[k], false);          // Bh
      put(fb, i, d2 + k, b[k], false);     // Bh
      put(fb, i, 2 * d2 + k, b[k], true);  // Bl
    }
  }
  if (hmax > 2.0e4) return false;  // fp16 range / cancellation: use the SIMT path
  if (cudaMalloc(&c->feat_a, fa.size() * 2) != cudaSuccess) return false;
  if (cudaMalloc(&c->feat_b, fb.size() * 2) != cudaSuccess) return false;
  cudaMemcpy(c->feat_a, fa.data(), fa.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(c->feat_b, fb.data(), fb.size() * 2, cudaMemcpyHostToDevice);
  c->npad = npad;
  c->kf = kf;
  return cudaGetLastError() == cudaSuccess;
}

ciq_status precond_power(ciq_ctx* c, int which, const float* v, int tp, int64_t rows, float* out,
                         const float* dotv);

// vals[0..m) <- sum over ranks of vals (allgather + rank-order sum): identical on every rank.
ciq_status global_sum(ciq_ctx* c, double* vals, int m) {
  if (!c->sharded) return CIQ_OK;
  ciq_status st = grow(c, &c->gsum, &c->gsum_cap, (size_t)c->world * m);
  if (st != CIQ_OK) return st;
  if (!c->comm->allgather(vals, c->gsum, (size_t)m * 8, c->stream))
    return set_err(c, CIQ_ERR_NCCL, "allgather: %s", c->comm->error());
  LAUNCH(c, launch_sum_ranks(c->gsum, c->world, m, vals, c->stream));
  return CIQ_OK;
}

// Every rank's row block [row0, row1) of a full-height (nfull x tp) vector -> all ranks.
ciq_status allgather_rows(ciq_ctx* c, float* full, int tp) {
  if (!c->sharded) return CIQ_OK;
  const size_t bytes = (size_t)c->per * tp * 4;
  if (!c->comm->allgather(full + (size_t)c->rank * c->per * tp, full, bytes, c->stream))
    return set_err(c, CIQ_ERR_NCCL, "allgather: %s", c->comm->error());
  return CIQ_OK;
}

// The split-fp16 V planes of this rank's rows to every rank: per layout chunk and plane (hi, lo)
// the rows [rank * per, (rank + 1) * per) are one contiguous run of per * tn halves.
ciq_status allgather_planes(ciq_ctx* c, int tp) {
  if (!c->sharded) return CIQ_OK;
  const int tn = plane_cols(c, tp);
  const int64_t vr = vrows(c);
  for (int ch = 0; ch < tp / tn; ++ch)
    for (int pl = 0; pl < 2; ++pl) {
      __half* base = c->planes + ((size_t)ch * 2 + pl) * vr * tn;
      if (!c->comm->allgather(base + (size_t)c->rank * c->per * tn, base, (size_t)c->per * tn * 2, c->stream))
        return set_err(c, CIQ_ERR_NCCL, "allgather (planes): %s", c->comm->error());
    }
  return CIQ_OK;
}

// Lambda estimation: Lanczos with full re-orthogonalisation on `cols` start
// columns; Ritz extremes pooled; margins of reading G6.
ciq_status estimate_lambda(ciq_ctx* c, const ciq_params* p, double lower_bound, double* lmin, double* lmax,
                           double* rmin, double* rmax, int* mvms) {
  const int cols = std::max(1, p->lanczos_cols);
  const int tpl = round16(cols);
  const int J = std::max(1, p->lanczos_iters);
  const int64_t n = c->op.n;
  const int64_t nf = c->nfull;                 // basis vectors are full height (row-sharded work)
  const int64_t rows = c->row1 - c->row0;
  const int64_t r0 = c->row0;
  LambdaWork& lw = c->lw;
  if (lw.tpl != tpl || lw.nb < J + 1 || lw.rows != rows) {
    free_lambda(lw);
    lw.tpl = tpl; lw.nb = J + 1; lw.rows = rows;
    CUDA_TRY(c, dalloc(&lw.basis, (size_t)(J + 1) * nf * tpl));
    CUDA_TRY(c, dalloc(&lw.p, (size_t)rows * tpl));
    CUDA_TRY(c, dalloc(&lw.part, (size_t)rowblocks(rows, tpl) * (J + 1) * tpl + (size_t)mvm_simt_blocks(rows) * tpl));
    CUDA_TRY(c, dalloc(&lw.h1, (size_t)(J + 1) * tpl));
    CUDA_TRY(c, dalloc(&lw.h2, (size_t)(J + 1) * tpl));
    CUDA_TRY(c, dalloc(&lw.bsq, (size_t)tpl));
    CUDA_TRY(c, dalloc(&lw.alphas, (size_t)(J + 1) * tpl));
    CUDA_TRY(c, dalloc(&lw.betas, (size_t)(J + 1) * tpl));
    CUDA_TRY(c, dalloc(&lw.inv, (size_t)tpl));
    CUDA_TRY(c, dalloc(&lw.len, (size_t)tpl));
  }
  cudaStream_t s = c->stream;
  const int64_t bstride = nf * tpl;
  auto vec = [&](int k) { return lw.basis + (size_t)k * bstride; };
  CUDA_TRY(c, cudaMemsetAsync(lw.basis, 0, (size_t)bstride * 4, s));
  if (p->lanczos_start != nullptr) {  // this rank's rows of the start block
    if (load_rows(c, p->lanczos_start, p->ld_start > 0 ? p->ld_start : cols, rows, cols, vec(0) + r0 * tpl, tpl) !=
        CIQ_OK)
      return CIQ_ERR_CUDA;
  } else {
    LAUNCH(c, launch_randn_fill(vec(0) + r0 * tpl, rows, cols, tpl, r0, p->seed, s));
  }
  const int nbr = rowblocks(rows, tpl);
  LAUNCH(c, launch_colsq_partials(vec(0) + r0 * tpl, rows, tpl, lw.part, s));
  LAUNCH(c, launch_reduce_cols(lw.part, nbr, tpl, lw.bsq, 0, s));
  ciq_status gst = global_sum(c, lw.bsq, tpl);
  if (gst != CIQ_OK) return gst;
  LAUNCH(c, launch_sqrt_inplace(lw.bsq, tpl, s));
  LAUNCH(c, launch_scale_cols(vec(0) + r0 * tpl, rows, tpl, lw.bsq, s));
  gst = allgather_rows(c, vec(0), tpl);
  if (gst != CIQ_OK) return gst;
  std::vector<int> len(tpl);
  for (int k = 0; k < tpl; ++k) len[k] = (k < cols) ? 0 : -1000000;
  CUDA_TRY(c, cudaMemcpyAsync(lw.len, len.data(), tpl * 4, cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaMemsetAsync(lw.alphas, 0, (size_t)(J + 1) * tpl * 8, s));
  CUDA_TRY(c, cudaMemsetAsync(lw.betas, 0, (size_t)(J + 1) * tpl * 8, s));
  const double bd = 1e-10;
  int done_mvms = 0;
  for (int j = 0; j < J; ++j) {
    const float* vj = vec(j);
    if (c->fp64_active) {   // fp64 route: Lanczos on the materialised M (fp32 basis)
      LAUNCH(c, launch_mvm64(c->pc.m64, c->pc.ldm, rows, n, vj, false, tpl, r0, lw.p, false, nullptr, nullptr, s));
    } else if (c->pc.on) {
      // Lanczos on M = P^{-1/2} K P^{-1/2} (App. A: the rule must cover the spectrum of M);
      // row-sharded: P^{-1/2} on this rank's rows, the result all-gathered for the K MVM
      PrecondDev& P = c->pc;
      ciq_status gs = grow(c, &P.t1, &P.t_cap, (size_t)2 * nf * tpl);
      if (gs != CIQ_OK) return gs;
      float* t2 = P.t1 + (size_t)nf * tpl;
      if (precond_power(c, PW_MHALF, vj + r0 * tpl, tpl, rows, P.t1 + r0 * tpl, nullptr) != CIQ_OK) return CIQ_ERR_CUDA;
      gs = allgather_rows(c, P.t1, tpl);
      if (gs != CIQ_OK) return gs;
      if (run_mvm(c, P.t1, tpl, t2, nullptr, nullptr, p->mvm_impl) != CIQ_OK) return CIQ_ERR_CUDA;
      if (precond_power(c, PW_MHALF, t2, tpl, rows, lw.p, nullptr) != CIQ_OK) return CIQ_ERR_CUDA;
    } else if (run_mvm(c, vj, tpl, lw.p, nullptr, nullptr, p->mvm_impl) != CIQ_OK) {
      return CIQ_ERR_CUDA;
    }
    ++done_mvms;
    for (int pass = 0; pass < 2; ++pass) {
      double* h = pass == 0 ? lw.h1 : lw.h2;
      LAUNCH(c, launch_basis_dots(vec(0) + r0 * tpl, bstride, j + 1, rows, tpl, lw.p, lw.part, s));
      LAUNCH(c, launch_reduce_cols(lw.part, nbr, (j + 1) * tpl, h, 0, s));
      gst = global_sum(c, h, (j + 1) * tpl);
      if (gst != CIQ_OK) return gst;
      LAUNCH(c, launch_basis_axpy(vec(0) + r0 * tpl, bstride, j + 1, rows, tpl, h, lw.p, s));
    }
    LAUNCH(c, launch_colsq_partials(lw.p, rows, tpl, lw.part, s));
    LAUNCH(c, launch_reduce_cols(lw.part, nbr, tpl, lw.bsq, 0, s));
    gst = global_sum(c, lw.bsq, tpl);
    if (gst != CIQ_OK) return gst;
    LAUNCH(c, launch_lanczos_coeffs(lw.h1, lw.h2, lw.bsq, j, J + 1, tpl, bd, lw.alphas, lw.betas, lw.len, lw.inv, s));
    CUDA_TRY(c, cudaMemcpyAsync(len.data(), lw.len, tpl * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    bool any = false;
    for (int k = 0; k < cols; ++k) any = any || (len[k] == j + 1);
    if (!any || j == J - 1) break;
    LAUNCH(c, launch_scale_cols_by(lw.p, vec(j + 1) + r0 * tpl, rows, tpl, lw.inv, s));
    gst = allgather_rows(c, vec(j + 1), tpl);
    if (gst != CIQ_OK) return gst;
  }
  std::vector<double> al((size_t)(J + 1) * tpl), be((size_t)(J + 1) * tpl);
  CUDA_TRY(c, cudaMemcpyAsync(al.data(), lw.alphas, al.size() * 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaMemcpyAsync(be.data(), lw.betas, be.size() * 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  double emin_all = INFINITY, emax_all = -INFINITY;
  std::vector<double> a(J + 1), b(J + 1);
  for (int k = 0; k < cols; ++k) {
    int m = std::abs(len[k]);
    if (m < 1) continue;
    for (int i = 0; i < m; ++i) a[i] = al[(size_t)i * tpl + k];
    for (int i = 0; i + 1 < m; ++i) b[i] = be[(size_t)i * tpl + k];
    double e0, e1;
    ciqh::tridiag_extremes(a.data(), b.data(), m, &e0, &e1);
    emin_all = std::min(emin_all, e0);
    emax_all = std::max(emax_all, e1);
  }
  *rmin = emin_all;
  *rmax = emax_all;
  *lmax = 1.01 * emax_all;
  *lmin = 0.99 * emin_all;
  if (lower_bound > 0) *lmin = std::min(*lmin, lower_bound);
  *mvms = done_mvms;
  if (!(*lmin > 0) || !std::isfinite(*lmax))
    return set_err(c, CIQ_ERR_NOT_PD, "lambda_min estimate %g <= 0: operator is not positive definite", *lmin);
  return CIQ_OK;
}

// Order the private work stream after everything already enqueued on the caller's stream.
ciq_status join_user_stream(ciq_ctx* c) {
  CUDA_TRY(c, cudaEventRecord(c->join_ev, c->user_stream));
  CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->join_ev, 0));
  return CIQ_OK;
}

// out = P^p v (p by index: PW_INV -1, PW_HALF 1/2, PW_MHALF -1/2) on rows x tp (device), optionally
// with fixed-order fp64 partials of sum_i out[i][c] dotv[i][c] into c->pc.bpart.
ciq_status precond_power(ciq_ctx* c, int which, const float* v, int tp, int64_t rows, float* out,
                         const float* dotv) {
  PrecondDev& P = c->pc;
  const int ns = utv_splits(rows);
  ciq_status st = grow(c, &P.part, &P.part_cap, (size_t)ns * P.r2 * tp);
  if (st != CIQ_OK) return st;
  st = grow(c, &P.h, &P.h_cap, (size_t)P.r2 * tp);
  if (st != CIQ_OK) return st;
  st = grow(c, &P.bpart, &P.bpart_cap, (size_t)uapply_blocks(rows) * tp);
  if (st != CIQ_OK) return st;
  LAUNCH(c, launch_utv(P.u, P.r2, P.r2, v, tp, rows, ns, P.part, c->stream));
  LAUNCH(c, launch_reduce_cols(P.part, ns, P.r2 * tp, P.h, 0, c->stream));
  st = global_sum(c, P.h, P.r2 * tp);   // U^T v over all ranks' rows (the L^T W sum of SURVEY §8(e))
  if (st != CIQ_OK) return st;
  LAUNCH(c, launch_uapply(P.u, P.r2, P.r2, P.g[which], P.h, v, P.a[which], tp, rows, out, dotv,
                          dotv ? P.bpart : nullptr, c->stream));
  return CIQ_OK;
}

// Build U, the gains and scalars from L (device, n x rank) and sigma2 (App. A).
ciq_status build_precond(ciq_ctx* c) {
  PrecondDev& P = c->pc;
  const int64_t n = c->row1 - c->row0;   // this rank's rows of L (all N on one GPU)
  const int r = P.rank;
  double* gram_d = nullptr;
  CUDA_TRY(c, dalloc(&gram_d, (size_t)r * r));
  LAUNCH(c, launch_gram(P.l, r, r, n, gram_d, c->stream));
  ciq_status gs = global_sum(c, gram_d, r * r);   // L^T L = sum over the ranks' row blocks
  if (gs != CIQ_OK) return gs;
  std::vector<double> gram((size_t)r * r), w(r), vec((size_t)r * r);
  CUDA_TRY(c, cudaMemcpyAsync(gram.data(), gram_d, gram.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  dfree(gram_d);
  ciqh::sym_eig_jacobi(gram.data(), r, w.data(), vec.data());   // L^T L = W diag(s^2) W^T
  const double smax2 = std::max(w[0], 0.0);
  int r2 = 0;
  while (r2 < r && w[r2] > 1e-12 * smax2 && w[r2] > 0) ++r2;
  P.r2 = std::max(r2, 1);
  std::vector<double> wsi((size_t)r * P.r2, 0.0);
  for (int k = 0; k < r; ++k)
    for (int j = 0; j < r2; ++j) wsi[(size_t)k * P.r2 + j] = vec[(size_t)k * r + j] / std::sqrt(w[j]);
  double* wsi_d = nullptr;
  CUDA_TRY(c, dalloc(&wsi_d, wsi.size()));
  CUDA_TRY(c, cudaMemcpyAsync(wsi_d, wsi.data(), wsi.size() * 8, cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, dalloc(&P.u, (size_t)n * P.r2));
  LAUNCH(c, launch_small_right_mul(P.l, r, r, wsi_d, P.r2, n, P.u, P.r2, c->stream));
  const double s2 = P.sigma2;
  const double pw[3] = {-1.0, 0.5, -0.5};
  for (int k = 0; k < 3; ++k) {
    std::vector<double> g(P.r2, 0.0);
    const double ap = std::pow(s2, pw[k]);
    for (int j = 0; j < r2; ++j) g[j] = std::pow(w[j] + s2, pw[k]) - ap;
    P.a[k] = (float)ap;
    P.ad[k] = ap;
    CUDA_TRY(c, dalloc(&P.g[k], (size_t)P.r2));
    CUDA_TRY(c, cudaMemcpyAsync(P.g[k], g.data(), g.size() * 8, cudaMemcpyHostToDevice, c->stream));
  }
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  dfree(wsi_d);
  P.on = true;
  return CIQ_OK;
}

void free_precond(PrecondDev& P) {
  dfree(P.l); dfree(P.u); dfree(P.m64);
  P.m64_ready = false;
  for (auto& g : P.g) dfree(g);
  dfree(P.part); dfree(P.h); dfree(P.bpart);
  dfree(P.t1);
}

// fp64 route (precond64.cu): M = P^{-1/2} (K + sigma2 I) P^{-1/2} formed once, in fp64, from fp64
// kernel entries (the given dense K, or COV* + jitter I = K** + jitter I - U U^T for a posterior
// ctx):  H = K U;  A = a K + U diag(g) H^T (= P^{-1/2} K);  H = A U;  M = a A + H diag(g) U^T.
bool use_m64(const ciq_ctx* c) {
  return c->pc.on && !c->pc.matrix_free && !c->pc.m64_failed && !c->sharded;
}

ciq_status ensure_m64(ciq_ctx* c) {
  PrecondDev& P = c->pc;
  if (P.m64_ready) return CIQ_OK;
  const int64_t n = c->op.n, rows = c->row1 - c->row0;
  const int64_t ldm = (n + 7) / 8 * 8;
  const int r2 = P.r2;
  cudaStream_t s = c->stream;
  double* h = nullptr;
  if (dalloc(&P.m64, (size_t)rows * ldm) != cudaSuccess || (r2 > 0 && dalloc(&h, (size_t)n * r2) != cudaSuccess)) {
    cudaGetLastError();
    dfree(P.m64);
    dfree(h);
    P.m64_failed = true;   // too large for this device: the matrix-free route (fp32 floor)
    return CIQ_ERR_OOM;
  }
  P.ldm = ldm;
  CUDA_TRY(c, cudaMemsetAsync(P.m64, 0, (size_t)rows * ldm * 8, s));
  LAUNCH(c, launch_materialize64(c->dev, c->row0, rows, P.m64, ldm, s));
  double* neg = nullptr;
  if (c->post.on) {   // COV* + jitter I = K** + jitter I - U U^T  (eq. thompson_sample)
    const int m = c->post.m;
    std::vector<double> ones((size_t)m, -1.0);
    CUDA_TRY(c, dalloc(&neg, (size_t)m));
    CUDA_TRY(c, cudaMemcpyAsync(neg, ones.data(), (size_t)m * 8, cudaMemcpyHostToDevice, s));
    LAUNCH(c, launch_gemm64(false, true, rows, n, m, c->post.u + c->row0 * m, m, c->post.u, m, neg, 1.0, P.m64, ldm, s));
  }
  if (!P.on) {   // params.fp64 without a preconditioner: M = K (+ sigma^2 I, COV* for a posterior ctx)
    CUDA_TRY(c, cudaStreamSynchronize(s));
    dfree(h);
    dfree(neg);
    P.m64_ready = true;
    return CIQ_OK;
  }
  const double a = P.ad[PW_MHALF];
  const double* g = P.g[PW_MHALF];
  LAUNCH(c, launch_gemm64(false, false, n, r2, n, P.m64, ldm, P.u, r2, nullptr, 0.0, h, r2, s));   // H = K U
  LAUNCH(c, launch_gemm64(false, true, n, n, r2, P.u, r2, h, r2, g, a, P.m64, ldm, s));            // A = P^-1/2 K
  LAUNCH(c, launch_gemm64(false, false, n, r2, n, P.m64, ldm, P.u, r2, nullptr, 0.0, h, r2, s));   // H = A U
  LAUNCH(c, launch_gemm64(false, true, n, n, r2, h, r2, P.u, r2, g, a, P.m64, ldm, s));            // M = A P^-1/2
  CUDA_TRY(c, cudaStreamSynchronize(s));
  dfree(h);
  dfree(neg);
  P.m64_ready = true;
  return CIQ_OK;
}

// out (fp64, rows x tp) = P^p v (fp64) for p = -1/2 (PW_MHALF) or 1/2 (PW_HALF):
// a v + U diag(g) (U^T v), with H = U^T v in c->pc.h.
ciq_status precond_power64(ciq_ctx* c, int which, const double* v, int tp, double* out) {
  PrecondDev& P = c->pc;
  const int64_t n = c->op.n;
  ciq_status st = grow(c, &P.h, &P.h_cap, (size_t)P.r2 * tp);
  if (st != CIQ_OK) return st;
  LAUNCH(c, launch_gemm64(true, false, P.r2, tp, n, P.u, P.r2, v, tp, nullptr, 0.0, P.h, tp, c->stream));
  if (out != v) CUDA_TRY(c, cudaMemcpyAsync(out, v, (size_t)n * tp * 8, cudaMemcpyDeviceToDevice, c->stream));
  LAUNCH(c, launch_gemm64(false, false, n, tp, P.r2, P.u, P.r2, P.h, tp, P.g[which], P.ad[which], out, tp, c->stream));
  return CIQ_OK;
}

void free_post(PostDev& Q) {
  dfree(Q.u); dfree(Q.uf); dfree(Q.mu); dfree(Q.part); dfree(Q.h); dfree(Q.bpart); dfree(Q.t); dfree(Q.f);
  dfree(Q.am_v); dfree(Q.am_i); dfree(Q.idx);
  Q = PostDev();
}

// k(r^2) of the kernel kinds, fp64 (the forms of kval / kfun on the device; reading G11)
double kernel_r2(int kind, double r2, double o2) {
  if (kind == CIQ_OP_RBF) return o2 * std::exp(-0.5 * r2);
  const double r = std::sqrt(r2);
  if (kind == CIQ_OP_MATERN52) return o2 * (1.0 + std::sqrt(5.0) * r + 5.0 / 3.0 * r2) * std::exp(-std::sqrt(5.0) * r);
  return o2 * (1.0 + std::sqrt(3.0) * r) * std::exp(-std::sqrt(3.0) * r);
}

struct EvTimer {
  cudaEvent_t e[5];
  EvTimer() { for (auto& x : e) cudaEventCreate(&x); }
  ~EvTimer() { for (auto& x : e) cudaEventDestroy(x); }
};

// The msMINRES iterations j0+1.. of one solve (a4-a6).  Buffers rotate with period 6 in j (W: j
// mod 3, D: j mod 2) and every kernel reads the iteration state from device memory, so a block of
// `poll_every` (a multiple of 6) iterations is captured once as a CUDA graph (cached in the ctx
// under `key`) and replayed, two blocks in flight while the host checks the stopping flag of the
// older one; iterations past the device-side stopping rule are no-ops.  Without a graph (profiling,
// CIQ_NO_GRAPH, a non-capturable transport) the iterations are enqueued directly.
template <class F>
ciq_status run_iterations(ciq_ctx* c, const ciq_params& p, int j0, uint64_t key_extra, F&& enqueue_iter, Ctrl* hc,
                          bool* replayed) {
  const Scal& sc = c->ws.sc;
  cudaStream_t s = c->stream;
  const int nq = p.Q;
  *replayed = false;
  const bool use_graph = !c->profiling && !experiment_env("CIQ_NO_GRAPH") &&
                         (!c->sharded || c->comm->capturable());
  if (use_graph) {
    const int block = std::max(6, (p.poll_every + 5) / 6 * 6);
    const uint64_t key[6] = {c->buf_gen, (uint64_t)c->ws.tp, (uint64_t)nq, key_extra, (uint64_t)block,
                             (uint64_t)(uintptr_t)c->ws.d};
    if (c->gexec == nullptr || std::memcmp(key, c->gkey, sizeof(key)) != 0) {
      if (c->gexec) { cudaGraphExecDestroy(c->gexec); c->gexec = nullptr; }
      const int64_t l0 = c->launches;
      CUDA_TRY(c, cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      ciq_status cst = CIQ_OK;
      for (int k = 1; k <= block && cst == CIQ_OK; ++k) cst = enqueue_iter(k, nq);
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(s, &g);
      if (cst != CIQ_OK) { if (g) cudaGraphDestroy(g); return cst; }
      CUDA_TRY(c, e);
      e = cudaGraphInstantiate(&c->gexec, g, 0);
      cudaGraphDestroy(g);
      CUDA_TRY(c, e);
      std::memcpy(c->gkey, key, sizeof(key));
      c->graph_nodes = c->launches - l0;
      c->launches = l0;
    } else {
      *replayed = true;
    }
    if (c->ctrl_host == nullptr) CUDA_TRY(c, cudaMallocHost(&c->ctrl_host, 2 * sizeof(Ctrl)));
    int launched = 0, checked = 0;
    cudaEvent_t evp[2];
    cudaEventCreateWithFlags(&evp[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&evp[1], cudaEventDisableTiming);
    auto launch_one = [&]() -> ciq_status {
      const int sl = launched & 1;
      CUDA_TRY(c, cudaGraphLaunch(c->gexec, s));
      c->launches += c->graph_nodes;
      CUDA_TRY(c, cudaMemcpyAsync(&c->ctrl_host[sl], sc.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
      CUDA_TRY(c, cudaEventRecord(evp[sl], s));
      ++launched;
      return CIQ_OK;
    };
    ciq_status st = CIQ_OK;
    for (;;) {
      while ((int64_t)launched * block < p.max_iters - j0 && launched - checked < 2) {
        st = launch_one();
        if (st != CIQ_OK) break;
      }
      if (st != CIQ_OK) break;
      if (cudaEventSynchronize(evp[checked & 1]) != cudaSuccess) {
        st = set_err(c, CIQ_ERR_CUDA, "graph replay failed: %s", cudaGetErrorString(cudaGetLastError()));
        break;
      }
      *hc = c->ctrl_host[checked & 1];
      ++checked;
      if (hc->done || checked == launched) break;
    }
    cudaStreamSynchronize(s);
    cudaEventDestroy(evp[0]);
    cudaEventDestroy(evp[1]);
    return st;
  }
  int j = j0;
  for (;;) {
    for (int k = 0; k < p.poll_every && j < p.max_iters; ++k) {
      ++j;
      ciq_status st = enqueue_iter(j, nq);
      if (st != CIQ_OK) return st;
    }
    CUDA_TRY(c, cudaMemcpyAsync(hc, sc.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    if (hc->done || j >= p.max_iters) break;
  }
  return CIQ_OK;
}

// Stored-basis variant: per column, the MINRES solution of each shifted system in the Lanczos basis,
// y_q = R_q^{-1} phi_q with R_q the Givens-QR factor of [T_J + t_q I; beta_{J+1} e_J^T] (the same
// recurrences as givens_kernel, fp64 on the host), z = sum_q w_q y_q, and Y = sum_j (z_j / nrm_j) W_j.
ciq_status combine_stored_basis(ciq_ctx* c, int J, int hlen, int tp, int cols, int nq, const double* t, const double* w,
                                int64_t rows, float* y) {
  cudaStream_t s = c->stream;
  std::vector<double> h((size_t)4 * hlen * tp + 2 * (size_t)tp);
  CUDA_TRY(c, cudaMemcpyAsync(h.data(), c->bhist, h.size() * 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  const double* ha = h.data();
  const double* hb = ha + (size_t)hlen * tp;
  const double* hn = hb + (size_t)hlen * tp;
  const double* hf = hn + (size_t)hlen * tp;
  const double* n0 = hf + (size_t)hlen * tp;
  const double* f0 = n0 + tp;
  std::vector<float> coef((size_t)J * tp, 0.f);
  std::vector<double> g(J), dl(J + 1), ep(J + 2), ph(J), yq(J + 2), z(J);
  for (int k = 0; k < cols; ++k) {
    if (f0[k] != 0.0) continue;   // zero column: Y = 0
    int m = 0;                    // steps taken before the column froze (its breakdown step included)
    while (m < J && (m == 0 || hf[(size_t)(m - 1) * tp + k] == 0.0)) ++m;
    std::fill(z.begin(), z.end(), 0.0);
    for (int q = 0; q < nq; ++q) {
      double c1 = 1, s1 = 0, c2 = 1, s2 = 0, phib = n0[k];
      for (int i = 0; i < m; ++i) {
        const double a = ha[(size_t)i * tp + k] + t[q];
        const double tb = i >= 1 ? hb[(size_t)(i - 1) * tp + k] : 0.0;   // beta_{i+1} of T (1-based: beta_i)
        const double tbn = hb[(size_t)i * tp + k];
        const double eps = s2 * tb, dp = c2 * tb;
        const double delta = c1 * dp + s1 * a, gbar = -s1 * dp + c1 * a;
        const double gamma = std::hypot(gbar, tbn);
        const double cs = gbar / gamma, sn = tbn / gamma;
        g[i] = gamma;
        dl[i] = delta;
        ep[i] = eps;
        ph[i] = cs * phib;
        phib = -sn * phib;
        c2 = c1; s2 = s1; c1 = cs; s1 = sn;
      }
      // back substitution R y = phi: R column i holds (eps_i, delta_i, gamma_i) at rows i-2, i-1, i
      yq[m] = yq[m + 1] = 0.0;
      for (int i = m - 1; i >= 0; --i) {
        double r = ph[i];
        if (i + 1 < m) r -= dl[i + 1] * yq[i + 1];
        if (i + 2 < m) r -= ep[i + 2] * yq[i + 2];
        yq[i] = r / g[i];
      }
      for (int i = 0; i < m; ++i) z[i] += w[q] * yq[i];
    }
    for (int i = 0; i < m; ++i) {
      const double nrm = i == 0 ? n0[k] : hn[(size_t)(i - 1) * tp + k];
      coef[(size_t)i * tp + k] = (float)(z[i] / nrm);
    }
  }
  CUDA_TRY(c, grow(c, &c->bcoef, &c->bcoef_elems, coef.size()) == CIQ_OK ? cudaSuccess : cudaErrorMemoryAllocation);
  CUDA_TRY(c, cudaMemcpyAsync(c->bcoef, coef.data(), coef.size() * 4, cudaMemcpyHostToDevice, s));
  LAUNCH(c, launch_combine_basis(c->basis, (size_t)rows * tp, J, c->bcoef, rows * tp, tp, y, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));   // coef (host vector) must outlive the copy
  return CIQ_OK;
}

ciq_status apply_fp64(ciq_ctx* c, const float* B, int64_t ldb, int64_t T, float* out, int64_t ldo, ciq_params p,
                      ciq_info* info);
ciq_status apply_nested(ciq_ctx* c, const float* B, int64_t ldb, int64_t T, float* out, int64_t ldo, ciq_params p,
                        ciq_info* info);

}  // namespace

extern "C" {

void ciq_params_default(ciq_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->Q = 8;
  p->max_iters = 400;
  p->tol = 1e-4;
  p->lanczos_iters = 10;
  p->lanczos_cols = 16;
  p->seed = 2;
  p->mode = CIQ_MODE_SQRT;
  p->mvm_impl = CIQ_MVM_AUTO;
  p->poll_every = 6;
  p->breakdown_tol = 1e-6;
  p->fp64 = 0;
  p->stored_basis = 0;
  p->mvm_relax = 1;
}

#ifndef CIQ_SOURCE_HASH
#define CIQ_SOURCE_HASH "unknown"
#endif
const char* ciq_source_hash(void) { return CIQ_SOURCE_HASH; }

const char* ciq_status_string(ciq_status s) {
  switch (s) {
    case CIQ_OK: return "CIQ_OK";
    case CIQ_NOT_CONVERGED: return "CIQ_NOT_CONVERGED";
    case CIQ_ERR_INVALID_ARG: return "CIQ_ERR_INVALID_ARG";
    case CIQ_ERR_DIM: return "CIQ_ERR_DIM";
    case CIQ_ERR_NOT_PD: return "CIQ_ERR_NOT_PD";
    case CIQ_ERR_ELLIPTIC: return "CIQ_ERR_ELLIPTIC";
    case CIQ_ERR_CUDA: return "CIQ_ERR_CUDA";
    case CIQ_ERR_NCCL: return "CIQ_ERR_NCCL";
    case CIQ_ERR_OOM: return "CIQ_ERR_OOM";
  }
  return "CIQ_UNKNOWN";
}

const char* ciq_last_error(const ciq_ctx* c) { return c ? c->err.c_str() : g_init_error.c_str(); }

void ciq_shard_rows(int64_t n, int32_t rank, int32_t world, int64_t* b, int64_t* e) {
  if (world <= 1) { *b = 0; *e = n; return; }
  int64_t per = (n + world - 1) / world;
  per = (per + 127) / 128 * 128;
  *b = std::min<int64_t>(n, (int64_t)rank * per);
  *e = std::min<int64_t>(n, *b + per);
}

ciq_status ciq_quadrature_rule(double lmin, double lmax, int32_t Q, double* t, double* w) {
  if (!t || !w || Q < 1 || Q > CIQ_MAX_Q || !(lmin > 0) || !(lmax > 0)) return CIQ_ERR_INVALID_ARG;
  int r = ciqh::hht_rule(lmin, lmax, Q, t, w);
  return r == 0 ? CIQ_OK : (r == -1 ? CIQ_ERR_INVALID_ARG : CIQ_ERR_ELLIPTIC);
}

ciq_status ciq_nccl_unique_id(void* out128) {
  if (!out128) return CIQ_ERR_INVALID_ARG;
  return nccl_unique_id(out128) ? CIQ_OK : set_err(nullptr, CIQ_ERR_NCCL, "%s", nccl_error());
}

void* ciq_loopback_group_create(int32_t world) { return world >= 1 ? new LoopbackGroup(world) : nullptr; }
void ciq_loopback_group_destroy(void* g) { delete static_cast<LoopbackGroup*>(g); }

ciq_status ciq_tridiag_extremes(const double* alpha, const double* beta, int32_t m, double* emin, double* emax) {
  if (!alpha || (m > 1 && !beta) || m < 1 || !emin || !emax) return CIQ_ERR_INVALID_ARG;
  return ciqh::tridiag_extremes(alpha, beta, m, emin, emax) == 0 ? CIQ_OK : CIQ_ERR_INVALID_ARG;
}

ciq_status ciq_init(ciq_ctx** out, const ciq_operator* op, const ciq_precond* pc, const ciq_comm* comm,
                    void* stream) {
  if (!out || !op) return set_err(nullptr, CIQ_ERR_INVALID_ARG, "null ctx or operator");
  *out = nullptr;
  if (op->n <= 0) return set_err(nullptr, CIQ_ERR_DIM, "n must be > 0");
  if (op->kind < CIQ_OP_DENSE || op->kind > CIQ_OP_SPARSE) return set_err(nullptr, CIQ_ERR_INVALID_ARG, "bad kind");
  if (!(op->diag >= 0)) return set_err(nullptr, CIQ_ERR_INVALID_ARG, "diag must be >= 0");
  if (op->kind == CIQ_OP_SPARSE) {
    if (!op->csr_indptr || !op->csr_indices || !op->csr_values || op->nnz < 0)
      return set_err(nullptr, CIQ_ERR_INVALID_ARG, "sparse operator needs csr_indptr / csr_indices / csr_values");
    if (pc) return set_err(nullptr, CIQ_ERR_INVALID_ARG, "sparse operator: no preconditioner (not supported)");
  } else if (op->kind == CIQ_OP_DENSE) {
    if (!op->K) return set_err(nullptr, CIQ_ERR_INVALID_ARG, "dense operator needs K");
    if (op->ldk < op->n) return set_err(nullptr, CIQ_ERR_DIM, "ldk < n");
  } else {
    if (!op->X || !op->lengthscale) return set_err(nullptr, CIQ_ERR_INVALID_ARG, "kernel operator needs X and lengthscale");
    if (op->d < 1 || op->d > 16) return set_err(nullptr, CIQ_ERR_DIM, "d must be in [1, 16]");
    if (op->ldx < op->d) return set_err(nullptr, CIQ_ERR_DIM, "ldx < d");
    if (!(op->outputscale > 0)) return set_err(nullptr, CIQ_ERR_INVALID_ARG, "outputscale must be > 0");
    for (int k = 0; k < (op->ard ? op->d : 1); ++k)
      if (!(op->lengthscale[k] > 0)) return set_err(nullptr, CIQ_ERR_INVALID_ARG, "lengthscale must be > 0");
  }
  if (pc && pc->kind == 1) {
    if (pc->block < 1) return set_err(nullptr, CIQ_ERR_DIM, "block-Jacobi preconditioner: block must be >= 1");
    if (comm) return set_err(nullptr, CIQ_ERR_INVALID_ARG, "block-Jacobi preconditioner: single GPU only");
  } else if (pc) {
    if (pc->kind != 0) return set_err(nullptr, CIQ_ERR_INVALID_ARG, "bad preconditioner kind");
    if (!pc->L || pc->rank < 1 || pc->ldl < pc->rank) return set_err(nullptr, CIQ_ERR_DIM, "bad preconditioner L / rank / ldl");
    if (!(pc->sigma2 > 0)) return set_err(nullptr, CIQ_ERR_INVALID_ARG, "preconditioner sigma2 must be > 0 (S:425)");
    if (pc->rank > 2048) return set_err(nullptr, CIQ_ERR_DIM, "preconditioner rank > 2048");
  }
  if (comm && comm->world >= 1) {
    if (comm->rank < 0 || comm->rank >= comm->world) return set_err(nullptr, CIQ_ERR_INVALID_ARG, "bad rank");
    if (!comm->loopback_group && !comm->nccl_unique_id)
      return set_err(nullptr, CIQ_ERR_INVALID_ARG, "row sharding needs an NCCL unique id or a loopback group");
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return set_err(nullptr, CIQ_ERR_CUDA, "no CUDA device");
  }
  ciq_ctx* c = new ciq_ctx();
  c->op = *op;
  c->user_stream = reinterpret_cast<cudaStream_t>(stream);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return set_err(nullptr, CIQ_ERR_CUDA, "stream creation failed");
  }
  if (comm && comm->world >= 1) {
    c->sharded = true;
    c->rank = comm->rank;
    c->world = comm->world;
    ciq_shard_rows(op->n, c->rank, c->world, &c->row0, &c->row1);
    c->per = (op->n + c->world - 1) / c->world;
    c->per = (c->per + 127) / 128 * 128;
    c->nfull = c->per * c->world;
    c->comm = comm->loopback_group
                  ? make_loopback_comm(static_cast<LoopbackGroup*>(comm->loopback_group), c->rank)
                  : make_nccl_comm(c->rank, c->world, comm->nccl_unique_id);
    if (c->comm == nullptr) {
      delete c;
      return set_err(nullptr, CIQ_ERR_NCCL, "communicator creation failed: %s", nccl_error());
    }
  } else {
    c->row0 = 0;
    c->row1 = op->n;
    c->per = op->n;
    c->nfull = op->n;
  }
  OpDev& dv = c->dev;
  dv.kind = op->kind;
  dv.n = op->n;
  dv.diag = op->diag;
  dv.o2 = op->outputscale;
  ciq_status st = CIQ_OK;
  if (op->kind == CIQ_OP_SPARSE) {
    // CSR of this rank's row block [row0, row1) (all rows on one GPU), copied to the device
    const int64_t lrows = c->row1 - c->row0, nnz = op->nnz;
    const bool dp = is_device_ptr(op->csr_indptr);
    const cudaMemcpyKind mk = dp ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (cudaMalloc(&c->csr_rp, (size_t)(lrows + 1) * 8) != cudaSuccess ||
        cudaMalloc(&c->csr_ci, (size_t)std::max<int64_t>(1, nnz) * 4) != cudaSuccess ||
        cudaMalloc(&c->csr_cv, (size_t)std::max<int64_t>(1, nnz) * 4) != cudaSuccess) {
      st = CIQ_ERR_OOM; goto fail;
    }
    if (cudaMemcpy(c->csr_rp, op->csr_indptr, (size_t)(lrows + 1) * 8, mk) != cudaSuccess ||
        (nnz > 0 && cudaMemcpy(c->csr_ci, op->csr_indices, (size_t)nnz * 4,
                               is_device_ptr(op->csr_indices) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice) != cudaSuccess) ||
        (nnz > 0 && cudaMemcpy(c->csr_cv, op->csr_values, (size_t)nnz * 4,
                               is_device_ptr(op->csr_values) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice) != cudaSuccess)) {
      st = CIQ_ERR_CUDA; goto fail;
    }
    dv.rp = c->csr_rp;
    dv.ci = c->csr_ci;
    dv.cv = c->csr_cv;
  } else if (op->kind == CIQ_OP_DENSE) {
    // K holds this rank's row block [row0, row1) (all rows on one GPU); the MVM kernels index it
    // by the global row, hence the pointer shift by -row0 rows.
    const int64_t lrows = c->row1 - c->row0;
    if (is_device_ptr(op->K)) {
      dv.k = op->K - c->row0 * op->ldk;
      dv.ldk = op->ldk;
    } else {
      if (cudaMalloc(&c->kcopy, (size_t)lrows * op->n * 4) != cudaSuccess) { st = CIQ_ERR_OOM; goto fail; }
      if (cudaMemcpy2D(c->kcopy, (size_t)op->n * 4, op->K, (size_t)op->ldk * 4, (size_t)op->n * 4, (size_t)lrows,
                       cudaMemcpyHostToDevice) != cudaSuccess) { st = CIQ_ERR_CUDA; goto fail; }
      dv.k = c->kcopy - c->row0 * op->n;
      dv.ldk = op->n;
    }
    if (!build_dense_planes(c)) cudaGetLastError();  // tensor-core dense path unavailable -> SIMT
  } else {
    const int64_t n = op->n, d = op->d;
    std::vector<float> xh((size_t)n * d);
    if (is_device_ptr(op->X)) {
      if (cudaMemcpy2D(xh.data(), d * 4, op->X, op->ldx * 4, d * 4, n, cudaMemcpyDeviceToHost) != cudaSuccess) {
        st = CIQ_ERR_CUDA; goto fail;
      }
    } else {
      for (int64_t i = 0; i < n; ++i) std::memcpy(&xh[i * d], op->X + i * op->ldx, d * 4);
    }
    // fp64 copy first: x / l of the caller's fp32 values without an fp32 rounding of the quotient
    // (the fp64 materialised route, precond64.cu, must see the same points as an fp64 reference)
    std::vector<double> xh64((size_t)n * d);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = 0; k < d; ++k) xh64[i * d + k] = (double)xh[i * d + k] / (double)op->lengthscale[op->ard ? k : 0];
    for (int64_t i = 0; i < n; ++i)
      for (int64_t k = 0; k < d; ++k) xh[i * d + k] /= op->lengthscale[op->ard ? k : 0];
    for (int64_t k = 0; k < d; ++k) c->ls.push_back(op->lengthscale[op->ard ? k : 0]);
    if (cudaMalloc(&c->xs, (size_t)n * d * 4) != cudaSuccess) { st = CIQ_ERR_OOM; goto fail; }
    if (cudaMemcpy(c->xs, xh.data(), (size_t)n * d * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
      st = CIQ_ERR_CUDA; goto fail;
    }
    dv.xs = c->xs;
    if (cudaMalloc(&c->xs64, (size_t)n * d * 8) != cudaSuccess) { st = CIQ_ERR_OOM; goto fail; }
    if (cudaMemcpy(c->xs64, xh64.data(), (size_t)n * d * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
      st = CIQ_ERR_CUDA; goto fail;
    }
    dv.xs64 = c->xs64;
    dv.d = (int)d;
    c->tc_ok = build_tc_features(c, xh);
  }
  if (pc && pc->kind == 1) {   // nested CIQ route: set up lazily (ensure_nested) at the first apply
    c->nest.on = true;
    c->nest.block = std::min<int64_t>(pc->block, op->n);
    c->has_precond = true;
  } else if (pc) {
    PrecondDev& P = c->pc;
    P.rank = (int)pc->rank;
    P.sigma2 = pc->sigma2;
    P.matrix_free = pc->matrix_free != 0;
    // L: this rank's row block [row0, row1) (all N rows on one GPU), like B
    const int64_t lrows = c->row1 - c->row0;
    if (cudaMalloc(&P.l, (size_t)lrows * P.rank * 4) != cudaSuccess) { st = CIQ_ERR_OOM; goto fail; }
    const cudaMemcpyKind kind = is_device_ptr(pc->L) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    if (cudaMemcpy2D(P.l, (size_t)P.rank * 4, pc->L, (size_t)pc->ldl * 4, (size_t)P.rank * 4, (size_t)lrows, kind) !=
        cudaSuccess) { st = CIQ_ERR_CUDA; goto fail; }
    st = build_precond(c);
    if (st != CIQ_OK) {
      g_init_error = c->err;
      ciq_free(c);
      return st;
    }
    c->has_precond = true;
  }
  *out = c;
  return CIQ_OK;
fail:
  set_err(nullptr, st, "ciq_init: device allocation/copy failed: %s", cudaGetErrorString(cudaGetLastError()));
  ciq_free(c);
  return st;
}

void ciq_free(ciq_ctx* c) {
  if (!c) return;
  if (c->stream) { cudaStreamSynchronize(c->stream); cudaStreamDestroy(c->stream); }
  if (c->join_ev) cudaEventDestroy(c->join_ev);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->ctrl_host) cudaFreeHost(c->ctrl_host);
  for (auto& t : c->timed) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  free_workspace(c->ws);
  free_lambda(c->lw);
  dfree(c->xs);
  dfree(c->xs64);
  dfree(c->nest.k64);
  dfree(c->nest.pinv);
  dfree(c->nest.work);
  dfree(c->kcopy);
  dfree(c->basis);
  dfree(c->bhist);
  dfree(c->bcoef);
  dfree(c->csr_rp);
  dfree(c->csr_ci);
  dfree(c->csr_cv);
  dfree(c->staging);
  dfree(c->kplanes);
  dfree(c->feat_a); dfree(c->feat_b); dfree(c->planes); dfree(c->inv_scale); dfree(c->psplit);
  dfree(c->stash); dfree(c->hist);
  dfree(c->vjp_xb); dfree(c->vjp_xv); dfree(c->vjp_y); dfree(c->vjp_g); dfree(c->vjp_w);
  dfree(c->apart_tc); dfree(c->cta_part); dfree(c->ticket);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->s2) cudaStreamDestroy(c->s2);
  dfree(c->sym_units); dfree(c->sym_base); dfree(c->sym_part);
  free_precond(c->pc);
  free_post(c->post);
  dfree(c->gsum);
  dfree(c->tsum);
  delete c->comm;
  delete c;
}

ciq_status ciq_pivoted_cholesky(ciq_ctx* c, int32_t rank, float* L, int64_t ldl) {
  if (!c || !L) return CIQ_ERR_INVALID_ARG;
  if (c->sharded)   // the pivot search and the kernel columns span all N rows
    return set_err(c, CIQ_ERR_INVALID_ARG, "ciq_pivoted_cholesky: single-GPU contexts only (not row-sharded)");
  if (c->op.kind == CIQ_OP_SPARSE)
    return set_err(c, CIQ_ERR_INVALID_ARG, "ciq_pivoted_cholesky: kernel or dense operators only");
  const int64_t n = c->op.n;
  if (rank < 1 || rank > n || ldl < rank) return set_err(c, CIQ_ERR_DIM, "bad rank / ldl");
  if (join_user_stream(c) != CIQ_OK) return CIQ_ERR_CUDA;
  float* ld = nullptr;
  double *diag = nullptr, *lcol = nullptr, *pivval = nullptr;
  int* piv = nullptr;
  CUDA_TRY(c, dalloc(&ld, (size_t)n * rank));
  CUDA_TRY(c, dalloc(&diag, (size_t)n));
  CUDA_TRY(c, dalloc(&lcol, (size_t)n * rank));
  CUDA_TRY(c, dalloc(&pivval, (size_t)rank));
  CUDA_TRY(c, dalloc(&piv, (size_t)rank));
  CUDA_TRY(c, cudaMemsetAsync(ld, 0, (size_t)n * rank * 4, c->stream));
  LAUNCH(c, launch_pivchol(c->dev, rank, ld, rank, diag, lcol, piv, pivval, c->post.on ? c->post.u : nullptr,
                           c->post.m, c->stream));
  ciq_status st = store_rows(c, ld, rank, n, rank, L, ldl);
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  dfree(ld); dfree(diag); dfree(lcol); dfree(pivval); dfree(piv);
  return st;
}

ciq_status ciq_matvec(ciq_ctx* c, const float* V, int64_t ldv, int64_t T, float* out, int64_t ldo, int32_t impl) {
  if (!c || !V || !out) return CIQ_ERR_INVALID_ARG;
  if (T <= 0 || ldv < T || ldo < T) return set_err(c, CIQ_ERR_DIM, "bad T / leading dimension");
  const int tp = round16(T);
  if (ensure_workspace(c, tp, std::max(1, c->ws.nq)) != CIQ_OK) return CIQ_ERR_OOM;
  if (join_user_stream(c) != CIQ_OK) return CIQ_ERR_CUDA;
  Workspace& ws = c->ws;
  ciq_status st = load_rows(c, V, ldv, c->op.n, (int)T, ws.w[0], tp);
  if (st != CIQ_OK) return st;
  LAUNCH(c, launch_colsq_partials(ws.w[0], c->op.n, tp, ws.bpart, c->stream));
  LAUNCH(c, launch_reduce_cols(ws.bpart, rowblocks(c->op.n, tp), tp, ws.colsq, 1, c->stream));
  st = run_mvm(c, ws.w[0], tp, ws.p, nullptr, nullptr, impl, ws.colsq);
  if (st != CIQ_OK) return st;
  st = store_rows(c, ws.p, tp, c->row1 - c->row0, (int)T, out, ldo);
  if (st != CIQ_OK) return st;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return CIQ_OK;
}

ciq_status ciq_vjp(ciq_ctx* c, const float* B, int64_t ldb, const float* V, int64_t ldv, int64_t T,
                   const ciq_params* params, float* G, int64_t ldg, ciq_info* info) {
  if (!c || !B || !V || !G) return CIQ_ERR_INVALID_ARG;
  if (c->sharded || c->has_precond)
    return set_err(c, CIQ_ERR_INVALID_ARG, "ciq_vjp: single GPU, unpreconditioned operators only");
  const int64_t n = c->op.n;
  if (T <= 0 || ldv < T || ldb < T || ldg < n) return set_err(c, CIQ_ERR_DIM, "bad T / leading dimension");
  ciq_params p;
  if (params) p = *params; else ciq_params_default(&p);
  const int nq = p.Q;
  if (nq < 1 || nq > CIQ_MAX_Q) return set_err(c, CIQ_ERR_INVALID_ARG, "Q must be in [1, %d]", CIQ_MAX_Q);
  ciq_status gs = grow(c, &c->vjp_xb, &c->vjp_xb_cap, (size_t)nq * n * T);
  if (gs == CIQ_OK) gs = grow(c, &c->vjp_xv, &c->vjp_xv_cap, (size_t)nq * n * T);
  if (gs == CIQ_OK) gs = grow(c, &c->vjp_y, &c->vjp_y_cap, (size_t)n * T);
  if (gs == CIQ_OK) gs = grow(c, &c->vjp_w, &c->vjp_w_cap, (size_t)nq);
  if (gs != CIQ_OK) return gs;
  float *xb = c->vjp_xb, *xv = c->vjp_xv, *yb = c->vjp_y;
  double* wd = c->vjp_w;
  // forward: x_q(b) with the estimated (or given) rule
  p.mode = CIQ_MODE_INVSQRT;
  p.keep_shift_solutions = 1;
  p.shift_solutions = xb;
  ciq_info i1{};
  ciq_status st = ciq_apply(c, B, ldb, T, yb, T, &p, &i1);
  if (st != CIQ_OK && st != CIQ_NOT_CONVERGED) return st;
  // backward: x_q(v) with the same rule ("another call to the msMINRES algorithm")
  double t[CIQ_MAX_Q], w[CIQ_MAX_Q];
  for (int q = 0; q < nq; ++q) { t[q] = i1.t[q]; w[q] = i1.w[q]; }
  p.t = t;
  p.w = w;
  p.Q = nq;
  p.lanczos_reuse = 0;
  p.shift_solutions = xv;
  ciq_info i2{};
  ciq_status st2 = ciq_apply(c, V, ldv, T, yb, T, &p, &i2);
  if (st2 != CIQ_OK && st2 != CIQ_NOT_CONVERGED) return st2;
  CUDA_TRY(c, cudaMemcpyAsync(wd, w, nq * 8, cudaMemcpyHostToDevice, c->stream));
  float* gdev = G;
  float* gtmp = nullptr;
  const bool gdevice = is_device_ptr(G);
  if (!gdevice) {
    ciq_status g2 = grow(c, &c->vjp_g, &c->vjp_g_cap, (size_t)n * n);
    if (g2 != CIQ_OK) return g2;
    gtmp = c->vjp_g;
    gdev = gtmp;
  }
  const int64_t ld = gdevice ? ldg : n;
  LAUNCH(c, launch_vjp_dense(xb, xv, wd, nq, n, (int)T, (int)T, gdev, ld, c->stream));
  if (!gdevice) {
    CUDA_TRY(c, cudaMemcpy2DAsync(G, (size_t)ldg * 4, gtmp, (size_t)n * 4, (size_t)n * 4, (size_t)n,
                                  cudaMemcpyDeviceToHost, c->stream));
  }
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (info) {
    *info = i1;
    info->mvms = i1.mvms + i2.mvms;
  }
  return (st == CIQ_OK && st2 == CIQ_OK) ? CIQ_OK : CIQ_NOT_CONVERGED;
}

ciq_status ciq_hyper_grad(ciq_ctx* c, const float* B, int64_t ldb, const float* V, int64_t ldv, int64_t T,
                          const ciq_params* params, double* grad, ciq_info* info) {
  if (!c || !B || !V || !grad) return CIQ_ERR_INVALID_ARG;
  if (c->sharded || c->has_precond || c->post.on || !is_kernel_op(c) || c->op.ard)
    return set_err(c, CIQ_ERR_INVALID_ARG,
                   "ciq_hyper_grad: single-GPU, unpreconditioned, isotropic kernel operators only");
  const int64_t n = c->op.n;
  if (T <= 0 || ldv < T || ldb < T) return set_err(c, CIQ_ERR_DIM, "bad T / leading dimension");
  ciq_params p;
  if (params) p = *params; else ciq_params_default(&p);
  const int nq = p.Q;
  if (nq < 1 || nq > CIQ_MAX_Q) return set_err(c, CIQ_ERR_INVALID_ARG, "Q must be in [1, %d]", CIQ_MAX_Q);
  ciq_status gs = grow(c, &c->vjp_xb, &c->vjp_xb_cap, (size_t)nq * n * T);
  if (gs == CIQ_OK) gs = grow(c, &c->vjp_xv, &c->vjp_xv_cap, (size_t)nq * n * T);
  if (gs == CIQ_OK) gs = grow(c, &c->vjp_y, &c->vjp_y_cap, (size_t)n * T);
  if (gs != CIQ_OK) return gs;
  float *xb = c->vjp_xb, *xv = c->vjp_xv, *yb = c->vjp_y;
  // the shifted solves x_q(b) (forward) and x_q(v) (same rule), as ciq_vjp
  p.mode = CIQ_MODE_INVSQRT;
  p.keep_shift_solutions = 1;
  p.shift_solutions = xb;
  ciq_info i1{};
  ciq_status st = ciq_apply(c, B, ldb, T, yb, T, &p, &i1);
  if (st != CIQ_OK && st != CIQ_NOT_CONVERGED) return st;
  double t[CIQ_MAX_Q], w[CIQ_MAX_Q];
  for (int q = 0; q < nq; ++q) { t[q] = i1.t[q]; w[q] = i1.w[q]; }
  p.t = t;
  p.w = w;
  p.Q = nq;
  p.lanczos_reuse = 0;
  p.shift_solutions = xv;
  ciq_info i2{};
  ciq_status st2 = ciq_apply(c, V, ldv, T, yb, T, &p, &i2);
  if (st2 != CIQ_OK && st2 != CIQ_NOT_CONVERGED) return st2;
  // dL/dtheta = -sum_q w_q sum_c x_q(v_c)^T (dK/dtheta) x_q(b_c)  (G of eq. ciq_deriv is symmetric
  // and dK/dtheta too): one dK/dl MVM and one K MVM per shift, on the matrix-free kernels
  const int tp = round16(T);
  if (ensure_workspace(c, tp, std::max(1, c->ws.nq)) != CIQ_OK) return CIQ_ERR_OOM;
  Workspace& ws = c->ws;
  ciq_status sg = grow(c, &c->gsum, &c->gsum_cap, (size_t)3 * dot_rows_blocks());
  if (sg != CIQ_OK) return sg;
  std::vector<double> hpart((size_t)3 * dot_rows_blocks());
  double dl = 0.0, dk = 0.0, dd = 0.0;
  for (int q = 0; q < nq; ++q) {
    const float* xbq = xb + (size_t)q * n * T;
    const float* xvq = xv + (size_t)q * n * T;
    ciq_status s3 = load_rows(c, xbq, T, n, (int)T, ws.w[0], tp);
    if (s3 != CIQ_OK) return s3;
    LAUNCH(c, launch_colsq_partials(ws.w[0], n, tp, ws.bpart, c->stream));
    LAUNCH(c, launch_reduce_cols(ws.bpart, rowblocks(n, tp), tp, ws.colsq, 1, c->stream));
    c->deriv = true;
    s3 = run_mvm(c, ws.w[0], tp, ws.p, nullptr, nullptr, p.mvm_impl, ws.colsq);
    c->deriv = false;
    if (s3 != CIQ_OK) return s3;
    LAUNCH(c, launch_dot_rows(xvq, T, ws.p, tp, n, (int)T, c->gsum, c->stream));
    s3 = run_mvm(c, ws.w[0], tp, ws.p, nullptr, nullptr, p.mvm_impl, ws.colsq);
    if (s3 != CIQ_OK) return s3;
    LAUNCH(c, launch_dot_rows(xvq, T, ws.p, tp, n, (int)T, c->gsum + dot_rows_blocks(), c->stream));
    LAUNCH(c, launch_dot_rows(xvq, T, xbq, T, n, (int)T, c->gsum + 2 * dot_rows_blocks(), c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(hpart.data(), c->gsum, hpart.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    double s_l = 0.0, s_k = 0.0, s_d = 0.0;   // fixed-order sums of the block partials
    for (int b = 0; b < dot_rows_blocks(); ++b) {
      s_l += hpart[b];
      s_k += hpart[dot_rows_blocks() + b];
      s_d += hpart[2 * dot_rows_blocks() + b];
    }
    dl += w[q] * s_l;
    dk += w[q] * s_k;
    dd += w[q] * s_d;
  }
  const double o2 = c->op.outputscale, s2 = c->op.diag;
  grad[0] = -dl;                         // dL/dl
  grad[1] = -(dk - s2 * dd) / o2;        // dL/d(o^2): dK/d(o^2) = (K - sigma^2 I) / o^2
  grad[2] = -dd;                         // dL/dsigma^2: dK/dsigma^2 = I
  if (info) {
    *info = i1;
    info->mvms = i1.mvms + i2.mvms + 2 * nq;
  }
  return (st == CIQ_OK && st2 == CIQ_OK) ? CIQ_OK : CIQ_NOT_CONVERGED;
}

ciq_status ciq_set_posterior(ciq_ctx* c, const float* Xt, int64_t ldxt, int64_t m, const float* y, double noise) {
  if (!c || !Xt) return CIQ_ERR_INVALID_ARG;
  if (!is_kernel_op(c) || c->sharded)
    return set_err(c, CIQ_ERR_INVALID_ARG, "ciq_set_posterior: single-GPU kernel operators only");
  const int d = (int)c->op.d;
  if (m < 1 || m > 4096 || ldxt < d) return set_err(c, CIQ_ERR_DIM, "ciq_set_posterior: need 1 <= m <= 4096, ldxt >= d");
  if (!(noise > 0)) return set_err(c, CIQ_ERR_INVALID_ARG, "ciq_set_posterior: noise must be > 0");
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return set_err(c, CIQ_ERR_CUDA, "stream error");
  // training inputs / targets to the host, scaled by the ctx's lengthscales
  std::vector<float> xt((size_t)m * d), yh((size_t)m, 0.f);
  if (is_device_ptr(Xt)) {
    CUDA_TRY(c, cudaMemcpy2D(xt.data(), (size_t)d * 4, Xt, (size_t)ldxt * 4, (size_t)d * 4, (size_t)m,
                             cudaMemcpyDeviceToHost));
  } else {
    for (int64_t i = 0; i < m; ++i) std::memcpy(&xt[i * d], Xt + i * ldxt, (size_t)d * 4);
  }
  if (y) {
    if (is_device_ptr(y)) CUDA_TRY(c, cudaMemcpy(yh.data(), y, (size_t)m * 4, cudaMemcpyDeviceToHost));
    else std::memcpy(yh.data(), y, (size_t)m * 4);
  }
  for (int64_t i = 0; i < m; ++i)
    for (int k = 0; k < d; ++k) xt[i * d + k] = (float)((double)xt[i * d + k] / c->ls[k]);
  // Kxx + noise I = L L^T (fp64 Cholesky, host), L^{-1} by forward substitution, z = L^{-1} y
  const double o2 = c->op.outputscale;
  std::vector<double> l((size_t)m * m, 0.0), linv((size_t)m * m, 0.0), z((size_t)m, 0.0);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j <= i; ++j) {
      double r2 = 0.0;
      for (int k = 0; k < d; ++k) {
        const double df = (double)xt[i * d + k] - (double)xt[j * d + k];
        r2 += df * df;
      }
      l[i * m + j] = kernel_r2(c->op.kind, r2, o2) + (i == j ? noise : 0.0);
    }
  for (int64_t j = 0; j < m; ++j) {
    double s = l[j * m + j];
    for (int64_t k = 0; k < j; ++k) s -= l[j * m + k] * l[j * m + k];
    if (!(s > 0)) return set_err(c, CIQ_ERR_NOT_PD, "ciq_set_posterior: Kxx + noise I not positive definite (pivot %lld)", (long long)j);
    const double ljj = std::sqrt(s);
    l[j * m + j] = ljj;
    for (int64_t i = j + 1; i < m; ++i) {
      double t = l[i * m + j];
      for (int64_t k = 0; k < j; ++k) t -= l[i * m + k] * l[j * m + k];
      l[i * m + j] = t / ljj;
    }
  }
  for (int64_t j = 0; j < m; ++j)       // column j of L^{-1}
    for (int64_t i = j; i < m; ++i) {
      double t = (i == j) ? 1.0 : 0.0;
      for (int64_t k = j; k < i; ++k) t -= l[i * m + k] * linv[k * m + j];
      linv[i * m + j] = t / l[i * m + i];
    }
  for (int64_t i = 0; i < m; ++i) {
    double t = 0.0;
    for (int64_t k = 0; k <= i; ++k) t += linv[i * m + k] * (double)yh[k];
    z[i] = t;
  }
  free_post(c->post);
  PostDev& Q = c->post;
  Q.m = (int)m;
  const int64_t n = c->op.n;
  float* xt_d = nullptr;
  double *linv_d = nullptr, *z_d = nullptr;
  CUDA_TRY(c, dalloc(&Q.u, (size_t)n * m));
  CUDA_TRY(c, dalloc(&Q.uf, (size_t)n * m));
  CUDA_TRY(c, dalloc(&Q.mu, (size_t)n));
  CUDA_TRY(c, dalloc(&xt_d, (size_t)m * d));
  CUDA_TRY(c, dalloc(&linv_d, (size_t)m * m));
  CUDA_TRY(c, dalloc(&z_d, (size_t)m));
  CUDA_TRY(c, cudaMemcpy(xt_d, xt.data(), (size_t)m * d * 4, cudaMemcpyHostToDevice));
  CUDA_TRY(c, cudaMemcpy(linv_d, linv.data(), (size_t)m * m * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(c, cudaMemcpy(z_d, z.data(), (size_t)m * 8, cudaMemcpyHostToDevice));
  LAUNCH(c, launch_build_u(c->op.kind, c->xs, xt_d, d, n, (int)m, o2, linv_d, Q.u, Q.uf, c->stream));
  LAUNCH(c, launch_post_mean(Q.u, z_d, n, (int)m, Q.mu, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  dfree(xt_d); dfree(linv_d); dfree(z_d);
  Q.on = true;
  ++c->buf_gen;   // the captured iteration graph must now include the downdate
  if (c->pc.m64_ready) {   // the fp64 route's M was formed from the prior operator: rebuild lazily
    dfree(c->pc.m64);
    c->pc.m64_ready = false;
  }
  return CIQ_OK;
}

ciq_status ciq_thompson(ciq_ctx* c, const float* eps, int64_t ld_eps, int64_t T, const ciq_params* params,
                        int64_t* idx, float* samples, int64_t ld_samples, ciq_info* info) {
  if (!c || !eps || !idx) return CIQ_ERR_INVALID_ARG;
  if (!c->post.on) return set_err(c, CIQ_ERR_INVALID_ARG, "ciq_thompson: call ciq_set_posterior first");
  if (T <= 0 || ld_eps < T || (samples && ld_samples < T)) return set_err(c, CIQ_ERR_DIM, "bad T / leading dimension");
  ciq_params p;
  if (params) p = *params; else ciq_params_default(&p);
  p.mode = CIQ_MODE_SQRT;
  PostDev& Q = c->post;
  const int64_t n = c->op.n;
  const bool sdev = samples && is_device_ptr(samples);
  float* f = samples;
  int64_t ldf = ld_samples;
  ciq_status st;
  if (!sdev) {
    st = grow(c, &Q.f, &Q.f_cap, (size_t)n * T);
    if (st != CIQ_OK) return st;
    f = Q.f;
    ldf = T;
  }
  ciq_status sa = ciq_apply(c, eps, ld_eps, T, f, ldf, &p, info);   // f = COV*^{1/2} eps
  if (sa != CIQ_OK && sa != CIQ_NOT_CONVERGED) return sa;
  const size_t nb = (size_t)argmin_blocks(n);
  st = grow(c, &Q.am_v, &Q.am_v_cap, nb * T);
  if (st == CIQ_OK) st = grow(c, &Q.am_i, &Q.am_i_cap, nb * T);
  if (st == CIQ_OK) st = grow(c, &Q.idx, &Q.idx_cap, (size_t)T);
  if (st != CIQ_OK) return st;
  LAUNCH(c, launch_add_mean_argmin(f, ldf, n, (int)T, Q.mu, Q.am_v, Q.am_i, Q.idx, c->stream));
  CUDA_TRY(c, cudaMemcpyAsync(idx, Q.idx, (size_t)T * 8, cudaMemcpyDefault, c->stream));
  if (samples && !sdev)
    CUDA_TRY(c, cudaMemcpy2DAsync(samples, (size_t)ld_samples * 4, f, (size_t)T * 4, (size_t)T * 4, (size_t)n,
                                  cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return sa;
}

ciq_status ciq_apply(ciq_ctx* c, const float* B, int64_t ldb, int64_t T, float* out, int64_t ldo,
                     const ciq_params* pp, ciq_info* info) {
  if (!c) return set_err(nullptr, CIQ_ERR_INVALID_ARG, "null ctx");
  if (!B || !out) return set_err(c, CIQ_ERR_INVALID_ARG, "null B or out");
  ciq_params p;
  if (pp) p = *pp; else ciq_params_default(&p);
  if (p.Q < 1 || p.Q > CIQ_MAX_Q) return set_err(c, CIQ_ERR_INVALID_ARG, "Q must be in [1, %d]", CIQ_MAX_Q);
  if (!(p.tol >= 0) || p.max_iters < 1) return set_err(c, CIQ_ERR_INVALID_ARG, "tol must be >= 0, max_iters >= 1");
  if (p.mode < CIQ_MODE_SQRT || p.mode > CIQ_MODE_WHITEN) return set_err(c, CIQ_ERR_INVALID_ARG, "bad mode");
  if (T <= 0 || ldb < T || ldo < T) return set_err(c, CIQ_ERR_DIM, "bad T / leading dimension");
  if ((p.t == nullptr) != (p.w == nullptr)) return set_err(c, CIQ_ERR_INVALID_ARG, "t and w must be given together");
  if (p.poll_every < 1) p.poll_every = 6;
  if (!(p.breakdown_tol > 0)) p.breakdown_tol = 1e-6;
  c->launches = 0;
  c->err.clear();
  c->profiling = p.profile_kernels != 0;
  for (auto& t : c->timed) { c->event_pool.push_back(t.a); c->event_pool.push_back(t.b); }
  c->timed.clear();
  if (c->nest.on) {   // block-Jacobi P: P^{-1}-only recurrence + nested CIQ for P^{1/2} B (App. A)
    if (c->post.on) return set_err(c, CIQ_ERR_INVALID_ARG, "block-Jacobi preconditioner: not on a posterior ctx");
    return apply_nested(c, B, ldb, T, out, ldo, p, info);
  }
  if (p.fp64 && !c->pc.on) {   // accuracy mode: K materialised in fp64, fp64 MVMs and vectors
    if (c->sharded || !is_kernel_op(c))
      return set_err(c, CIQ_ERR_INVALID_ARG, "params.fp64: single-GPU kernel operators only");
    const ciq_status sm = ensure_m64(c);
    if (sm != CIQ_OK) return set_err(c, sm, "params.fp64: N^2 doubles do not fit in device memory");
    c->fp64_active = true;
    const ciq_status sa = apply_fp64(c, B, ldb, T, out, ldo, p, info);
    c->fp64_active = false;
    return sa;
  }
  if (use_m64(c)) {   // preconditioned: the fp64 route when M fits in device memory (precond64.cu)
    const ciq_status sm = ensure_m64(c);
    c->fp64_active = sm == CIQ_OK;
    const ciq_status sa = sm == CIQ_OK ? apply_fp64(c, B, ldb, T, out, ldo, p, info) : sm;
    c->fp64_active = false;
    if (sm == CIQ_OK) return sa;
    if (sm != CIQ_ERR_OOM) return sm;
    c->err.clear();   // M does not fit: the matrix-free route below
  }
  const int tp = round16(T);
  const int nq = p.Q;
  const int64_t n = c->op.n;
  const int64_t rows = c->row1 - c->row0;
  cudaStream_t s = c->stream;
  ciq_status st = ensure_workspace(c, tp, nq);
  if (st != CIQ_OK) return st;
  Workspace& ws = c->ws;
  const Scal& sc = ws.sc;
  st = join_user_stream(c);
  if (st != CIQ_OK) return st;
  EvTimer ev;
  CUDA_TRY(c, cudaEventRecord(ev.e[0], s));

  // a1: RHS -> W[1] (= nrm_1 v_1 with nrm_1 = ||b||), zero W_prev, Y, D.  With row sharding B is
  // this rank's row block; the full first Lanczos block is all-gathered.
  for (auto& wb : ws.w) CUDA_TRY(c, cudaMemsetAsync(wb, 0, (size_t)c->nfull * tp * 4, s));
  st = load_rows(c, B, ldb, rows, (int)T, ws.w[1] + c->row0 * tp, tp);
  if (st != CIQ_OK) return st;
  st = allgather_rows(c, ws.w[1], tp);
  if (st != CIQ_OK) return st;
  st = grow(c, &c->tsum, &c->tsum_cap, (size_t)2 * tp);
  if (st != CIQ_OK) return st;
  double* tsum_a = c->tsum;        // world > 1: globally summed alpha partials
  double* tsum_b = c->tsum + tp;   // world > 1: globally summed beta^2 partials
  CUDA_TRY(c, cudaMemsetAsync(ws.y, 0, (size_t)rows * tp * 4, s));
  const bool keep = p.keep_shift_solutions != 0 && p.shift_solutions != nullptr;
  if (keep) {
    if (c->pc.on) return set_err(c, CIQ_ERR_INVALID_ARG, "keep_shift_solutions: not with a preconditioner");
    st = grow(c, &ws.xq, &ws.xq_elems, (size_t)nq * rows * tp);
    if (st != CIQ_OK) return st;
    CUDA_TRY(c, cudaMemsetAsync(ws.xq, 0, (size_t)nq * rows * tp * 4, s));
  }
  float* xqk = keep ? ws.xq : nullptr;
  // stored-basis variant: the loop runs the Lanczos step and
  // the shifted Givens scalars only (stopping rule unchanged), keeping W_1 .. W_J; Y = sum_j coef_j
  // W_j at the end from the per-shift MINRES on T_J (host, fp64).  ~5 vectors of HBM traffic per
  // iteration instead of 3Q + 6, O(J N T) memory (Property 1's O(Q N T) traded away).
  const int hlen = p.max_iters + 1;
  bool stored = p.stored_basis != 0 && !c->pc.on && !keep;
  if (stored) {
    if (grow(c, &c->basis, &c->basis_elems, (size_t)hlen * rows * tp) != CIQ_OK ||
        grow(c, &c->bhist, &c->bhist_elems, (size_t)4 * hlen * tp + 2 * (size_t)tp) != CIQ_OK) {
      c->err.clear();   // does not fit: the streaming recurrence
      stored = false;
    }
  }
  CUDA_TRY(c, cudaMemsetAsync(ws.d, 0, (size_t)2 * nq * rows * tp * 4, s));
  Ctrl hctrl{};
  hctrl.max_iters = p.max_iters;
  hctrl.nq = nq;
  hctrl.tp = tp;
  hctrl.tol = p.tol;
  hctrl.bd_tol = p.breakdown_tol;
  CUDA_TRY(c, cudaMemcpyAsync(sc.ctrl, &hctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, s));
  const int nbs = rowblocks(rows, tp);
  PrecondDev& P = c->pc;
  LAUNCH(c, launch_colsq_partials(ws.w[1] + c->row0 * tp, rows, tp, ws.bpart, s));
  LAUNCH(c, launch_reduce_cols(ws.bpart, nbs, tp, ws.colsq, 0, s));
  st = global_sum(c, ws.colsq, tp);
  if (st != CIQ_OK) return st;
  LAUNCH(c, launch_init_state(sc, nq, tp, ws.colsq, s));
  if (P.on) {  // work buffers of precond_power / apply_m at this tp (before any graph capture)
    st = grow(c, &P.part, &P.part_cap, (size_t)utv_splits(rows) * P.r2 * tp);
    if (st == CIQ_OK) st = grow(c, &P.h, &P.h_cap, (size_t)P.r2 * tp);
    if (st == CIQ_OK) st = grow(c, &P.bpart, &P.bpart_cap, (size_t)uapply_blocks(rows) * tp);
    if (st == CIQ_OK) st = grow(c, &P.t1, &P.t_cap, (size_t)2 * c->nfull * tp);
    if (st != CIQ_OK) return st;
  }

  // a2/a3: spectrum estimate and quadrature rule.  lanczos_reuse: the estimate comes from the
  // first kReuse Lanczos steps of the solve itself (run below, before the shifted updates).
  constexpr int kReuse = 12;   // a multiple of 6: the captured graph's buffer rotation is kept
  const bool reuse = p.lanczos_reuse != 0 && p.t == nullptr && !(p.lambda_min > 0 && p.lambda_max > 0) && !P.on &&
                     p.max_iters > 2 * kReuse;
  double t[CIQ_MAX_Q], w[CIQ_MAX_Q];
  double lmin = NAN, lmax = NAN, rmin = NAN, rmax = NAN;
  int lambda_mvms = 0;
  CUDA_TRY(c, cudaEventRecord(ev.e[1], s));
  if (reuse) {
    // rule computed after the warm-up
  } else if (p.t != nullptr) {
    for (int q = 0; q < nq; ++q) { t[q] = p.t[q]; w[q] = p.w[q]; }
  } else {
    if (p.lambda_min > 0 && p.lambda_max > 0) {
      lmin = p.lambda_min;
      lmax = p.lambda_max;
    } else {
      // rigorous lower bound on lambda_min (reading G6): sigma2 for K, 1 for P^{-1/2} K P^{-1/2}
      st = estimate_lambda(c, &p, P.on ? 1.0 : (double)c->op.diag, &lmin, &lmax, &rmin, &rmax, &lambda_mvms);
      if (st != CIQ_OK) return st;
    }
    int r = ciqh::hht_rule(lmin, lmax, nq, t, w);
    if (r != 0) return set_err(c, r == -1 ? CIQ_ERR_INVALID_ARG : CIQ_ERR_ELLIPTIC, "quadrature rule failed");
  }
  if (!reuse) {
    CUDA_TRY(c, cudaMemcpyAsync(sc.shifts, t, nq * 8, cudaMemcpyHostToDevice, s));
    CUDA_TRY(c, cudaMemcpyAsync(sc.weights, w, nq * 8, cudaMemcpyHostToDevice, s));
  }
  CUDA_TRY(c, cudaEventRecord(ev.e[2], s));

  // a4-a6: msMINRES iterations.  Buffers rotate with period 6 in j (W: j mod 3, D: j mod 2) and
  // every kernel reads the iteration state from device memory, so a block of `poll_every`
  // (a multiple of 6) iterations is captured once as a CUDA graph and replayed; iterations past
  // the device-side stopping rule are no-ops.
  float* dslot[2] = {ws.d, ws.d + (size_t)nq * rows * tp};
  Ctrl hc{};
  int loop_nsplit = 1, loop_impl = 0;
  // Preconditioned operator M = P^{-1/2} K P^{-1/2} (App. A): out = M v with the fixed-order
  // partials of v.out (the alpha partials); the column norms of P^{-1/2} v (needed by the split-
  // fp16 packing) come from the same streaming pass.
  auto apply_m = [&](const float* v, float* out, double** apart, int* nbm) -> ciq_status {
    // v: full-height Lanczos block (this rank's rows valid); t1 = P^{-1/2} v on this rank's rows,
    // all-gathered for the K MVM; out (local rows) = P^{-1/2} K t1 with the alpha partials of out.v
    const float* vl = v + c->row0 * tp;
    float* t1l = P.t1 + c->row0 * tp;
    ciq_status st2 = precond_power(c, PW_MHALF, vl, tp, rows, t1l, t1l);
    if (st2 != CIQ_OK) return st2;
    LAUNCH(c, launch_reduce_cols(P.bpart, uapply_blocks(rows), tp, ws.colsq, c->sharded ? 0 : 1, s));
    if (c->sharded) {   // column norms of the full t1 (the MVM operand's pack scale) and the block
      st2 = global_sum(c, ws.colsq, tp);
      if (st2 != CIQ_OK) return st2;
      LAUNCH(c, launch_sqrt_inplace(ws.colsq, tp, s));
      st2 = allgather_rows(c, P.t1, tp);
      if (st2 != CIQ_OK) return st2;
    }
    float* t2 = P.t1 + (size_t)c->nfull * tp;   // second half of the t1 allocation (2 nfull tp)
    st2 = run_mvm(c, P.t1, tp, t2, nullptr, nullptr, p.mvm_impl, ws.colsq);
    if (st2 != CIQ_OK) return st2;
    st2 = precond_power(c, PW_MHALF, t2, tp, rows, out, vl);
    if (st2 != CIQ_OK) return st2;
    *apart = P.bpart;
    *nbm = uapply_blocks(rows);
    return CIQ_OK;
  };
  // single GPU, tensor-core MVM: the streaming pass of iteration j writes W_{j+1}'s split-fp16
  // planes (scale from nrm_j), so no iteration packs; W_1's planes are written here, outside the
  // captured graph (graph replays and direct launches then run identical kernels)
  // (row-sharded: each rank packs its own rows and the ranks all-gather the planes instead of
  // the fp32 block -- the same bytes, already in the MVM's operand layout)
  const bool fuse_pack = !P.on && use_tc(c, p.mvm_impl, tp) && !experiment_env("CIQ_NO_FUSED_PACK");
  if (fuse_pack) {
    st = prepare_mvm_buffers(c, tp, p.mvm_impl);
    if (st != CIQ_OK) return st;
    LAUNCH(c, launch_pack_v(ws.w[1], c->op.n, vrows(c), tp, plane_cols(c, tp), sc.nrm_cur, c->planes, c->inv_scale, s));
  }
  const bool overlap = fuse_pack && use_overlap(c, p.mvm_impl, tp);
  // Relaxed inexact Krylov (params.mvm_relax; Simoncini & Szyld): the MVM's
  // error may grow as 1 / ||r_j|| without moving the result, so once the max relative residual is
  // <= kRelaxThr the full-tile kernel runs with 4x longer TMEM accumulation chains (kTc2RelaxedChain:
  // 4x the round-toward-zero bias, fewer column splits and partial products)
  // Second level: once <= kRelaxThr2 the kernel entries are rounded to fp16
  // (k_hi only: the K_lo . V_hi product and the low split dropped, error ~2^-12 per entry, ~15-30x
  // the accurate chains'): relaxation bound 1/30, kept with a 3x margin
#ifdef CIQ_EXPERIMENTS
  static const double kRelaxThr = getenv("CIQ_RELAX_THR") ? atof(getenv("CIQ_RELAX_THR")) : 0.1;
  static const double kRelaxThr2 = getenv("CIQ_RELAX_THR2") ? atof(getenv("CIQ_RELAX_THR2")) : 0.01;
#else
  constexpr double kRelaxThr = 0.1;
  constexpr double kRelaxThr2 = 0.01;
#endif
  int ns_acc = 0, ns_rel = 0;
  bool relax = false, relax_dense = false;
#ifndef CIQ_NO_ALPHA_FUSE
  if (p.mvm_relax && !P.on && !overlap && !c->sharded && !c->deriv && use_tc(c, p.mvm_impl, tp) &&
      is_kernel_op(c) && !use_mat(c, tp) && !use_sym(c, p.mvm_impl, tp) && !use_tc3(c, tp)) {
    int64_t nb = 0;
    mvm_geometry(c, tp, p.mvm_impl, &ns_acc, &nb);
    ns_rel = tc2_choose_nsplit(rows, c->op.n, tp / tc_chunk_cols(tp), sm_count(), 4, kTc2RelaxedChain);
    relax = ns_rel < ns_acc;
  }
  // dense K (and the materialised kernel operator): level 2 only -- the HBM-bound dense kernel
  // streams the K_hi planes alone (half the bytes); no long-chain level (its chains are short)
  if (p.mvm_relax && !P.on && !overlap && !c->sharded && !c->post.on && !c->deriv && use_tc(c, p.mvm_impl, tp) &&
      (c->op.kind == CIQ_OP_DENSE || use_mat(c, tp)))
    relax_dense = true;
#endif
  {
    const double thr[2] = {relax ? kRelaxThr : 0.0, relax || relax_dense ? kRelaxThr2 : 0.0};
    const int zero[3] = {0, 0, 0};
    CUDA_TRY(c, cudaMemcpyAsync(&sc.ctrl->relax_thr, thr, 2 * sizeof(double), cudaMemcpyHostToDevice, s));
    CUDA_TRY(c, cudaMemcpyAsync(&sc.ctrl->relaxed, zero, 3 * sizeof(int), cudaMemcpyHostToDevice, s));   // + the _from steps
  }
  const OverlapGeo og = overlap ? overlap_geometry(c, tp) : OverlapGeo{};
  auto enqueue_iter = [&](int j, int nqe) -> ciq_status {
    float* wcur = ws.w[j % 3];
    float* wprev = ws.w[(j + 2) % 3];
    float* wnew = ws.w[(j + 1) % 3];
    begin_timed(c, j, 0);
    int nsplit = 1, nbm = 0;
    double* apart = nullptr;
    // single GPU, tensor-core MVM: the streaming pass of iteration j writes W_{j+1}'s split-fp16
    // planes, so iteration j+1 skips pack_v (the first iteration of a block always packs)
    ciq_status st2 = CIQ_OK;
    if (overlap) {
      // row-sharded overlap: W_j's planes of this rank's rows were written by the
      // previous streaming pass, so the MVM of the local diagonal block (K[rows, rows] W_j[rows],
      // on s2, sigma^2 W_j included) runs while the ranks all-gather W_j's planes on `stream`;
      // then the remote column tiles.  The consumer sums both launches' partial products.
      CUDA_TRY(c, cudaEventRecord(c->ev_fork, s));
      CUDA_TRY(c, cudaStreamWaitEvent(c->s2, c->ev_fork, 0));
      int nsl = 0, nbl = 0;
      double* apl = nullptr;
      c->mvm_win = ciq_ctx::MvmWinArgs{true, og.lo, og.hi, 0, 0, 0, std::max(1, sm_count() - kOverlapReservedSMs),
                                       og.nsr, og.nbr};
      c->stream = c->s2;
      st2 = run_mvm(c, wcur, tp, ws.p, ws.apart, sc.ctrl, p.mvm_impl, sc.nrm_cur, true, &nsl, &apl, &nbl, true);
      c->stream = s;
      c->mvm_win = ciq_ctx::MvmWinArgs{};
      if (st2 != CIQ_OK) return st2;
      CUDA_TRY(c, cudaEventRecord(c->ev_join, c->s2));
      st2 = allgather_planes(c, tp);
      if (st2 != CIQ_OK) return st2;
      CUDA_TRY(c, cudaStreamWaitEvent(s, c->ev_join, 0));
      if (og.nsr > 0) {
        int nsr = 0, nbr = 0;
        double* apr = nullptr;
        c->mvm_win = ciq_ctx::MvmWinArgs{true, 0, 0, og.lo, og.hi, 1, 0, 0, 0};
        c->mvm_win.hi = (int)((c->op.n + 63) / 64);
        st2 = run_mvm(c, wcur, tp, ws.p, ws.apart, sc.ctrl, p.mvm_impl, sc.nrm_cur, true, &nsr, &apr, &nbr, true);
        c->mvm_win = ciq_ctx::MvmWinArgs{};
        if (st2 != CIQ_OK) return st2;
      }
      nsplit = og.nsr + og.nsl;
      nbm = (int)(og.nbr + og.nbl);
      apart = c->apart_tc;
    } else if (relax && !c->post.on) {
      // relaxed schedule (params.mvm_relax): the kernel takes the accurate or the relaxed column
      // splits from ctrl->relaxed (set by the Givens pass once max relres <= relax_thr); alpha_j in
      // its tail either way (the consumer's split count follows the same flag)
      c->alpha_fuse = &sc;
      c->mvm_gate = ciq_ctx::MvmGate{true, ns_acc, ns_rel};
      st2 = run_mvm(c, wcur, tp, ws.p, ws.apart, sc.ctrl, p.mvm_impl, sc.nrm_cur, true, &nsplit, &apart, &nbm,
                    fuse_pack);
      if (st2 == CIQ_OK && !c->alpha_fused)
        st2 = set_err(c, CIQ_ERR_INVALID_ARG, "internal: relaxed MVM schedule without the fused alpha");
      c->mvm_gate = ciq_ctx::MvmGate{};
      c->alpha_fuse = nullptr;
    } else {
      c->alpha_fuse = P.on ? nullptr : &sc;   // the full-tile kernel computes alpha_j in its tail
      // posterior operator (f2): the relaxed schedule applies to the K** MVM and its split sum; the
      // downdate and alpha follow the posterior path
      if (relax || relax_dense) c->mvm_gate = ciq_ctx::MvmGate{true, ns_acc, ns_rel};
      st2 = P.on ? apply_m(wcur, ws.p, &apart, &nbm)
                 : run_mvm(c, wcur, tp, ws.p, ws.apart, sc.ctrl, p.mvm_impl, sc.nrm_cur, true, &nsplit,
                           &apart, &nbm, fuse_pack);
      c->mvm_gate = ciq_ctx::MvmGate{};
      c->alpha_fuse = nullptr;
    }
    const bool alpha_done = !P.on && c->alpha_fused;
    c->alpha_fused = false;
    end_timed(c);
    if (st2 != CIQ_OK) return st2;
    const float* pin = (nsplit > 1 || overlap) ? c->psplit : ws.p;
    loop_nsplit = nsplit;
    loop_impl = c->mvm_kind_used;
    if (!c->sharded) {
      if (!alpha_done) LAUNCH(c, launch_alpha(sc, apart, nbm, tp, s));
    } else {
      LAUNCH(c, launch_reduce_cols(apart, nbm, tp, tsum_a, 0, s));
      st2 = global_sum(c, tsum_a, tp);
      if (st2 != CIQ_OK) return st2;
      LAUNCH(c, launch_alpha_from_sum(sc, tsum_a, tp, s));
    }
    float* d1 = dslot[j & 1];
    float* d2 = dslot[(j + 1) & 1];
    begin_timed(c, j, 1);
    LAUNCH(c, launch_lanczos_update(sc, pin, nsplit, (size_t)rows * tp, wcur + c->row0 * tp, wprev + c->row0 * tp,
                                    wnew + c->row0 * tp, &d1, &d2, ws.y, stored ? 0 : nqe, rows, tp, ws.bpart, 0, s,
                                    fuse_pack ? c->planes : nullptr, c->inv_scale, vrows(c), plane_cols(c, tp), c->op.n,
                                    xqk, c->row0, stored ? c->basis : nullptr, (size_t)rows * tp, hlen,
                                    relax && !c->post.on ? ns_rel : 0));
    end_timed(c);
    // stored basis: the streaming pass wrote W_{j+1} to its basis slot, the Givens pass writes the
    // step's scalars (no separate copy pass)
    if (!c->sharded) {
      LAUNCH(c, launch_givens(sc, ws.bpart, update_blocks(rows), nqe, tp, s, stored ? c->bhist : nullptr, hlen));
    } else {
      LAUNCH(c, launch_reduce_cols(ws.bpart, update_blocks(rows), tp, tsum_b, 0, s));
      st2 = global_sum(c, tsum_b, tp);
      if (st2 != CIQ_OK) return st2;
      LAUNCH(c, launch_givens(sc, tsum_b, 1, nqe, tp, s, stored ? c->bhist : nullptr, hlen));
      // next Lanczos block to every rank: its split-fp16 planes when the streaming
      // pass packed them, else the fp32 rows (overlap: the planes at the start of the next
      // iteration, next to the local block's MVM)
      if (!overlap) {
        st2 = fuse_pack ? allgather_planes(c, tp) : allgather_rows(c, wnew, tp);
        if (st2 != CIQ_OK) return st2;
      }
    }
    return CIQ_OK;
  };
  if (stored) {   // slot 0: W_1 (= b), and nrm_1 / the columns frozen before step 1
    CUDA_TRY(c, cudaMemcpyAsync(c->basis, ws.w[1] + c->row0 * tp, (size_t)rows * tp * 4, cudaMemcpyDeviceToDevice, s));
    double* h0 = c->bhist + (size_t)4 * hlen * tp;
    CUDA_TRY(c, cudaMemcpyAsync(h0, sc.nrm_cur, (size_t)tp * 8, cudaMemcpyDeviceToDevice, s));
    LAUNCH(c, launch_int_to_double(sc.frozen, tp, h0 + tp, s));
  }
  int j0 = 0;   // iterations already done (lanczos_reuse warm-up)
  if (reuse) {
    // Warm-up: kReuse plain Lanczos steps of the solve (no shifts yet: nq_eff = 0, no stopping),
    // keeping W_j and the per-step scalars; lambda from the pooled Ritz extremes of the T_j; then
    // the shifted QR / descent updates of those steps are replayed from the history (P:1338-1379:
    // the Lanczos step is shift-independent; only the per-shift QR needs t_q).
    const int R = kReuse;
    const size_t wsz = (size_t)c->nfull * tp;
    st = grow(c, &c->stash, &c->stash_elems, (size_t)R * wsz);
    if (st == CIQ_OK) st = grow(c, &c->hist, &c->hist_elems, (size_t)7 * R * tp);
    if (st != CIQ_OK) return st;
    double* hA = c->hist;                       // alpha_j
    double* hN = hA + (size_t)R * tp;           // nrm_j (norm of W_j)
    double* hP = hN + (size_t)R * tp;           // nrm_{j-1}
    double* hT = hP + (size_t)R * tp;           // beta_j (T off-diagonal before step j)
    double* hB = hT + (size_t)R * tp;           // beta_{j+1}
    double* hQ = hB + (size_t)R * tp;           // beta_{j+1}^2 (replay input)
    int* hF = reinterpret_cast<int*>(hQ + (size_t)R * tp);   // frozen flags before step j
    const int big = 1 << 30;
    const double zero = 0.0;
    CUDA_TRY(c, cudaMemcpyAsync(&sc.ctrl->max_iters, &big, sizeof(int), cudaMemcpyHostToDevice, s));
    CUDA_TRY(c, cudaMemcpyAsync(&sc.ctrl->tol, &zero, sizeof(double), cudaMemcpyHostToDevice, s));
    for (int j = 1; j <= R; ++j) {
      const size_t o = (size_t)(j - 1) * tp;
      CUDA_TRY(c, cudaMemcpyAsync(c->stash + (size_t)(j - 1) * wsz, ws.w[j % 3], wsz * 4, cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(c, cudaMemcpyAsync(hN + o, sc.nrm_cur, tp * 8, cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(c, cudaMemcpyAsync(hP + o, sc.nrm_prev, tp * 8, cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(c, cudaMemcpyAsync(hT + o, sc.tb_cur, tp * 8, cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(c, cudaMemcpyAsync(hF + o, sc.frozen, tp * 4, cudaMemcpyDeviceToDevice, s));
      st = enqueue_iter(j, 0);
      if (st != CIQ_OK) return st;
      CUDA_TRY(c, cudaMemcpyAsync(hA + o, sc.alpha, tp * 8, cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(c, cudaMemcpyAsync(hB + o, sc.tb_cur, tp * 8, cudaMemcpyDeviceToDevice, s));
    }
    std::vector<double> al((size_t)R * tp), bn((size_t)R * tp);
    std::vector<int> fr((size_t)R * tp), frz_end(tp);
    CUDA_TRY(c, cudaMemcpyAsync(al.data(), hA, al.size() * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaMemcpyAsync(bn.data(), hB, bn.size() * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaMemcpyAsync(fr.data(), hF, fr.size() * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaMemcpyAsync(frz_end.data(), sc.frozen, tp * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    // per column: T_m with m = steps taken before the column froze (breakdown / zero column)
    double emin_all = INFINITY, emax_all = -INFINITY;
    std::vector<double> a(R), b(R);
    for (int k = 0; k < (int)T; ++k) {
      int m = 0;
      while (m < R && fr[(size_t)m * tp + k] == 0) ++m;
      if (m < 1) continue;
      for (int i = 0; i < m; ++i) a[i] = al[(size_t)i * tp + k];
      for (int i = 0; i + 1 < m; ++i) b[i] = bn[(size_t)i * tp + k];
      double e0, e1;
      ciqh::tridiag_extremes(a.data(), b.data(), m, &e0, &e1);
      emin_all = std::min(emin_all, e0);
      emax_all = std::max(emax_all, e1);
    }
    rmin = emin_all;
    rmax = emax_all;
    lmax = 1.01 * emax_all;              // reading G6, as estimate_lambda
    lmin = 0.99 * emin_all;
    if (c->op.diag > 0) lmin = std::min(lmin, (double)c->op.diag);
    if (!(lmin > 0) || !std::isfinite(lmax))
      return set_err(c, CIQ_ERR_NOT_PD, "lambda_min estimate %g <= 0: operator is not positive definite", lmin);
    int r = ciqh::hht_rule(lmin, lmax, nq, t, w);
    if (r != 0) return set_err(c, r == -1 ? CIQ_ERR_INVALID_ARG : CIQ_ERR_ELLIPTIC, "quadrature rule failed");
    CUDA_TRY(c, cudaMemcpyAsync(sc.shifts, t, nq * 8, cudaMemcpyHostToDevice, s));
    CUDA_TRY(c, cudaMemcpyAsync(sc.weights, w, nq * 8, cudaMemcpyHostToDevice, s));
    for (auto& x : bn) x = x * x;       // sqrt(fl(x^2)) == x: the replayed givens sees beta_{j+1}
    CUDA_TRY(c, cudaMemcpyAsync(hQ, bn.data(), bn.size() * 8, cudaMemcpyHostToDevice, s));
    // replay: fresh Givens state, then per step the recorded scalars and beta_{j+1}^2 (one block);
    // the descent update of step k (pending) is applied with the stored v_k (W_k / nrm_k)
    LAUNCH(c, launch_init_state(sc, nq, tp, ws.colsq, s));
    for (int k = 1; k <= R; ++k) {
      const size_t o = (size_t)(k - 1) * tp;
      CUDA_TRY(c, cudaMemcpyAsync(sc.alpha, hA + o, tp * 8, cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(c, cudaMemcpyAsync(sc.nrm_cur, hN + o, tp * 8, cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(c, cudaMemcpyAsync(sc.nrm_prev, hP + o, tp * 8, cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(c, cudaMemcpyAsync(sc.tb_cur, hT + o, tp * 8, cudaMemcpyDeviceToDevice, s));
      CUDA_TRY(c, cudaMemcpyAsync(sc.frozen, hF + o, tp * 4, cudaMemcpyDeviceToDevice, s));
      LAUNCH(c, launch_givens(sc, hQ + o, 1, nq, tp, s));
      if (k < R && !stored) {   // step R's update stays pending for iteration R + 1
        float* d1 = dslot[(k + 1) & 1];
        float* d2 = dslot[k & 1];
        float* wk = c->stash + (size_t)(k - 1) * wsz;
        LAUNCH(c, launch_lanczos_update(sc, nullptr, 1, 0, nullptr, wk + c->row0 * tp, nullptr, &d1, &d2, ws.y, nq,
                                        rows, tp, nullptr, 1, s, nullptr, nullptr, 0, 0, 0, xqk));
      }
    }
    CUDA_TRY(c, cudaMemcpyAsync(&sc.ctrl->max_iters, &hctrl.max_iters, sizeof(int), cudaMemcpyHostToDevice, s));
    CUDA_TRY(c, cudaMemcpyAsync(&sc.ctrl->tol, &hctrl.tol, sizeof(double), cudaMemcpyHostToDevice, s));
    j0 = R;
  }
  st = prepare_mvm_buffers(c, tp, p.mvm_impl);   // every buffer the MVM may (re)allocate, before any capture
  if (st != CIQ_OK) return st;
  bool replayed = false;
  // graph-cache key: every host-side decision that changes the captured kernels (the relaxed MVM
  // schedule's gate and split counts included)
  st = run_iterations(c, p, j0, (uint64_t)p.mvm_impl ^ ((uint64_t)(uintptr_t)xqk << 1) ^ (stored ? 0x10000ull : 0ull) ^
                                    (relax ? 0x20000ull : 0ull) ^ (relax_dense ? 0x40000ull : 0ull),
                      enqueue_iter, &hc, &replayed);
  if (st != CIQ_OK) return st;
  if (replayed) {   // cached graph: the MVM kind / splits are those of the capture
    loop_impl = c->last_kind;
    loop_nsplit = c->last_nsplit;
  } else {
    c->last_nsplit = loop_nsplit;
    c->last_kind = loop_impl;
  }
  const int J = hc.iters;
  if (stored && J >= 1) {
    ciq_status sb = combine_stored_basis(c, J, hlen, tp, (int)T, nq, t, w, rows, ws.y);
    if (sb != CIQ_OK) return sb;
  }
  // last pending update (step J): v_J lives in the buffer that was W_cur at iteration J
  if (J >= 1 && !stored) {
    float* d1 = dslot[(J + 1) & 1];  // d_{J-1}
    float* d2 = dslot[J & 1];        // d_{J-2}, overwritten by d_J
    float* wv = ws.w[J % 3];
    LAUNCH(c, launch_lanczos_update(sc, nullptr, 1, 0, nullptr, wv + c->row0 * tp, nullptr, &d1, &d2, ws.y, nq, rows, tp,
                                    nullptr, 1, s, nullptr, nullptr, 0, 0, 0, xqk));
  }
  CUDA_TRY(c, cudaEventRecord(ev.e[3], s));
  if (keep)
    for (int q = 0; q < nq; ++q) {
      st = store_rows(c, ws.xq + (size_t)q * rows * tp, tp, rows, (int)T, p.shift_solutions + (size_t)q * rows * T, T);
      if (st != CIQ_OK) return st;
    }

  // a7: finalise.  With P: Y = M^{-1/2} b in M-space, R' b = P^{-1/2} Y (eq. precond_sqrt_inverse,
  // P:55-64) and R b = K R' b (eq. precond_sqrt).
  float* yout = ws.y;
  if (P.on) {
    st = precond_power(c, PW_MHALF, ws.y, tp, rows, P.t1, nullptr);
    if (st != CIQ_OK) return st;
    yout = P.t1;
  }
  int final_mvm = 0;
  if (p.mode == CIQ_MODE_SQRT) {
    // K . Y: Y is this rank's row block -> all-gather it into a free full-height W buffer
    float* yfull = yout;
    if (c->sharded) {
      yfull = ws.w[(J + 1) % 3];
      CUDA_TRY(c, cudaMemcpyAsync(yfull + c->row0 * tp, yout, (size_t)rows * tp * 4, cudaMemcpyDeviceToDevice, s));
      st = allgather_rows(c, yfull, tp);
      if (st != CIQ_OK) return st;
    }
    LAUNCH(c, launch_colsq_partials(yfull, c->op.n, tp, ws.bpart, s));
    LAUNCH(c, launch_reduce_cols(ws.bpart, rowblocks(c->op.n, tp), tp, ws.colsq, 1, s));
    st = run_mvm(c, yfull, tp, ws.p, nullptr, nullptr, p.mvm_impl, ws.colsq);
    if (st != CIQ_OK) return st;
    final_mvm = 1;
    st = store_rows(c, ws.p, tp, rows, (int)T, out, ldo);
  } else {
    st = store_rows(c, yout, tp, rows, (int)T, out, ldo);
  }
  if (st != CIQ_OK) return st;
  CUDA_TRY(c, cudaEventRecord(ev.e[4], s));
  CUDA_TRY(c, cudaEventSynchronize(ev.e[4]));
  CUDA_TRY(c, cudaGetLastError());

  // a NaN / inf residual or beta (overflow, a non-PSD operator) is never reported as converged,
  // also at fixed J (tol = 0)
  const bool finite = hc.nonfinite == 0 && std::isfinite(hc.max_relres);
  if (!finite) set_err(c, CIQ_NOT_CONVERGED, "non-finite msMINRES residual at iteration %d", hc.iters);
  const bool converged =
      finite && ((p.tol == 0) || (hc.max_relres <= p.tol) || (hc.breakdown > 0 && hc.done && J < p.max_iters));
  if (info) {
    std::memset(info, 0, sizeof(*info));
    info->iters = J;
    info->mvms = lambda_mvms + J + final_mvm;
    info->converged = converged ? 1 : 0;
    info->rotated = c->has_precond ? 1 : 0;
    info->breakdown_cols = hc.breakdown;
    info->Q = nq;
    info->lambda_min = lmin;
    info->lambda_max = lmax;
    info->ritz_min = rmin;
    info->ritz_max = rmax;
    info->max_rel_residual = hc.max_relres;
    for (int q = 0; q < nq; ++q) { info->t[q] = t[q]; info->w[q] = w[q]; }
    cudaEventElapsedTime(&info->ms_total, ev.e[0], ev.e[4]);
    cudaEventElapsedTime(&info->ms_lambda, ev.e[1], ev.e[2]);
    cudaEventElapsedTime(&info->ms_loop, ev.e[2], ev.e[3]);
    cudaEventElapsedTime(&info->ms_final, ev.e[3], ev.e[4]);
    info->kernel_launches = c->launches;
    info->mvm_impl_used = loop_impl;
    info->overlap = overlap ? 1 : 0;
    info->relaxed_from = hc.relaxed_from;
    info->relaxed2_from = hc.relaxed2_from;
    info->mvm_splits = loop_nsplit;
    info->fp64_route = 0;
    for (auto& tm : c->timed) {
      if (tm.j > J) continue;  // iterations launched after convergence are no-ops
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tm.a, tm.b);
      if (tm.kind == 0) { info->ms_mvm += ms; ++info->mvm_timed; }
      else { info->ms_update += ms; ++info->update_timed; }
    }
  }
  return converged ? CIQ_OK : CIQ_NOT_CONVERGED;
}

}  // extern "C"

namespace {

// The fp64 route of the preconditioned variant (precond64.cu; App. A): the same steps as
// ciq_apply -- a1 RHS normalisation, a2/a3 lambda estimate on M and the HHT rule, a4-a6 the
// msMINRES iterations (MVM with M, alpha, streaming update, Givens), a7 finalise -- with fp64
// vectors and the materialised fp64 M:  R' b = P^{-1/2} M^{-1/2} b,  R b = P^{1/2} M (M^{-1/2} b).
ciq_status apply_fp64(ciq_ctx* c, const float* B, int64_t ldb, int64_t T, float* out, int64_t ldo, ciq_params p,
                      ciq_info* info) {
  PrecondDev& P = c->pc;
  const int tp = round16(T);
  const int nq = p.Q;
  const int64_t n = c->op.n, rows = c->row1 - c->row0;
  cudaStream_t s = c->stream;
  ciq_status st = ensure_workspace(c, tp, nq, 8);
  if (st != CIQ_OK) return st;
  Workspace& ws = c->ws;
  const Scal& sc = ws.sc;
  auto D = [](float* f) { return reinterpret_cast<double*>(f); };
  st = join_user_stream(c);
  if (st != CIQ_OK) return st;
  EvTimer ev;
  CUDA_TRY(c, cudaEventRecord(ev.e[0], s));
  // a1: B -> W_1 = nrm_1 v_1 (fp64)
  for (auto& wb : ws.w) CUDA_TRY(c, cudaMemsetAsync(wb, 0, (size_t)c->nfull * tp * 8, s));
  if (is_device_ptr(B)) {
    LAUNCH(c, launch_f32_to_f64(B, ldb, rows, (int)T, D(ws.w[1]) + c->row0 * tp, tp, s));
  } else {
    st = ensure_staging(c, rows * tp);
    if (st != CIQ_OK) return st;
    CUDA_TRY(c, cudaMemcpy2DAsync(c->staging, (size_t)tp * 4, B, (size_t)ldb * 4, (size_t)T * 4, (size_t)rows,
                                  cudaMemcpyHostToDevice, s));
    LAUNCH(c, launch_f32_to_f64(c->staging, tp, rows, (int)T, D(ws.w[1]) + c->row0 * tp, tp, s));
  }
  CUDA_TRY(c, cudaMemsetAsync(ws.y, 0, (size_t)rows * tp * 8, s));
  CUDA_TRY(c, cudaMemsetAsync(ws.d, 0, (size_t)2 * nq * rows * tp * 8, s));
  Ctrl hctrl{};
  hctrl.max_iters = p.max_iters;
  hctrl.nq = nq;
  hctrl.tp = tp;
  hctrl.tol = p.tol;
  hctrl.bd_tol = p.breakdown_tol;
  CUDA_TRY(c, cudaMemcpyAsync(sc.ctrl, &hctrl, sizeof(Ctrl), cudaMemcpyHostToDevice, s));
  LAUNCH(c, launch_colsq_partials64(D(ws.w[1]) + c->row0 * tp, rows, tp, ws.bpart, s));
  LAUNCH(c, launch_reduce_cols(ws.bpart, rowblocks(rows, tp), tp, ws.colsq, 0, s));
  LAUNCH(c, launch_init_state(sc, nq, tp, ws.colsq, s));
  // a2/a3: rule (lambda_min(M) >= 1: reading G6 / G13)
  double t[CIQ_MAX_Q], w[CIQ_MAX_Q];
  double lmin = NAN, lmax = NAN, rmin = NAN, rmax = NAN;
  int lambda_mvms = 0;
  CUDA_TRY(c, cudaEventRecord(ev.e[1], s));
  if (p.t != nullptr) {
    for (int q = 0; q < nq; ++q) { t[q] = p.t[q]; w[q] = p.w[q]; }
  } else {
    if (p.lambda_min > 0 && p.lambda_max > 0) {
      lmin = p.lambda_min;
      lmax = p.lambda_max;
    } else {
      // lambda_min bound: 1 for the preconditioned M (reading G6 / G13), sigma^2 for M = K + sigma^2 I
      st = estimate_lambda(c, &p, P.on ? 1.0 : (double)c->op.diag, &lmin, &lmax, &rmin, &rmax, &lambda_mvms);
      if (st != CIQ_OK) return st;
    }
    const int r = ciqh::hht_rule(lmin, lmax, nq, t, w);
    if (r != 0) return set_err(c, r == -1 ? CIQ_ERR_INVALID_ARG : CIQ_ERR_ELLIPTIC, "quadrature rule failed");
  }
  CUDA_TRY(c, cudaMemcpyAsync(sc.shifts, t, nq * 8, cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaMemcpyAsync(sc.weights, w, nq * 8, cudaMemcpyHostToDevice, s));
  CUDA_TRY(c, cudaEventRecord(ev.e[2], s));
  // a4-a6
  double* dslot[2] = {D(ws.d), D(ws.d) + (size_t)nq * rows * tp};
  const int nb = mvm64_blocks(rows);
  auto enqueue_iter = [&](int j, int nqe) -> ciq_status {
    double* wcur = D(ws.w[j % 3]);
    double* wprev = D(ws.w[(j + 2) % 3]);
    double* wnew = D(ws.w[(j + 1) % 3]);
    begin_timed(c, j, 0);
    LAUNCH(c, launch_mvm64(P.m64, P.ldm, rows, n, wcur, true, tp, c->row0, D(ws.p), true, ws.apart, sc.ctrl, s));
    end_timed(c);
    LAUNCH(c, launch_alpha(sc, ws.apart, nb, tp, s));
    double* d1 = dslot[j & 1];
    double* d2 = dslot[(j + 1) & 1];
    begin_timed(c, j, 1);
    LAUNCH(c, launch_lanczos_update64(sc, D(ws.p), wcur + c->row0 * tp, wprev + c->row0 * tp, wnew + c->row0 * tp,
                                      &d1, &d2, D(ws.y), nqe, rows, tp, ws.bpart, 0, s));
    end_timed(c);
    LAUNCH(c, launch_givens(sc, ws.bpart, update_blocks64(rows), nqe, tp, s));
    return CIQ_OK;
  };
  Ctrl hc{};
  bool replayed = false;
  st = run_iterations(c, p, 0, 1000, enqueue_iter, &hc, &replayed);
  if (st != CIQ_OK) return st;
  const int J = hc.iters;
  if (J >= 1) {   // last pending update (step J)
    double* d1 = dslot[(J + 1) & 1];
    double* d2 = dslot[J & 1];
    LAUNCH(c, launch_lanczos_update64(sc, nullptr, nullptr, D(ws.w[J % 3]) + c->row0 * tp, nullptr, &d1, &d2,
                                      D(ws.y), nq, rows, tp, nullptr, 1, s));
  }
  CUDA_TRY(c, cudaEventRecord(ev.e[3], s));
  // a7: R' b = P^{-1/2} y (eq. precond_sqrt_inverse); R b = P^{1/2} (M y) (eq. precond_sqrt)
  double* res = D(ws.w[0]);   // free after the loop (rows x tp)
  int final_mvm = 0;
  if (p.mode == CIQ_MODE_SQRT) {
    LAUNCH(c, launch_mvm64(P.m64, P.ldm, rows, n, D(ws.y), true, tp, c->row0, D(ws.p), true, nullptr, nullptr, s));
    if (P.on) st = precond_power64(c, PW_HALF, D(ws.p), tp, res);
    else res = D(ws.p);   // K^{1/2} b = K y (eq. contour_integral_quad)
    final_mvm = 1;
  } else if (P.on) {
    st = precond_power64(c, PW_MHALF, D(ws.y), tp, res);
  } else {
    res = D(ws.y);        // K^{-1/2} b = y
  }
  if (st != CIQ_OK) return st;
  if (is_device_ptr(out)) {
    LAUNCH(c, launch_f64_to_f32(res, tp, rows, (int)T, out, ldo, s));
  } else {
    st = ensure_staging(c, rows * tp);
    if (st != CIQ_OK) return st;
    LAUNCH(c, launch_f64_to_f32(res, tp, rows, (int)T, c->staging, T, s));
    CUDA_TRY(c, cudaMemcpy2DAsync(out, (size_t)ldo * 4, c->staging, (size_t)T * 4, (size_t)T * 4, (size_t)rows,
                                  cudaMemcpyDeviceToHost, s));
  }
  CUDA_TRY(c, cudaEventRecord(ev.e[4], s));
  CUDA_TRY(c, cudaEventSynchronize(ev.e[4]));
  CUDA_TRY(c, cudaGetLastError());
  const bool finite = hc.nonfinite == 0 && std::isfinite(hc.max_relres);
  if (!finite) set_err(c, CIQ_NOT_CONVERGED, "non-finite msMINRES residual at iteration %d", hc.iters);
  const bool converged =
      finite && ((p.tol == 0) || (hc.max_relres <= p.tol) || (hc.breakdown > 0 && hc.done && J < p.max_iters));
  if (info) {
    std::memset(info, 0, sizeof(*info));
    info->iters = J;
    info->mvms = lambda_mvms + J + final_mvm;
    info->converged = converged ? 1 : 0;
    info->rotated = P.on ? 1 : 0;
    info->breakdown_cols = hc.breakdown;
    info->Q = nq;
    info->lambda_min = lmin;
    info->lambda_max = lmax;
    info->ritz_min = rmin;
    info->ritz_max = rmax;
    info->max_rel_residual = hc.max_relres;
    for (int q = 0; q < nq; ++q) { info->t[q] = t[q]; info->w[q] = w[q]; }
    cudaEventElapsedTime(&info->ms_total, ev.e[0], ev.e[4]);
    cudaEventElapsedTime(&info->ms_lambda, ev.e[1], ev.e[2]);
    cudaEventElapsedTime(&info->ms_loop, ev.e[2], ev.e[3]);
    cudaEventElapsedTime(&info->ms_final, ev.e[3], ev.e[4]);
    info->kernel_launches = c->launches;
    info->mvm_impl_used = CIQ_MVM_FP64_TC;   // FP64 tensor pipe (mvm64_kernel, DMMA)
    info->mvm_splits = 1;
    info->fp64_route = 1;
    for (auto& tm : c->timed) {
      if (tm.j > J) continue;
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tm.a, tm.b);
      if (tm.kind == 0) { info->ms_mvm += ms; ++info->mvm_timed; }
      else { info->ms_update += ms; ++info->update_timed; }
    }
  }
  return converged ? CIQ_OK : CIQ_NOT_CONVERGED;
}


// ---------------- nested CIQ with a block-Jacobi preconditioner (App. A) ----------------

// a (m x m, row-major, SPD) <- a^{-1} in fp64: Cholesky a = L L^T, then L^{-1}, then L^{-T} L^{-1}.
bool spd_inverse_host(std::vector<double>& a, int m) {
  for (int j = 0; j < m; ++j) {
    double d = a[(size_t)j * m + j];
    for (int k = 0; k < j; ++k) d -= a[(size_t)j * m + k] * a[(size_t)j * m + k];
    if (!(d > 0)) return false;
    d = std::sqrt(d);
    a[(size_t)j * m + j] = d;
    for (int i = j + 1; i < m; ++i) {
      double v = a[(size_t)i * m + j];
      for (int k = 0; k < j; ++k) v -= a[(size_t)i * m + k] * a[(size_t)j * m + k];
      a[(size_t)i * m + j] = v / d;
    }
  }
  std::vector<double> li((size_t)m * m, 0.0);   // L^{-1}, lower triangular
  for (int j = 0; j < m; ++j) {
    li[(size_t)j * m + j] = 1.0 / a[(size_t)j * m + j];
    for (int i = j + 1; i < m; ++i) {
      double v = 0.0;
      for (int k = j; k < i; ++k) v -= a[(size_t)i * m + k] * li[(size_t)k * m + j];
      li[(size_t)i * m + j] = v / a[(size_t)i * m + i];
    }
  }
  for (int i = 0; i < m; ++i)
    for (int j = 0; j <= i; ++j) {
      double v = 0.0;
      for (int k = i; k < m; ++k) v += li[(size_t)k * m + i] * li[(size_t)k * m + j];
      a[(size_t)i * m + j] = v;
      a[(size_t)j * m + i] = v;
    }
  return true;
}

ciq_status ensure_nested(ciq_ctx* c) {
  NestedDev& Nd = c->nest;
  if (Nd.ready) return CIQ_OK;
  const int64_t n = c->op.n;
  cudaStream_t s = c->stream;
  Nd.ldk = (n + 7) / 8 * 8;
  Nd.b0.clear();
  for (int64_t i = 0; i < n; i += Nd.block) Nd.b0.push_back(i);
  Nd.b0.push_back(n);
  const int nb = (int)Nd.b0.size() - 1;
  if (dalloc(&Nd.k64, (size_t)n * Nd.ldk) != cudaSuccess || dalloc(&Nd.pinv, (size_t)n * Nd.block) != cudaSuccess) {
    cudaGetLastError();
    return set_err(c, CIQ_ERR_OOM, "nested preconditioner: N^2 doubles do not fit in device memory");
  }
  CUDA_TRY(c, cudaMemsetAsync(Nd.k64, 0, (size_t)n * Nd.ldk * 8, s));
  LAUNCH(c, launch_materialize64(c->dev, 0, n, Nd.k64, Nd.ldk, s));
  CUDA_TRY(c, cudaStreamSynchronize(s));
  for (int b = 0; b < nb; ++b) {   // P_b = (K + sigma^2 I)[b, b];  P_b^{-1} on the host (fp64)
    const int64_t i0 = Nd.b0[b];
    const int m = (int)(Nd.b0[b + 1] - i0);
    std::vector<double> blk((size_t)m * m);
    CUDA_TRY(c, cudaMemcpy2D(blk.data(), (size_t)m * 8, Nd.k64 + i0 * Nd.ldk + i0, (size_t)Nd.ldk * 8, (size_t)m * 8,
                             (size_t)m, cudaMemcpyDeviceToHost));
    if (!spd_inverse_host(blk, m)) return set_err(c, CIQ_ERR_NOT_PD, "preconditioner block %d is not positive definite", b);
    CUDA_TRY(c, cudaMemcpy(Nd.pinv + i0 * Nd.block, blk.data(), (size_t)m * m * 8, cudaMemcpyHostToDevice));
  }
  Nd.ready = true;
  return CIQ_OK;
}

// P^{-1}-only preconditioned msMINRES (precond_nested.cu header) on columns of c0 (n x tp, fp64),
// pencil (A, P) given as device operators; per-column scalars and the Q x tp Givens rotations on the
// host (fp64).  Returns y = sum_q w_q x_q (x_q = (A + t_q P)^{-1} c0) in yout.  lanczos_only: run
// `max_iters` Lanczos steps and return the per-column tridiagonal (alphas, betas) instead.
struct PencilOps {
  std::function<ciq_status(const double*, double*)> apply_a, apply_pinv;
};

ciq_status pmsminres(ciq_ctx* c, const PencilOps& ops, const double* c0, int tp, int cols, int nq, const double* t,
                     const double* w, int max_iters, double tol, double* yout, int* iters, double* relres,
                     bool lanczos_only, std::vector<std::vector<double>>* alphas, std::vector<std::vector<double>>* betas) {
  const int64_t n = c->op.n;
  const size_t vsz = (size_t)n * tp;
  const int nqe = lanczos_only ? 0 : nq;
  const int nbk = coldot64_blocks(n);
  const size_t need = vsz * (5 + 2 * (size_t)nqe) + (size_t)nbk * tp + (size_t)4 * std::max(1, nqe) * tp + 4 * (size_t)tp;
  NestedDev& Nd = c->nest;
  if (Nd.work_cap < need) {
    dfree(Nd.work);
    Nd.work_cap = 0;
    CUDA_TRY(c, dalloc(&Nd.work, need));
    Nd.work_cap = need;
  }
  cudaStream_t s = c->stream;
  double* r1 = Nd.work;
  double* r2 = r1 + vsz;
  double* yv = r2 + vsz;
  double* v = yv + vsz;
  double* tmp = v + vsz;
  double* dA = tmp + vsz;                      // [nqe][n][tp]
  double* dB = dA + (size_t)nqe * vsz;
  double* part = dB + (size_t)nqe * vsz;
  double* coef = part + (size_t)nbk * tp;      // [4][nqe][tp]
  double* sca = coef + (size_t)4 * std::max(1, nqe) * tp;
  double* scb = sca + tp;
  double* sums = scb + tp;
  std::vector<double> ha(tp), hb(tp), hs(tp);
  auto coldot = [&](const double* a, const double* b, std::vector<double>& outv) -> ciq_status {
    LAUNCH(c, launch_coldot64(a, b, n, tp, part, s));
    LAUNCH(c, launch_reduce_cols(part, nbk, tp, sums, 0, s));
    CUDA_TRY(c, cudaMemcpyAsync(outv.data(), sums, (size_t)tp * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(c, cudaStreamSynchronize(s));
    return CIQ_OK;
  };
  auto axpby = [&](double* out, const std::vector<double>& a, const double* x, const std::vector<double>& b,
                   const double* y) -> ciq_status {
    CUDA_TRY(c, cudaMemcpyAsync(sca, a.data(), (size_t)tp * 8, cudaMemcpyHostToDevice, s));
    CUDA_TRY(c, cudaMemcpyAsync(scb, b.data(), (size_t)tp * 8, cudaMemcpyHostToDevice, s));
    LAUNCH(c, launch_axpby_cols64(out, sca, x, scb, y, n, tp, s));
    return CIQ_OK;
  };
  // r1 = r2 = c0; y = P^{-1} r1; beta_1 = sqrt(r1^T y)
  CUDA_TRY(c, cudaMemcpyAsync(r1, c0, vsz * 8, cudaMemcpyDeviceToDevice, s));
  CUDA_TRY(c, cudaMemcpyAsync(r2, c0, vsz * 8, cudaMemcpyDeviceToDevice, s));
  ciq_status st = ops.apply_pinv(r1, yv);
  if (st != CIQ_OK) return st;
  std::vector<double> b2(tp);
  st = coldot(r1, yv, b2);
  if (st != CIQ_OK) return st;
  std::vector<double> beta1(tp), beta(tp), oldb(tp, 0.0);
  std::vector<int> active(tp);
  for (int k = 0; k < tp; ++k) {
    beta1[k] = (k < cols && b2[k] > 0) ? std::sqrt(b2[k]) : 0.0;
    beta[k] = beta1[k];
    active[k] = beta1[k] > 0;
  }
  std::vector<double> c1((size_t)nq * tp, 1.0), s1((size_t)nq * tp, 0.0), c2((size_t)nq * tp, 1.0), s2((size_t)nq * tp, 0.0),
      phib((size_t)nq * tp), hcoef((size_t)4 * std::max(1, nqe) * tp, 0.0);
  for (int q = 0; q < nq; ++q)
    for (int k = 0; k < tp; ++k) phib[(size_t)q * tp + k] = beta1[k];
  if (alphas) { alphas->assign(tp, {}); betas->assign(tp, {}); }
  if (!lanczos_only) {
    CUDA_TRY(c, cudaMemsetAsync(dA, 0, (size_t)2 * nqe * vsz * 8, s));
    CUDA_TRY(c, cudaMemsetAsync(yout, 0, vsz * 8, s));
  }
  double worst = 0.0;
  int j = 0;
  for (j = 1; j <= max_iters; ++j) {
    bool any = false;
    for (int k = 0; k < tp; ++k) any = any || active[k];
    if (!any) { --j; break; }
    // v = y / beta_j ; y = A v - (beta_j / beta_{j-1}) r1 ; alpha = v^T y ; y -= (alpha / beta_j) r2
    std::vector<double> inv(tp), zero(tp, 0.0), one(tp, 1.0), m1(tp), m2(tp);
    for (int k = 0; k < tp; ++k) inv[k] = active[k] ? 1.0 / beta[k] : 0.0;
    st = axpby(v, inv, yv, zero, nullptr);
    if (st != CIQ_OK) return st;
    st = ops.apply_a(v, yv);
    if (st != CIQ_OK) return st;
    if (j >= 2) {
      for (int k = 0; k < tp; ++k) m1[k] = (active[k] && oldb[k] > 0) ? -beta[k] / oldb[k] : 0.0;
      st = axpby(yv, one, yv, m1, r1);
      if (st != CIQ_OK) return st;
    }
    std::vector<double> alpha(tp);
    st = coldot(v, yv, alpha);
    if (st != CIQ_OK) return st;
    for (int k = 0; k < tp; ++k) m2[k] = active[k] ? -alpha[k] / beta[k] : 0.0;
    st = axpby(yv, one, yv, m2, r2);
    if (st != CIQ_OK) return st;
    std::swap(r1, r2);   // r1 <- r2 ; r2 <- y (the old r1 buffer takes y's values below)
    CUDA_TRY(c, cudaMemcpyAsync(r2, yv, vsz * 8, cudaMemcpyDeviceToDevice, s));
    st = ops.apply_pinv(r2, yv);
    if (st != CIQ_OK) return st;
    st = coldot(r2, yv, b2);
    if (st != CIQ_OK) return st;
    std::vector<double> bnew(tp);
    for (int k = 0; k < tp; ++k) bnew[k] = (active[k] && b2[k] > 0) ? std::sqrt(b2[k]) : 0.0;
    if (alphas)
      for (int k = 0; k < cols; ++k)
        if (active[k]) { (*alphas)[k].push_back(alpha[k]); (*betas)[k].push_back(bnew[k]); }
    if (!lanczos_only) {   // per-shift Givens QR of column j of [T_j + t_q I; beta_{j+1} e_j^T]
      worst = 0.0;
      for (int q = 0; q < nq; ++q)
        for (int k = 0; k < tp; ++k) {
          const size_t i = (size_t)q * tp + k;
          double* ca = &hcoef[i];
          double* cb = &hcoef[(size_t)nq * tp + i];
          double* ce = &hcoef[(size_t)2 * nq * tp + i];
          double* cf = &hcoef[(size_t)3 * nq * tp + i];
          if (!active[k]) { *ca = *cb = *ce = *cf = 0.0; continue; }
          const double tb = j >= 2 ? beta[k] : 0.0, tbn = bnew[k];
          const double a = alpha[k] + t[q];
          const double eps = s2[i] * tb, dp = c2[i] * tb;
          const double delta = c1[i] * dp + s1[i] * a, gbar = -s1[i] * dp + c1[i] * a;
          const double gamma = std::hypot(gbar, tbn);
          const double cs = gbar / gamma, sn = tbn / gamma;
          const double phi = cs * phib[i];
          phib[i] = -sn * phib[i];
          *ca = 1.0 / gamma;
          *cb = -delta / gamma;
          *ce = -eps / gamma;
          *cf = w[q] * phi;
          c2[i] = c1[i]; s2[i] = s1[i]; c1[i] = cs; s1[i] = sn;
          const double r = std::fabs(phib[i]) / beta1[k];
          worst = std::isfinite(r) ? std::max(worst, r) : INFINITY;
        }
      CUDA_TRY(c, cudaMemcpyAsync(coef, hcoef.data(), (size_t)4 * nq * tp * 8, cudaMemcpyHostToDevice, s));
      LAUNCH(c, launch_shift_update64(v, dA, dB, yout, coef, nq, n, tp, s));
      std::swap(dA, dB);   // the new d (written over dB) is d_{j}: next step's d1
    }
    for (int k = 0; k < tp; ++k) {
      if (!active[k]) continue;
      if (!(bnew[k] > 1e-14 * (std::fabs(alpha[k]) + beta[k]))) active[k] = 0;   // invariant subspace: frozen
      oldb[k] = beta[k];
      beta[k] = bnew[k];
    }
    if (!lanczos_only && tol > 0 && worst <= tol) break;
  }
  *iters = std::min(j, max_iters);
  *relres = worst;
  return CIQ_OK;
}

// Extremes of the pooled Ritz values of the per-column tridiagonals (host Sturm bisection).
void pooled_ritz(const std::vector<std::vector<double>>& al, const std::vector<std::vector<double>>& be, int cols,
                 double* rmin, double* rmax) {
  *rmin = INFINITY;
  *rmax = -INFINITY;
  for (int k = 0; k < cols; ++k) {
    const int m = (int)al[k].size();
    if (m == 0) continue;
    double e0 = 0, e1 = 0;
    if (ciqh::tridiag_extremes(al[k].data(), be[k].data(), m, &e0, &e1) == 0) {
      *rmin = std::min(*rmin, e0);
      *rmax = std::max(*rmax, e1);
    }
  }
}

ciq_status apply_nested(ciq_ctx* c, const float* B, int64_t ldb, int64_t T, float* out, int64_t ldo, ciq_params p,
                        ciq_info* info) {
  ciq_status st = ensure_nested(c);
  if (st != CIQ_OK) return st;
  NestedDev& Nd = c->nest;
  const int64_t n = c->op.n;
  const int tp = round16(T);
  const int nq = p.Q;
  cudaStream_t s = c->stream;
  st = join_user_stream(c);
  if (st != CIQ_OK) return st;
  EvTimer ev;
  CUDA_TRY(c, cudaEventRecord(ev.e[0], s));
  const size_t vsz = (size_t)n * tp;
  double *b64 = nullptr, *c0 = nullptr, *yin = nullptr, *yout = nullptr;
  CUDA_TRY(c, dalloc(&b64, 4 * vsz));
  c0 = b64 + vsz;
  yin = c0 + vsz;
  yout = yin + vsz;
  struct Freer { double* p; ~Freer() { dfree(p); } } fr{b64};
  CUDA_TRY(c, cudaMemsetAsync(b64, 0, vsz * 8, s));
  if (is_device_ptr(B)) {
    LAUNCH(c, launch_f32_to_f64(B, ldb, n, (int)T, b64, tp, s));
  } else {
    st = ensure_staging(c, n * tp);
    if (st != CIQ_OK) return st;
    CUDA_TRY(c, cudaMemcpy2DAsync(c->staging, (size_t)tp * 4, B, (size_t)ldb * 4, (size_t)T * 4, (size_t)n,
                                  cudaMemcpyHostToDevice, s));
    LAUNCH(c, launch_f32_to_f64(c->staging, tp, n, (int)T, b64, tp, s));
  }
  int kmvms = 0, pmvms = 0;
  auto blockdiag = [&](const double* mats, bool inverse, const double* in, double* outv) -> ciq_status {
    for (size_t b = 0; b + 1 < Nd.b0.size(); ++b) {
      const int64_t i0 = Nd.b0[b], m = Nd.b0[b + 1] - i0;
      const double* a = inverse ? Nd.pinv + i0 * Nd.block : mats + i0 * Nd.ldk + i0;
      const int64_t lda = inverse ? m : Nd.ldk;
      LAUNCH(c, launch_gemm64(false, false, m, tp, m, a, lda, in + i0 * tp, tp, nullptr, 0.0, outv + i0 * tp, tp, s));
    }
    return CIQ_OK;
  };
  PencilOps inner{[&](const double* in, double* o) { ++pmvms; return blockdiag(Nd.k64, false, in, o); },
                  [&](const double* in, double* o) -> ciq_status {
                    CUDA_TRY(c, cudaMemcpyAsync(o, in, vsz * 8, cudaMemcpyDeviceToDevice, s));
                    return CIQ_OK;
                  }};
  PencilOps outer{[&](const double* in, double* o) -> ciq_status {
                    ++kmvms;
                    LAUNCH(c, launch_mvm64(Nd.k64, Nd.ldk, n, n, in, true, tp, 0, o, true, nullptr, nullptr, s));
                    return CIQ_OK;
                  },
                  [&](const double* in, double* o) { return blockdiag(nullptr, true, in, o); }};
  const int lz = std::max(12, p.lanczos_iters + 2);
  std::vector<std::vector<double>> al, be;
  int it = 0;
  double rr = 0.0;
  // (1) c0 = P^{1/2} b by CIQ on P ("run the CIQ algorithm on P"): lambda_min(P) >= sigma^2
  //     (P = blockdiag(K_kern) + sigma^2 I, reading G6); Q_in = max(Q, 16) so the inner quadrature
  //     error stays far below the outer one; K-after form (reading G2): P^{1/2} b = P (P^{-1/2} b)
  st = pmsminres(c, inner, b64, tp, (int)T, 1, nullptr, nullptr, lz, 0.0, nullptr, &it, &rr, true, &al, &be);
  if (st != CIQ_OK) return st;
  double pmin = 0, pmax = 0;
  pooled_ritz(al, be, (int)T, &pmin, &pmax);
  double plo = 0.99 * pmin, phi_ = 1.01 * pmax;
  if (c->op.diag > 0) plo = std::min(plo, (double)c->op.diag);
  const int qin = std::max(nq, 16);
  double tin[CIQ_MAX_Q], win[CIQ_MAX_Q];
  if (!(plo > 0) || ciqh::hht_rule(plo, phi_, qin, tin, win) != 0)
    return set_err(c, CIQ_ERR_ELLIPTIC, "nested CIQ: rule for P failed (lambda [%g, %g])", plo, phi_);
  const double tol_in = p.tol > 0 ? 0.1 * p.tol : 0.0;
  int it_in = 0;
  double rr_in = 0.0;
  st = pmsminres(c, inner, b64, tp, (int)T, qin, tin, win, p.max_iters, tol_in, yin, &it_in, &rr_in, false, nullptr, nullptr);
  if (st != CIQ_OK) return st;
  st = inner.apply_a(yin, c0);
  if (st != CIQ_OK) return st;
  CUDA_TRY(c, cudaEventRecord(ev.e[1], s));
  // (2) the rule for the pencil (K, P): explicit, or Ritz extremes of the P-Lanczos process started
  //     at c0 (margins of reading G6; no rigorous lower bound for a block-Jacobi P)
  double t[CIQ_MAX_Q], w[CIQ_MAX_Q], lmin = NAN, lmax = NAN, rmin = NAN, rmax = NAN;
  int lambda_mvms = 0;
  if (p.t != nullptr) {
    for (int q = 0; q < nq; ++q) { t[q] = p.t[q]; w[q] = p.w[q]; }
  } else {
    if (p.lambda_min > 0 && p.lambda_max > 0) {
      lmin = p.lambda_min;
      lmax = p.lambda_max;
    } else {
      const int k0 = kmvms;
      st = pmsminres(c, outer, c0, tp, (int)T, 1, nullptr, nullptr, lz, 0.0, nullptr, &it, &rr, true, &al, &be);
      if (st != CIQ_OK) return st;
      lambda_mvms = kmvms - k0;
      pooled_ritz(al, be, (int)T, &rmin, &rmax);
      lmin = 0.99 * rmin;
      lmax = 1.01 * rmax;
      // rigorous lower bound (reading G6 for the pencil): lambda_min(P^{-1} K) >= lambda_min(K) /
      // lambda_max(P) >= sigma^2 / lambda_max(P) -- a few Lanczos steps overestimate lambda_min, and
      // an overestimated kappa only costs log(kappa)
      if (c->op.diag > 0) lmin = std::min(lmin, (double)c->op.diag / phi_);
    }
    if (!(lmin > 0) || ciqh::hht_rule(lmin, lmax, nq, t, w) != 0)
      return set_err(c, CIQ_ERR_NOT_PD, "nested CIQ: lambda_min of the pencil estimate %g <= 0", lmin);
  }
  CUDA_TRY(c, cudaEventRecord(ev.e[2], s));
  // (3) sum_q w_q (K + t_q P)^{-1} c0 = R' b  (eq. precond_sqrt_inverse)
  int J = 0;
  double relres = 0.0;
  const int k1 = kmvms;
  st = pmsminres(c, outer, c0, tp, (int)T, nq, t, w, p.max_iters, p.tol, yout, &J, &relres, false, nullptr, nullptr);
  if (st != CIQ_OK) return st;
  const int loop_mvms = kmvms - k1;
  CUDA_TRY(c, cudaEventRecord(ev.e[3], s));
  double* res = yout;
  int final_mvm = 0;
  if (p.mode == CIQ_MODE_SQRT) {   // R b = K R' b (eq. precond_sqrt)
    st = outer.apply_a(yout, yin);
    if (st != CIQ_OK) return st;
    res = yin;
    final_mvm = 1;
  }
  if (is_device_ptr(out)) {
    LAUNCH(c, launch_f64_to_f32(res, tp, n, (int)T, out, ldo, s));
  } else {
    st = ensure_staging(c, n * tp);
    if (st != CIQ_OK) return st;
    LAUNCH(c, launch_f64_to_f32(res, tp, n, (int)T, c->staging, T, s));
    CUDA_TRY(c, cudaMemcpy2DAsync(out, (size_t)ldo * 4, c->staging, (size_t)T * 4, (size_t)T * 4, (size_t)n,
                                  cudaMemcpyDeviceToHost, s));
  }
  CUDA_TRY(c, cudaEventRecord(ev.e[4], s));
  CUDA_TRY(c, cudaEventSynchronize(ev.e[4]));
  const bool converged = std::isfinite(relres) && (p.tol == 0 || relres <= p.tol);
  if (info) {
    std::memset(info, 0, sizeof(*info));
    info->iters = J;
    info->mvms = lambda_mvms + loop_mvms + final_mvm;   // MVMs with K (the P MVMs of the inner CIQ: nested_p_mvms)
    info->converged = converged ? 1 : 0;
    info->rotated = 1;
    info->Q = nq;
    info->lambda_min = lmin;
    info->lambda_max = lmax;
    info->ritz_min = rmin;
    info->ritz_max = rmax;
    info->max_rel_residual = relres;
    for (int q = 0; q < nq; ++q) { info->t[q] = t[q]; info->w[q] = w[q]; }
    cudaEventElapsedTime(&info->ms_total, ev.e[0], ev.e[4]);
    cudaEventElapsedTime(&info->ms_lambda, ev.e[1], ev.e[2]);
    cudaEventElapsedTime(&info->ms_loop, ev.e[2], ev.e[3]);
    cudaEventElapsedTime(&info->ms_final, ev.e[3], ev.e[4]);
    info->mvm_impl_used = CIQ_MVM_FP64_TC;   // K MVMs on the FP64 tensor pipe (mvm64_kernel, DMMA)
    info->mvm_splits = 1;
    info->fp64_route = 1;
    info->nested_p_mvms = pmvms;
    info->nested_iters = it_in;
  }
  return converged ? CIQ_OK : CIQ_NOT_CONVERGED;
}

}  // namespace
