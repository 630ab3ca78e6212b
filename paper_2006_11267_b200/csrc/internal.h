// internal.h -- launchers shared between the C-ABI layer (ciq_api.cu) and the kernel files.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <vector>

#include "common.cuh"

namespace ciq {

// The operator as seen by the MVM kernels (device pointers).
struct OpDev {
  int kind;            // ciq_op_kind
  int64_t n;           // global N
  int d;               // point dimension (kernels)
  const float* xs;     // N x d points scaled by 1/lengthscale (row-major, ld = d)
  const double* xs64;  // the same scaled in fp64 from the caller's fp32 points (fp64 route only)
  const float* k;      // dense: N x N (row-major, ld = ldk)
  int64_t ldk;
  float o2;            // outputscale
  float diag;          // sigma^2 added to the diagonal
  const int64_t* rp;   // sparse: CSR row pointers of the local row block (rp[0] = 0)
  const int32_t* ci;   //         global column indices
  const float* cv;     //         values
};

// Per-solve scalar state (device), one allocation; see recurrence.cu.
struct Scal {
  double* beta1;      // [tp]   ||b_c||
  double* nrm_prev;   // [tp]   nrm_{j-1}: v_{j-1} = W_prev / nrm_{j-1}
  double* nrm_cur;    // [tp]   nrm_j:     v_j     = W_cur  / nrm_j
  double* tb_cur;     // [tp]   T-matrix off-diagonal beta_j (0 at j = 1)
  double* alpha;      // [tp]   alpha_j
  int* frozen;        // [tp]   1: column finished (b = 0 or invariant subspace)
  double* c1; double* s1; double* c2; double* s2; double* phibar;   // [Q][tp] Givens state
  float* ca; float* cb; float* ce; float* cf;                       // [Q][tp] pending-update coefs
  double* da; double* db; double* de; double* df;                   // [Q][tp] the same in fp64 (fp64 route)
  float* cphi;        // [Q][tp] phi of the pending step (x_q += phi d, kept solutions only)
  double* shifts;     // [Q]
  double* weights;    // [Q]
  double* col_rel;    // [tp]   per-column max relative residual of the last Givens step
  int* col_state;     // [tp]   0 frozen before, 1 active, 2 broke in the last step
  Ctrl* ctrl;
};

// ---- MVM (mvm_simt.cu / mvm_tc.cu) ----
// P[i - row0][c] = sum_j K[i][j] V[j][c] + diag V[i][c] for rows [row0, row1), columns [0, tp).
// alpha_part (may be null): [nblk][tp] partials sum_{i in block} V[i][c] P[i][c]; nblk is
// returned by mvm_simt_blocks.  done (may be null): skip when *done != 0.
int mvm_simt_blocks(int64_t rows);
// K rows [row0, row0 + rows) of a kernel operator, fp32 row-major (rows x n), without sigma^2
cudaError_t launch_materialize(const OpDev& op, int64_t row0, int64_t rows, float* k, cudaStream_t s);
cudaError_t launch_mvm_simt(const OpDev& op, const float* v, int tp, int64_t row0, int64_t row1,
                            float* p, int ldp, double* alpha_part, const Ctrl* done, cudaStream_t s);
// sparse (CSR) operator, mvm_sparse.cu: same contract as launch_mvm_simt (alpha partials per
// mvm_simt_blocks(rows) blocks of 64 rows)
cudaError_t launch_spmm(const OpDev& op, const float* v, int tp, int64_t row0, int64_t row1, float* p, int ldp,
                        double* alpha_part, const Ctrl* done, cudaStream_t s);

// tcgen05 MVMs.  Matrix-free (mvm_tc2.cu): persistent 256-row units; dense (mvm_dense.cu):
// persistent 128-row units streaming the split K planes.  Both write nsplit partial products P_s
// (row block, tp columns, stride p_split_stride floats); P = sum_s P_s.
struct TcArgs {
  int kind;
  int64_t n, npad, row0, row1;
  int64_t vrows;             // rows of the split V planes (npad; >= the all-gathered height when sharded)
  int tp, nsplit;
  int nunits, chunks;        // units = row tiles x splits x chunks (round-robin over persistent CTAs)
  int kf;                    // feature contraction (32, or 64 for d > 8: pair kernel only)
  const __half* feat_a;      // [npad/8][4][8][8] A-role features (rows)
  const __half* feat_b;      // [npad/8][4][8][8] B-role features (columns)
  const __half* vplanes;     // [tp/TN][2][npad*TN] split V planes (pack_v)
  const float* inv_scale;    // [tp]
  const float* v;            // fp32 input V (N x tp), for diag*V and alpha
  float* p;
  size_t p_split_stride;
  double* apart;
  float o2, diag;
  const Ctrl* done;
  const __half* kplanes;     // dense path: split K planes [hi | lo], each kplane_elems
  int64_t kplane_elems;
  float kscale_inv;          // dense path: 1 / global K scale
  int dbg;                   // experiments only (-DCIQ_TC_TRACE, env CIQ_TC_DEBUG): 1 skip KV, 2 skip exp
  long long* dbg_clk;        // experiments only: per-tile clock stamps of CTA 0
  // symmetric-tile kernel (mvm_sym.cu)
  const int2* sym_units;     // [nunits / chunks] (column group G, row range k), largest first
  const int* sym_base;       // [sym_nb + 1] first partial slot of each 128-row block
  float* sym_part;           // [chunks][sym_slots][128][TN] fp32 partial products
  int sym_nb, sym_ng, sym_b, sym_slots;
  // fused alpha (mvm_tc2.cu; single-GPU recurrence; null: off): after its read-outs each CTA sums
  // its own units' alpha partials into cta_part[blockIdx][tp] (unit order, slot order); the last CTA
  // to finish (ticket) sums those in CTA order and writes alpha_out[c] = sum / nrm[c]^2 (0 for
  // frozen columns) -- the alpha_kernel pass without its launch
  double* alpha_out;
  const double* alpha_nrm;
  const int* alpha_frozen;
  double* cta_part;
  unsigned* ticket;
  // column window of the full-tile kernel (row-sharded overlap): the launch covers the
  // 64-column tiles [win_lo, win_hi) minus [skip_lo, skip_hi) (win_hi = 0: all tiles, no skip);
  // no_diag: do not add sigma^2 V (another launch of the same product adds it); grid_cap: at most
  // that many CTAs (0: one per SM) -- leaves SMs to a concurrent collective
  int win_lo, win_hi, skip_lo, skip_hi, no_diag, grid_cap;
  // relaxed MVM schedule (params.mvm_relax, full-tile kernel): when *gate != 0 the launch uses
  // nsplit_alt column splits / nunits_alt units (longer accumulation chains); null: never
  const int* gate;
  int nsplit_alt, nunits_alt;
};
// tiles of a (possibly windowed) full-tile launch
#ifdef __CUDACC__
__host__ __device__
#endif
inline int tc2_window_tiles(const TcArgs& a) {
  const int all = (int)((a.n + 63) / 64);
  return (a.win_hi > 0 ? a.win_hi - a.win_lo : all) - (a.skip_hi - a.skip_lo);
}
int tc_chunk_cols(int tp);
// tn: column width of one layout chunk (tc_chunk_cols(tp), halved for the pair kernel)
cudaError_t launch_pack_v(const float* v, int64_t n, int64_t npad, int tp, int tn, const double* nrm, __half* planes,
                          float* inv_scale, cudaStream_t s);
// persistent 256-row matrix-free kernel (mvm_tc2.cu); alpha partials: [row tiles * nsplit * 8][tp]
int tc2_units(int64_t rows, int nsplit, int chunks);
// min_tiles: column tiles each unit keeps (4 for mvm_tc2.cu, tc3_min_tiles() for mvm_tc3.cu)
int tc2_choose_nsplit(int64_t rows, int64_t n, int chunks, int nsm, int min_tiles = 4, int64_t max_chain = 0);
constexpr int64_t kTc2MaxChain = 66;          // accurate TMEM accumulation chain (tiles), mvm_tc2.cu
constexpr int64_t kTc2RelaxedChain = 264;     // the relaxed schedule's chain (4x)
cudaError_t launch_mvm_tc2(const TcArgs& a, int nsm, cudaStream_t s);
// CTA-pair kernel (mvm_tc3.cu): same units / alpha partials as tc2, V planes in TN/2-wide chunks
bool tc3_supported(int tn, int64_t n, int nsplit);
int tc3_min_tiles();
int tc3_units(int64_t rows, int nsplit, int chunks);
cudaError_t launch_mvm_tc3(const TcArgs& a, int nsm, cudaStream_t s);
// symmetric-tile matrix-free kernel (mvm_sym.cu, f4(ii)): single GPU, KF = 32, TN = 16 / 32;
// writes the complete P and alpha partials [sym_nb][tp]
bool sym_supported(int tn);
int sym_group_blocks(int tn);
void sym_geometry(int64_t n, int tn, std::vector<int2>* units, std::vector<int>* base, int* ng, int* slots);
cudaError_t launch_mvm_sym(const TcArgs& a, int nsm, cudaStream_t s);
// persistent dense kernel (mvm_dense.cu): alpha partials [units/chunks * 4][tp]
cudaError_t launch_mvm_dense2(const TcArgs& a, int nsm, cudaStream_t s);
cudaError_t launch_absmax(const float* k, int64_t ldk, int64_t rows, int64_t n, unsigned int* out, cudaStream_t s);
cudaError_t launch_split_dense(const float* k, int64_t ldk, int64_t rows, int64_t n, int64_t npad, float scale,
                               __half* hi, __half* lo, cudaStream_t s);

// ---- vector kernels (recurrence.cu) ----
// part[0 .. dot_rows_blocks()) fp64 partials of sum_{i < rows, c < cols} a[i][c] b[i][c] (fixed order)
int dot_rows_blocks();
cudaError_t launch_dot_rows(const float* a, int64_t lda, const float* b, int64_t ldb, int64_t rows, int cols,
                            double* part, cudaStream_t s);
int rowblocks(int64_t rows, int tp);   // number of CTAs of the row-streaming kernels
int update_blocks(int64_t rows);       // CTAs (= beta^2 partial rows) of lanczos_update_kernel
int update_blocks64(int64_t rows);     // ... of its fp64 instance (launch_lanczos_update64)
// relaxed (may be null): nsplit_relaxed partial products once *relaxed (params.mvm_relax)
cudaError_t launch_sum_splits(const float* parts, int nsplit, size_t stride, int64_t elems, float* out,
                              cudaStream_t s, const int* relaxed = nullptr, int nsplit_relaxed = 0);
cudaError_t launch_load_block(const float* src, int64_t ld_src, int64_t rows, int cols, float* dst, int tp,
                              cudaStream_t s);
cudaError_t launch_store_block(const float* src, int tp, int64_t rows, int cols, float* dst, int64_t ld_dst,
                               cudaStream_t s);
cudaError_t launch_randn_fill(float* dst, int64_t rows, int cols, int tp, int64_t row_offset, uint64_t seed,
                              cudaStream_t s);
cudaError_t launch_colsq_partials(const float* v, int64_t rows, int tp, double* part, cudaStream_t s);
cudaError_t launch_reduce_cols(const double* part, int nblk, int m, double* out, int op_sqrt, cudaStream_t s);
cudaError_t launch_scale_cols(float* v, int64_t rows, int tp, const double* nrm, cudaStream_t s);
cudaError_t launch_init_state(const Scal& sc, int nq, int tp, const double* colsq, cudaStream_t s);
cudaError_t launch_alpha(const Scal& sc, const double* apart, int nblk, int tp, cudaStream_t s);
cudaError_t launch_lanczos_update(const Scal& sc, const float* p, int nsplit, size_t split_stride, const float* wcur, const float* wprev,
                                  float* wnew, float* const* d1, float* const* d2, float* y, int nq,
                                  int64_t rows, int tp, double* bpart, int final_only, cudaStream_t s,
                                  __half* planes = nullptr, float* inv_scale = nullptr, int64_t npad = 0, int tn = 0,
                                  int64_t n = 0,    // planes: also write W_{j+1}'s split-fp16 MVM operand
                                  float* xq = nullptr,    // [Q][rows][tp]: also accumulate x_q += phi_q d_q
                                  int64_t plane_row0 = 0,   // planes: global row of local row 0 (sharded)
                                  float* basis = nullptr, size_t basis_stride = 0,   // stored basis: W_{j+1} to slot j
                                  int hlen = 0,
                                  int nsplit_relaxed = 0);   // > 0: nsplit_relaxed partial products once ctrl->relaxed
// fp64 route (preconditioned path, precond64.cu): the same streaming pass on fp64 vectors (no
// fused packing, no kept solutions); p may be nsplit = 1 only.
cudaError_t launch_lanczos_update64(const Scal& sc, const double* p, const double* wcur, const double* wprev,
                                    double* wnew, double* const* d1, double* const* d2, double* y, int nq,
                                    int64_t rows, int tp, double* bpart, int final_only, cudaStream_t s);
cudaError_t launch_colsq_partials64(const double* v, int64_t rows, int tp, double* part, cudaStream_t s);
// ---- fp64 route of the preconditioned variant (precond64.cu) ----
cudaError_t launch_materialize64(const OpDev& op, int64_t row0, int64_t rows, double* k, int64_t ldk, cudaStream_t s);
// C = beta C + op(A) diag(g) op(B): op(A) m x kk (ta: A stored kk x m), op(B) kk x n (tb: B stored n x kk)
cudaError_t launch_gemm64(bool ta, bool tb, int64_t m, int64_t n, int64_t kk, const double* a, int64_t lda,
                          const double* b, int64_t ldb, const double* g, double beta, double* c, int64_t ldc,
                          cudaStream_t s);
// P = M V (+ alpha partials [mvm64_blocks(rows)][tp]); V (float or double) full height, P local rows
int mvm64_blocks(int64_t rows);
cudaError_t launch_mvm64(const double* m, int64_t ldm, int64_t rows, int64_t n, const void* v, bool v_double, int tp,
                         int64_t row0, void* p, bool p_double, double* apart, const Ctrl* done, cudaStream_t s);
cudaError_t launch_f32_to_f64(const float* src, int64_t ld, int64_t rows, int cols, double* dst, int tp,
                              cudaStream_t s);
cudaError_t launch_f64_to_f32(const double* src, int tp, int64_t rows, int cols, float* dst, int64_t ld,
                              cudaStream_t s);
// ---- stored-basis variant (recurrence.cu) ----
// basis slot ctrl->iters <- w (elems floats); history [4][hlen][tp]: alpha_j, beta_{j+1}, nrm_{j+1}, frozen
cudaError_t launch_int_to_double(const int* a, int m, double* out, cudaStream_t s);
cudaError_t launch_combine_basis(const float* basis, size_t stride, int nb, const float* coef, int64_t elems, int tp,
                                 float* y, cudaStream_t s);
// ---- P^{-1}-only preconditioned msMINRES / nested CIQ (precond_nested.cu), fp64, rows x tp ----
int coldot64_blocks(int64_t rows);
// part[coldot64_blocks(rows)][tp]: per-block column dot products of a and b
cudaError_t launch_coldot64(const double* a, const double* b, int64_t rows, int tp, double* part, cudaStream_t s);
// out = ca[c] x + cb[c] y (y may be null); ca, cb device [tp]
cudaError_t launch_axpby_cols64(double* out, const double* ca, const double* x, const double* cb, const double* y,
                                int64_t rows, int tp, cudaStream_t s);
// d2_q <- ca v + cb d1_q + ce d2_q;  y += cf d2_q   (coef = [ca | cb | ce | cf], each [nq][tp])
cudaError_t launch_shift_update64(const double* v, double* d1, double* d2, double* y, const double* coef, int nq,
                                  int64_t rows, int tp, cudaStream_t s);
// Backward pass: G[i][j] = -1/2 sum_{q,c} w_q (xv[q][i][c] xb[q][j][c] + xb[q][i][c] xv[q][j][c])
cudaError_t launch_vjp_dense(const float* xb, const float* xv, const double* w, int nq, int64_t n, int tp, int cols,
                             float* g, int64_t ldg, cudaStream_t s);
cudaError_t launch_alpha_from_sum(const Scal& sc, const double* sums, int tp, cudaStream_t s);
cudaError_t launch_sum_ranks(const double* g, int world, int m, double* out, cudaStream_t s);
// hist (stored basis, may be null): the step's alpha_j, beta_{j+1}, nrm_{j+1}, frozen at slot j - 1
cudaError_t launch_givens(const Scal& sc, const double* bpart, int nblk, int nq, int tp, cudaStream_t s,
                          double* hist = nullptr, int hlen = 0);
// Lambda-estimation Lanczos (full re-orthogonalisation)
cudaError_t launch_basis_dots(const float* basis, int64_t bstride, int nb, int64_t rows, int tp, const float* p,
                              double* part, cudaStream_t s);
cudaError_t launch_basis_axpy(const float* basis, int64_t bstride, int nb, int64_t rows, int tp, const double* h,
                              float* p, cudaStream_t s);
cudaError_t launch_sqrt_inplace(double* v, int m, cudaStream_t s);
cudaError_t launch_lanczos_coeffs(const double* h1, const double* h2, const double* bsq, int j, int nb_total,
                                  int tp, double bd_tol, double* alphas, double* betas, int* len,
                                  double* inv_beta, cudaStream_t s);
cudaError_t launch_scale_cols_by(const float* src, float* dst, int64_t rows, int tp, const double* inv,
                                 cudaStream_t s);

// ---- Thompson sampling: GP posterior at the candidates (posterior.cu) ----
cudaError_t launch_build_u(int kind, const float* xs, const float* xt, int d, int64_t n, int m, double o2,
                           const double* linv, double* u, float* uf, cudaStream_t s);
int post_splits(int64_t rows);
int post_apply_blocks(int64_t rows);
cudaError_t launch_post_downdate(const float* uf, int m, const float* v, const float* t, int tp, int64_t rows,
                                 float* part, float* h, float* out, double* bpart, cudaStream_t s);
cudaError_t launch_post_mean(const double* u, const double* z, int64_t n, int m, float* mu, cudaStream_t s);
int argmin_blocks(int64_t n);
cudaError_t launch_add_mean_argmin(float* samples, int64_t ld, int64_t n, int t, const float* mu, float* part_v,
                                   int64_t* part_i, int64_t* idx, cudaStream_t s);

// ---- preconditioner P = L L^T + sigma2 I (precond.cu) ----
int utv_splits(int64_t rows);
int uapply_blocks(int64_t rows);
cudaError_t launch_utv(const double* u, int ldu, int r, const float* v, int tp, int64_t rows, int nsplit, double* part,
                       cudaStream_t s);
cudaError_t launch_uapply(const double* u, int ldu, int r, const double* g, const double* h, const float* v, float a,
                          int tp, int64_t rows, float* out, const float* dotv, double* bpart, cudaStream_t s);
cudaError_t launch_gram(const float* l, int ldl, int r, int64_t n, double* gram, cudaStream_t s);
cudaError_t launch_small_right_mul(const float* l, int ldl, int r, const double* wsi, int r2, int64_t n, double* u,
                                   int ldu, cudaStream_t s);
cudaError_t launch_pivchol(const OpDev& op, int rank, float* l, int ldl, double* diag, double* lcol, int* piv,
                           double* pivval, const double* pu, int mu, cudaStream_t s);

}  // namespace ciq
