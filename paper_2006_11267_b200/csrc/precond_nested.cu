// precond_nested.cu -- vector kernels of the P^{-1}-only preconditioned msMINRES and of nested CIQ
// (App. A), fp64.
//
// For a preconditioner P that "does not readily decompose into P^{1/2} P^{1/2}" the paper runs the
// preconditioned recurrence, which "only needs access to P^{-1}", on
// c = P^{1/2} b, and obtains c itself by "the CIQ algorithm on P".  The shifted solves are
// x_q = (K + t_q P)^{-1} c (the pencil keeps the shift invariance), and
// sum_q w_q x_q = P^{-1/2} (P^{-1/2} K P^{-1/2})^{-1/2} P^{-1/2} c = R' b (eq. precond_sqrt_inverse).
// The recurrence (Paige-Saunders form; reading G13):
//     r1 = c;  y = P^{-1} r1;  beta_1 = sqrt(r1^T y);  r2 = r1
//     v = y / beta_j;  y = K v - (beta_j / beta_{j-1}) r1 - (alpha_j / beta_j) r2,  alpha_j = v^T K v
//     r1 = r2;  r2 = y;  y = P^{-1} r2;  beta_{j+1} = sqrt(r2^T y)
// and per shift the same Givens QR of [T_j + t_q I; beta_{j+1} e_j^T] as the unpreconditioned
// path, with d_j = (v_j - delta d_{j-1} - eps d_{j-2}) / gamma,  x_q += phi d_j.
// The per-column scalars and the Q x T Givens rotations are done on the host in fp64 (ciq_api.cu,
// pmsminres); the kernels here are the N x T vector passes.
#include <cuda_runtime.h>

#include "internal.h"

namespace ciq {
namespace {

constexpr int NT = 256;

// part[b][c0 + c] = sum over block b's rows of a[i][c0 + c] * b[i][c0 + c], c < nc <= 256 (fixed
// order; reduced across blocks by reduce_cols)
__global__ void __launch_bounds__(NT) coldot64_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                      int64_t rows, int tp, int c0, int nc, int64_t rows_per_blk,
                                                      double* __restrict__ part) {
  const int lanes = NT / nc;
  const int c = threadIdx.x % nc, lr = threadIdx.x / nc;
  __shared__ double red[NT];
  double s = 0.0;
  if (lr < lanes) {
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_blk, r1 = min(rows, r0 + rows_per_blk);
    for (int64_t i = r0 + lr; i < r1; i += lanes) s = fma(a[i * tp + c0 + c], b[i * tp + c0 + c], s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < nc) {
    double t = 0.0;
    for (int l = 0; l < lanes; ++l) t += red[l * nc + threadIdx.x];
    part[(int64_t)blockIdx.x * tp + c0 + threadIdx.x] = t;
  }
}

// out[i][c] = ca[c] x[i][c] + cb[c] y[i][c]   (y may be null: cb ignored)
__global__ void axpby_cols64_kernel(double* out, const double* __restrict__ ca, const double* x,
                                    const double* __restrict__ cb, const double* y, int64_t total, int tp) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % tp);
    double r = ca[c] * x[e];
    if (y != nullptr) r = fma(cb[c], y[e], r);
    out[e] = r;
  }
}

// for each shift q: dn = ca[q][c] v + cb[q][c] d1_q + ce[q][c] d2_q  (written over d2_q),
//                   y += cf[q][c] dn
__global__ void shift_update64_kernel(const double* __restrict__ v, double* __restrict__ d1, double* __restrict__ d2,
                                      double* __restrict__ y, const double* __restrict__ coef, int nq, int64_t rows,
                                      int tp) {
  const int64_t total = rows * tp;
  const size_t qs = (size_t)rows * tp;
  const double* ca = coef;
  const double* cb = coef + (size_t)nq * tp;
  const double* ce = coef + (size_t)2 * nq * tp;
  const double* cf = coef + (size_t)3 * nq * tp;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % tp);
    const double ve = v[e];
    double acc = y[e];
    for (int q = 0; q < nq; ++q) {
      const int k = q * tp + c;
      const double dn = fma(ca[k], ve, fma(cb[k], d1[q * qs + e], ce[k] * d2[q * qs + e]));
      d2[q * qs + e] = dn;
      acc = fma(cf[k], dn, acc);
    }
    y[e] = acc;
  }
}

unsigned grid_for(int64_t total) {
  const int64_t g = (total + NT - 1) / NT;
  return (unsigned)(g < 4 * 148 * 8 ? g : 4 * 148 * 8);
}

}  // namespace

int coldot64_blocks(int64_t rows) { return (int)((rows + 255) / 256); }

cudaError_t launch_coldot64(const double* a, const double* b, int64_t rows, int tp, double* part, cudaStream_t s) {
  for (int c0 = 0; c0 < tp; c0 += NT) {
    const int nc = tp - c0 < NT ? tp - c0 : NT;
    coldot64_kernel<<<coldot64_blocks(rows), NT, 0, s>>>(a, b, rows, tp, c0, nc, 256, part);
  }
  return cudaGetLastError();
}

cudaError_t launch_axpby_cols64(double* out, const double* ca, const double* x, const double* cb, const double* y,
                                int64_t rows, int tp, cudaStream_t s) {
  axpby_cols64_kernel<<<grid_for(rows * tp), NT, 0, s>>>(out, ca, x, cb, y, rows * tp, tp);
  return cudaGetLastError();
}

cudaError_t launch_shift_update64(const double* v, double* d1, double* d2, double* y, const double* coef, int nq,
                                  int64_t rows, int tp, cudaStream_t s) {
  shift_update64_kernel<<<grid_for(rows * tp), NT, 0, s>>>(v, d1, d2, y, coef, nq, rows, tp);
  return cudaGetLastError();
}

}  // namespace ciq
