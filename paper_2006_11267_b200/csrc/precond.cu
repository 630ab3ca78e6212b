// precond.cu -- the low-rank-plus-diagonal preconditioner P = L L^T + sigma2 I of App. A,
// applied in O(N R) per column, and its partial pivoted Cholesky build
// (K7, row a9; Harbrecht et al.).
//
// With the eigendecomposition L^T L = W diag(s^2) W^T (fp64 on the host) and U = L W diag(1/s)
// (orthonormal N x r), every power of P is
//     P^p v = sigma2^p v + U diag((s^2 + sigma2)^p - sigma2^p) U^T v,
// so P^{-1} ("matrix inversion lemma") and P^{+-1/2} are all the same two skinny GEMMs with U.
// The solver runs on M = P^{-1/2} K P^{-1/2} (reading G13): per iteration
// M v = P^{-1/2} (K (P^{-1/2} v)), and R' b = P^{-1/2} M^{-1/2} b at the end:
//     H = U^T V  (r x T, split-K over row blocks, fixed-order fp64 reduction)
//     out = a V + U (g o H)       (optionally with the fp64 partials of sum_i out_ic x_ic)
// U is orthonormal and kept in fp64 with fp64 accumulation: P^{-1/2} amplifies by 1/sigma, and fp32
// storage of U alone costs ~1e-4 relative error at kappa(K) ~ 3e4 (numpy emulation);
// inputs/outputs stay fp32.
#include <cuda_runtime.h>
#include <math.h>

#include "internal.h"

namespace ciq {
namespace {

constexpr int TB = 64;   // tile of the skinny GEMMs (rows x columns)
constexpr int KB = 16;   // contraction step

// part[split][k][c] = sum_{i in split rows} U[i][k] V[i][c]   (k < r, c < tp)
__global__ void __launch_bounds__(256) utv_kernel(const double* __restrict__ u, int ldu, int r,
                                                  const float* __restrict__ v, int tp, int64_t rows, int nsplit,
                                                  double* __restrict__ part) {
  __shared__ double us[KB][TB + 1];
  __shared__ double vs[KB][TB + 1];   // V converted to fp64 once, when staged
  const int k0 = blockIdx.x * TB, c0 = blockIdx.y * TB, sp = blockIdx.z;
  const int64_t i_begin = rows * sp / nsplit, i_end = rows * (sp + 1) / nsplit;
  // 4x4 outputs per thread: k = tk*4 + x, c = tc + 16*y (consecutive lanes read consecutive
  // doubles of vs: no bank conflicts)
  const int tid = threadIdx.x, tk = tid / 16, tc = tid % 16;
  double acc[4][4] = {};
  for (int64_t i0 = i_begin; i0 < i_end; i0 += KB) {
    __syncthreads();
    for (int e = tid; e < KB * TB; e += 256) {
      const int ii = e / TB, cc = e % TB;
      const int64_t i = i0 + ii;
      us[ii][cc] = (i < i_end && k0 + cc < r) ? u[i * ldu + k0 + cc] : 0.0;
      vs[ii][cc] = (i < i_end && c0 + cc < tp) ? (double)v[i * tp + c0 + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ii = 0; ii < KB; ++ii) {
      double a[4], b[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) { a[x] = us[ii][tk * 4 + x]; b[x] = vs[ii][tc + 16 * x]; }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
    }
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int k = k0 + tk * 4 + x, c = c0 + tc + 16 * y;
      if (k < r && c < tp) part[((size_t)sp * r + k) * tp + c] = acc[x][y];
    }
}

// out[i][c] = a * V[i][c] + sum_k U[i][k] g[k] H[k][c];  bpart (optional): partial sums over the
// CTA's rows of out[i][c] * dotv[i][c] (fp64, fixed order).
__global__ void __launch_bounds__(256) uapply_kernel(const double* __restrict__ u, int ldu, int r,
                                                     const double* __restrict__ g, const double* __restrict__ h,
                                                     const float* __restrict__ v, float a, int tp, int64_t rows,
                                                     float* __restrict__ out, const float* __restrict__ dotv,
                                                     double* __restrict__ bpart) {
  __shared__ double us[TB][KB + 1];
  __shared__ double hs[KB][TB + 1];
  __shared__ double red[16][TB];
  const int64_t i0 = (int64_t)blockIdx.x * TB;
  const int c0 = blockIdx.y * TB;
  // 4x4 outputs per thread: rows ti*4 + p, columns tc + 16*q (conflict-free reads of hs,
  // coalesced stores of out)
  const int tid = threadIdx.x, ti = tid / 16, tc = tid % 16;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < r; k0 += KB) {
    __syncthreads();
    for (int e = tid; e < TB * KB; e += 256) {
      const int ii = e / KB, kk = e % KB;
      const int64_t i = i0 + ii;
      us[ii][kk] = (i < rows && k0 + kk < r) ? u[i * ldu + k0 + kk] : 0.0;
      const int kk2 = e / TB, cc = e % TB;
      hs[kk2][cc] = (k0 + kk2 < r && c0 + cc < tp) ? g[k0 + kk2] * h[(size_t)(k0 + kk2) * tp + c0 + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) {
      double x[4], y[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { x[q] = us[ti * 4 + q][kk]; y[q] = hs[kk][tc + 16 * q]; }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(x[p], y[q], acc[p][q]);
    }
  }
  double part[4] = {0, 0, 0, 0};
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int64_t i = i0 + ti * 4 + p;
    if (i >= rows) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c0 + tc + 16 * q;
      if (c >= tp) continue;
      const float o = (float)fma((double)a, (double)v[i * tp + c], acc[p][q]);
      out[i * tp + c] = o;
      if (dotv) part[q] += (double)o * (double)dotv[i * tp + c];
    }
  }
  if (bpart != nullptr) {
#pragma unroll
    for (int q = 0; q < 4; ++q) red[ti][tc + 16 * q] = part[q];
    __syncthreads();
    for (int c = tid; c < TB; c += 256) {
      double s = 0.0;
      for (int t = 0; t < 16; ++t) s += red[t][c];
      if (c0 + c < tp) bpart[(size_t)blockIdx.x * tp + c0 + c] = s;
    }
  }
}

// G[k][l] = sum_i L[i][k] L[i][l] in fp64 (one thread per entry, upper triangle mirrored)
__global__ void gram_kernel(const float* __restrict__ l, int ldl, int r, int64_t n, double* __restrict__ gram) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y;
  if (k >= r || k < m) return;
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += (double)l[i * ldl + k] * (double)l[i * ldl + m];
  gram[(size_t)k * r + m] = s;
  gram[(size_t)m * r + k] = s;
}

// U[i][c] = sum_k L[i][k] Wsi[k][c]   (Wsi = W diag(1/s), r x r2, fp64)
__global__ void small_right_mul_kernel(const float* __restrict__ l, int ldl, int r, const double* __restrict__ wsi,
                                       int r2, int64_t n, double* __restrict__ u, int ldu) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * ldu) return;
  const int64_t i = e / ldu;
  const int c = (int)(e % ldu);
  if (c >= r2) { u[e] = 0.0; return; }
  double s = 0.0;
  for (int k = 0; k < r; ++k) s += (double)l[i * ldl + k] * wsi[(size_t)k * r2 + c];
  u[e] = s;
}

// ---- partial pivoted Cholesky of the kernel part k(X, X) (rows a9) ----

// argmax of diag (lowest index on ties, reading G18) -> piv[step]; single CTA, fixed order.
__global__ void pivot_argmax_kernel(const double* __restrict__ diag, int64_t n, int* __restrict__ piv, int step,
                                    double* __restrict__ pivval) {
  __shared__ double sv[1024];
  __shared__ int si[1024];
  double best = -1.0;
  int bi = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double d = diag[i];
    if (d > best) { best = d; bi = (int)i; }   // strictly greater: lowest index per thread
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double a = sv[threadIdx.x], b = sv[threadIdx.x + s];
      const int ia = si[threadIdx.x], ib = si[threadIdx.x + s];
      if (b > a || (b == a && ib < ia)) { sv[threadIdx.x] = b; si[threadIdx.x] = ib; }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { piv[step] = si[0]; pivval[step] = sv[0]; }
}

template <int KIND>
__device__ __forceinline__ double kval(const float* xs, int d, int64_t i, int64_t j, double o2) {
  double r2 = 0.0;
  for (int k = 0; k < d; ++k) {
    const double df = (double)xs[i * d + k] - (double)xs[j * d + k];
    r2 += df * df;
  }
  if (KIND == 1) return o2 * exp(-0.5 * r2);
  const double r = sqrt(r2);
  if (KIND == 2) return o2 * (1.0 + 2.23606797749979 * r + 5.0 / 3.0 * r2) * exp(-2.23606797749979 * r);
  return o2 * (1.0 + 1.7320508075688772 * r) * exp(-1.7320508075688772 * r);
}

// column m of L: L[i][m] = (k(x_i, x_p) - sum_{l<m} L[i][l] L[p][l]) / sqrt(d_p); diag[i] -= L[i][m]^2
// (pu, mu: the posterior downdate U (n x mu, fp64) of a Thompson-sampling ctx, or null: the factor
// is then of COV* = k(X, X) - U U^T, posterior.cu)
__global__ void pivchol_column_kernel(OpDev op, const int* __restrict__ piv, const double* __restrict__ pivval,
                                      int m, float* __restrict__ l, int ldl, double* __restrict__ diag,
                                      double* __restrict__ lcol, const double* __restrict__ pu, int mu) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= op.n) return;
  const int p = piv[m];
  const double dp = pivval[m];
  double kv;
  if (op.kind == 0) kv = (double)op.k[i * op.ldk + p];
  else if (op.kind == 1) kv = kval<1>(op.xs, op.d, i, p, op.o2);
  else if (op.kind == 2) kv = kval<2>(op.xs, op.d, i, p, op.o2);
  else kv = kval<3>(op.xs, op.d, i, p, op.o2);
  if (pu != nullptr)
    for (int k = 0; k < mu; ++k) kv -= pu[i * mu + k] * pu[(int64_t)p * mu + k];
  double s = kv;
  for (int k = 0; k < m; ++k) s -= lcol[(size_t)k * op.n + i] * lcol[(size_t)k * op.n + p];
  const double v = (dp > 0) ? s / sqrt(dp) : 0.0;
  lcol[(size_t)m * op.n + i] = v;
  l[i * ldl + m] = (float)v;
  diag[i] = (i == p) ? 0.0 : diag[i] - v * v;
}

__global__ void pivchol_init_diag(OpDev op, double* __restrict__ diag, const double* __restrict__ pu, int mu) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= op.n) return;
  double dv = (op.kind == 0) ? (double)op.k[i * op.ldk + i] : (double)op.o2;  // k(x, x) = o^2
  if (pu != nullptr)
    for (int k = 0; k < mu; ++k) dv -= pu[i * mu + k] * pu[i * mu + k];
  diag[i] = dv;
}

inline unsigned nbk(int64_t e, int bs) { return (unsigned)((e + bs - 1) / bs); }

}  // namespace

int utv_splits(int64_t rows) { return (int)std::min<int64_t>(32, std::max<int64_t>(1, rows / 256)); }

cudaError_t launch_utv(const double* u, int ldu, int r, const float* v, int tp, int64_t rows, int nsplit, double* part,
                       cudaStream_t s) {
  dim3 grid((r + TB - 1) / TB, (tp + TB - 1) / TB, nsplit);
  utv_kernel<<<grid, 256, 0, s>>>(u, ldu, r, v, tp, rows, nsplit, part);
  return cudaGetLastError();
}

cudaError_t launch_uapply(const double* u, int ldu, int r, const double* g, const double* h, const float* v, float a,
                          int tp, int64_t rows, float* out, const float* dotv, double* bpart, cudaStream_t s) {
  dim3 grid((unsigned)((rows + TB - 1) / TB), (tp + TB - 1) / TB);
  uapply_kernel<<<grid, 256, 0, s>>>(u, ldu, r, g, h, v, a, tp, rows, out, dotv, bpart);
  return cudaGetLastError();
}
int uapply_blocks(int64_t rows) { return (int)((rows + TB - 1) / TB); }

cudaError_t launch_gram(const float* l, int ldl, int r, int64_t n, double* gram, cudaStream_t s) {
  dim3 grid((r + 127) / 128, r);
  gram_kernel<<<grid, 128, 0, s>>>(l, ldl, r, n, gram);
  return cudaGetLastError();
}

cudaError_t launch_small_right_mul(const float* l, int ldl, int r, const double* wsi, int r2, int64_t n, double* u,
                                   int ldu, cudaStream_t s) {
  small_right_mul_kernel<<<nbk(n * ldu, 256), 256, 0, s>>>(l, ldl, r, wsi, r2, n, u, ldu);
  return cudaGetLastError();
}

cudaError_t launch_pivchol(const OpDev& op, int rank, float* l, int ldl, double* diag, double* lcol, int* piv,
                           double* pivval, const double* pu, int mu, cudaStream_t s) {
  pivchol_init_diag<<<nbk(op.n, 256), 256, 0, s>>>(op, diag, pu, mu);
  for (int m = 0; m < rank; ++m) {
    pivot_argmax_kernel<<<1, 1024, 0, s>>>(diag, op.n, piv, m, pivval);
    pivchol_column_kernel<<<nbk(op.n, 256), 256, 0, s>>>(op, piv, pivval, m, l, ldl, diag, lcol, pu, mu);
  }
  return cudaGetLastError();
}

}  // namespace ciq
