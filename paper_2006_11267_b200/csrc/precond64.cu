// precond64.cu -- the fp64 route of the preconditioned variant (App. A).
//
// Why fp64 (measured, DESIGN.md §5 "Preconditioned path"): the rotated root R' b = P^{-1/2} M^{-1/2} b
// of eq. precond_sqrt_inverse is far more sensitive to rounding than K^{-1/2} b itself.
// At C4 (M = 5000 Matern-5/2, sigma2 = 1e-3, rank-200 pivoted Cholesky, kappa(K) ~ 1e6) rounding
// only the entries of K to fp32 -- everything else exact -- moves R' b by 2.1e-4 (K^{-1/2} b: 5e-6),
// and an fp32 Krylov recurrence on M moves it by 1.4e-4 whatever the MVM: no fp32 route meets the
// north_star's 1e-4 there.  So for operators small enough to hold N^2 doubles:
//
//   M = P^{-1/2} (K + sigma2 I) P^{-1/2} is formed ONCE in fp64 from fp64 kernel entries:
//       K64      = k(X, X) + sigma2 I          (or the given dense K, or COV* = K** - U U^T)
//       H1       = K64 U                        (n x r)
//       A        = a K64 + U diag(g) H1^T       (= P^{-1/2} K64, in place)
//       H2       = A U
//       M        = a A + H2 diag(g) U^T         (= A P^{-1/2}, in place)
//   with P^{-1/2} = a I + U diag(g) U^T, a = sigma2^{-1/2}, g = (s^2 + sigma2)^{-1/2} - a (precond.cu);
//   every MVM of the solve is P = M V on the fp64 FMA pipe (mvm64_kernel), and the Lanczos /
//   msMINRES vectors are fp64 (lanczos_update_kernel<double>).  The final R' b = P^{-1/2} y and
//   R b = P^{1/2} (M y) use the same fp64 GEMM.
#include <cuda_runtime.h>
#include <math.h>

#include "internal.h"

namespace ciq {
namespace {

// ---- kernel entries in fp64 (reading G11; the same forms as kernel_of_r2 in mvm_simt.cu) ----
__device__ __forceinline__ double kernel64(int kind, double r2, double o2) {
  if (kind == 1) return o2 * exp(-0.5 * r2);
  const double r = sqrt(r2);
  if (kind == 2) {
    const double s5 = 2.23606797749978969641 * r;
    return o2 * (1.0 + s5 + s5 * s5 / 3.0) * exp(-s5);
  }
  const double s3 = 1.73205080756887729353 * r;
  return o2 * (1.0 + s3) * exp(-s3);
}

// k[i][j] = K(row0 + i, j) + diag [row0 + i == j], i < rows, j < n (fp64).
__global__ void materialize64_kernel(OpDev op, int64_t row0, int64_t rows, double* __restrict__ k, int64_t ldk) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = (int64_t)blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= rows || j >= op.n) return;
  const int64_t gi = row0 + i;
  double v;
  if (op.kind == 0) {
    v = (double)op.k[gi * op.ldk + j];
  } else {
    double r2 = 0.0;
    for (int c = 0; c < op.d; ++c) {
      const double df = op.xs64[gi * op.d + c] - op.xs64[j * op.d + c];
      r2 = fma(df, df, r2);
    }
    v = kernel64(op.kind, r2, (double)op.o2);
  }
  if (gi == j) v += (double)op.diag;
  k[i * ldk + j] = v;
}

// ---- fp64 GEMM: C = beta C + op(A) diag(g) op(B) (row-major, explicit leading dimensions) ----
// op(A) is m x kk (TA: A stored kk x m), op(B) is kk x n (TB: B stored n x kk); g may be null (1).
// 64 x 64 tile per CTA, 256 threads with 4 x 4 outputs each, contraction staged 16 at a time.
constexpr int GT = 64, GK = 16;

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) gemm64_kernel(int64_t m, int64_t n, int64_t kk, const double* __restrict__ a,
                                                     int64_t lda, const double* __restrict__ b, int64_t ldb,
                                                     const double* __restrict__ g, double beta,
                                                     double* __restrict__ c, int64_t ldc) {
  __shared__ double as[GK][GT + 1];
  __shared__ double bs[GK][GT + 1];
  const int64_t i0 = (int64_t)blockIdx.y * GT, j0 = (int64_t)blockIdx.x * GT;
  const int tid = threadIdx.x, ti = tid / 16, tj = tid % 16;
  double acc[4][4] = {};
  for (int64_t k0 = 0; k0 < kk; k0 += GK) {
    __syncthreads();
    for (int e = tid; e < GK * GT; e += 256) {
      // A: as[k][i]; B: bs[k][j] (coalesced along the stored row of each operand)
      int r, q;
      if (TA) { r = e / GT; q = e % GT; } else { q = e / GK; r = e % GK; }
      const int64_t ia = i0 + q, ka = k0 + r;
      double va = 0.0;
      if (ia < m && ka < kk) va = TA ? a[ka * lda + ia] : a[ia * lda + ka];
      if (g != nullptr && ka < kk) va *= g[ka];
      as[r][q] = va;
      if (TB) { q = e / GK; r = e % GK; } else { r = e / GT; q = e % GT; }
      const int64_t jb = j0 + q, kb = k0 + r;
      double vb = 0.0;
      if (jb < n && kb < kk) vb = TB ? b[jb * ldb + kb] : b[kb * ldb + jb];
      bs[r][q] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < GK; ++k) {
      double x[4], y[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { x[u] = as[k][ti + 16 * u]; y[u] = bs[k][tj + 16 * u]; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(x[u], y[v], acc[u][v]);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t i = i0 + ti + 16 * u;
    if (i >= m) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t j = j0 + tj + 16 * v;
      if (j >= n) continue;
      const double prev = (beta != 0.0) ? beta * c[i * ldc + j] : 0.0;
      c[i * ldc + j] = prev + acc[u][v];
    }
  }
}

// ---- the solve's MVM on the materialised M: P = M V (+ fixed-order alpha partials) ----
// M: rows x n (ld ldm, even, columns [n, ldm) zero), fp64.  V: n x tp (TV = float or double; rows >= n are never read).
// P: rows x tp (TP).  128 x 128 output tile per CTA, 256 threads with 8 x 8 outputs each
// (4 FMAs per shared-memory load), contraction staged 8 at a time, double-buffered through
// registers.  apart[blockIdx.x][c] = sum_{i in the tile} V[row0 + i][c] P[i][c] (fixed order).
constexpr int MB = 128, MK = 8;

template <class TV>
__device__ __forceinline__ void ld2(const TV* p, double& x, double& y);
template <>
__device__ __forceinline__ void ld2<float>(const float* p, double& x, double& y) {
  const float2 f = *reinterpret_cast<const float2*>(p);
  x = f.x; y = f.y;
}
template <>
__device__ __forceinline__ void ld2<double>(const double* p, double& x, double& y) {
  const double2 f = *reinterpret_cast<const double2*>(p);
  x = f.x; y = f.y;
}

template <class TV, class TP>
__global__ void __launch_bounds__(256) mvm64_kernel(const double* __restrict__ mtx, int64_t ldm, int64_t rows, int64_t n,
                                                    const TV* __restrict__ v, int tp, int64_t row0,
                                                    TP* __restrict__ p, double* __restrict__ apart,
                                                    const Ctrl* __restrict__ done) {
  if (done != nullptr && done->done) return;
  __shared__ double as[2][MK][MB];
  __shared__ double bs[2][MK][MB];
  double (*red)[MB] = reinterpret_cast<double (*)[MB]>(&as[0][0][0]);   // epilogue reuse: 16 x MB
  const int64_t i0 = (int64_t)blockIdx.x * MB;
  const int c0 = blockIdx.y * MB;
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  // global -> register staging: A (128 rows x 8 k) and B (8 k x 128 cols), 2 double pairs each
  double ra[4], rb[4];
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int e = tid + it * 256;
      const int r = e / 4, kq = (e % 4) * 2;          // A: row r, k pair kq
      const int64_t i = i0 + r, k = k0 + kq;
      double x = 0.0, y = 0.0;
      if (i < rows) {
        // ldm even (padded): the pair is aligned; columns in [n, ldm) are zero
        if (k < n) { const double2 f = *reinterpret_cast<const double2*>(mtx + i * ldm + k); x = f.x; y = f.y; }
      }
      ra[2 * it] = x; ra[2 * it + 1] = y;
      const int kb = e / 64, cq = (e % 64) * 2;          // B: k row kb, column pair cq
      const int64_t kr = k0 + kb;
      const int cc = c0 + cq;
      double bx = 0.0, by = 0.0;
      if (kr < n && cc < tp) ld2<TV>(v + kr * tp + cc, bx, by);   // tp % 16 == 0: pairs never straddle
      rb[2 * it] = bx; rb[2 * it + 1] = by;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int e = tid + it * 256;
      const int r = e / 4, kq = (e % 4) * 2;
      as[buf][kq][r] = ra[2 * it];
      as[buf][kq + 1][r] = ra[2 * it + 1];
      const int kb = e / 64, cq = (e % 64) * 2;
      bs[buf][kb][cq] = rb[2 * it];
      bs[buf][kb][cq + 1] = rb[2 * it + 1];
    }
  };
  double acc[8][8] = {};
  const int64_t nk = (n + MK - 1) / MK;
  load(0);
  store(0);
  __syncthreads();
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int buf = (int)(kt & 1);
    if (kt + 1 < nk) load((kt + 1) * MK);
#pragma unroll
    for (int k = 0; k < MK; ++k) {
      double x[8], y[8];
      // rows ty*4 + {0..3} and 64 + ty*4 + {0..3}; columns tx*4 + {0..3} and 64 + tx*4 + {0..3}
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double2 a01 = *reinterpret_cast<const double2*>(&as[buf][k][h * 64 + ty * 4]);
        const double2 a23 = *reinterpret_cast<const double2*>(&as[buf][k][h * 64 + ty * 4 + 2]);
        const double2 b01 = *reinterpret_cast<const double2*>(&bs[buf][k][h * 64 + tx * 4]);
        const double2 b23 = *reinterpret_cast<const double2*>(&bs[buf][k][h * 64 + tx * 4 + 2]);
        x[4 * h + 0] = a01.x; x[4 * h + 1] = a01.y; x[4 * h + 2] = a23.x; x[4 * h + 3] = a23.y;
        y[4 * h + 0] = b01.x; y[4 * h + 1] = b01.y; y[4 * h + 2] = b23.x; y[4 * h + 3] = b23.y;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int w = 0; w < 8; ++w) acc[u][w] = fma(x[u], y[w], acc[u][w]);
    }
    if (kt + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
  // epilogue: write P, alpha partials over this tile's rows (fixed order: rows within a thread,
  // then the 16 row-groups in order)
  double cs[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) cs[w] = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int64_t i = i0 + (u / 4) * 64 + ty * 4 + (u % 4);
    if (i >= rows) continue;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const int c = c0 + (w / 4) * 64 + tx * 4 + (w % 4);
      if (c >= tp) continue;
      p[i * tp + c] = (TP)acc[u][w];
      if (apart != nullptr) cs[w] = fma((double)v[(row0 + i) * tp + c], acc[u][w], cs[w]);
    }
  }
  if (apart != nullptr) {
#pragma unroll
    for (int w = 0; w < 8; ++w) red[ty][(w / 4) * 64 + tx * 4 + (w % 4)] = cs[w];
    __syncthreads();
    if (tid < MB) {
      double s = 0.0;
      for (int r = 0; r < 16; ++r) s += red[r][tid];
      if (c0 + tid < tp) apart[(int64_t)blockIdx.x * tp + c0 + tid] = s;
    }
  }
}

// fp32 rows x cols (ld) -> fp64 rows x tp (zero-padded columns); fp64 -> fp32 (ld)
__global__ void f32_to_f64_kernel(const float* __restrict__ src, int64_t ld, int64_t rows, int cols,
                                  double* __restrict__ dst, int tp) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * tp) return;
  const int64_t i = e / tp;
  const int c = (int)(e % tp);
  dst[e] = (c < cols) ? (double)src[i * ld + c] : 0.0;
}
__global__ void f64_to_f32_kernel(const double* __restrict__ src, int tp, int64_t rows, int cols,
                                  float* __restrict__ dst, int64_t ld) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  const int64_t i = e / cols;
  const int c = (int)(e % cols);
  dst[i * ld + c] = (float)src[i * tp + c];
}

inline unsigned nblk(int64_t e, int bs) { return (unsigned)((e + bs - 1) / bs); }

}  // namespace

cudaError_t launch_materialize64(const OpDev& op, int64_t row0, int64_t rows, double* k, int64_t ldk, cudaStream_t s) {
  dim3 blk(32, 8), grid(nblk(op.n, 32), nblk(rows, 8));
  materialize64_kernel<<<grid, blk, 0, s>>>(op, row0, rows, k, ldk);
  return cudaGetLastError();
}

cudaError_t launch_gemm64(bool ta, bool tb, int64_t m, int64_t n, int64_t kk, const double* a, int64_t lda,
                          const double* b, int64_t ldb, const double* g, double beta, double* c, int64_t ldc,
                          cudaStream_t s) {
  dim3 grid(nblk(n, GT), nblk(m, GT));
  if (ta && tb) gemm64_kernel<true, true><<<grid, 256, 0, s>>>(m, n, kk, a, lda, b, ldb, g, beta, c, ldc);
  else if (ta) gemm64_kernel<true, false><<<grid, 256, 0, s>>>(m, n, kk, a, lda, b, ldb, g, beta, c, ldc);
  else if (tb) gemm64_kernel<false, true><<<grid, 256, 0, s>>>(m, n, kk, a, lda, b, ldb, g, beta, c, ldc);
  else gemm64_kernel<false, false><<<grid, 256, 0, s>>>(m, n, kk, a, lda, b, ldb, g, beta, c, ldc);
  return cudaGetLastError();
}

int mvm64_blocks(int64_t rows) { return (int)((rows + MB - 1) / MB); }

cudaError_t launch_mvm64(const double* m, int64_t ldm, int64_t rows, int64_t n, const void* v, bool v_double, int tp,
                         int64_t row0, void* p, bool p_double, double* apart, const Ctrl* done, cudaStream_t s) {
  if (ldm % 2 != 0) return cudaErrorInvalidValue;
  dim3 grid((unsigned)mvm64_blocks(rows), nblk(tp, MB));
  if (v_double && p_double)
    mvm64_kernel<double, double><<<grid, 256, 0, s>>>(m, ldm, rows, n, (const double*)v, tp, row0, (double*)p, apart, done);
  else if (v_double)
    mvm64_kernel<double, float><<<grid, 256, 0, s>>>(m, ldm, rows, n, (const double*)v, tp, row0, (float*)p, apart, done);
  else if (p_double)
    mvm64_kernel<float, double><<<grid, 256, 0, s>>>(m, ldm, rows, n, (const float*)v, tp, row0, (double*)p, apart, done);
  else
    mvm64_kernel<float, float><<<grid, 256, 0, s>>>(m, ldm, rows, n, (const float*)v, tp, row0, (float*)p, apart, done);
  return cudaGetLastError();
}

cudaError_t launch_f32_to_f64(const float* src, int64_t ld, int64_t rows, int cols, double* dst, int tp,
                              cudaStream_t s) {
  f32_to_f64_kernel<<<nblk(rows * tp, 256), 256, 0, s>>>(src, ld, rows, cols, dst, tp);
  return cudaGetLastError();
}

cudaError_t launch_f64_to_f32(const double* src, int tp, int64_t rows, int cols, float* dst, int64_t ld,
                              cudaStream_t s) {
  f64_to_f32_kernel<<<nblk(rows * cols, 256), 256, 0, s>>>(src, tp, rows, cols, dst, ld);
  return cudaGetLastError();
}

}  // namespace ciq
