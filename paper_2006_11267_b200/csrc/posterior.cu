// posterior.cu -- the Thompson-sampling step of SS5.2 (eq. thompson_sample; SURVEY
// §8(f) row f2): the GP posterior covariance at the candidates X*,
//     COV* + jitter I = K** + jitter I - K*x (Kxx + noise I)^{-1} Kx*  =  K** + jitter I - U U^T,
// with U = K*x L^{-T} (N x m, fp64; L L^T = Kxx + noise I factorised once on the host, m small),
// and  x~ = argmin(mu* + COV*^{1/2} eps)  per sample column.
//
// The candidate block K** stays matrix-free (the tcgen05 MVM of mvm_tc2.cu); each COV* MVM adds
// a low-rank downdate (H = U^T v split over row blocks, then out = K** v - U H with the alpha
// partials of out . v).  This file builds U and mu*, runs the downdate, and the final mean-add +
// argmin of the Thompson step.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>

#include "internal.h"

namespace ciq {
namespace {

constexpr int TB = 64;   // tile: 64 candidates x 64 outputs
constexpr int KB = 16;   // contraction step over the training points

template <int KIND>
__device__ __forceinline__ double kfun(double r2, double o2) {
  if (KIND == 1) return o2 * exp(-0.5 * r2);
  const double r = sqrt(r2);
  if (KIND == 2) return o2 * (1.0 + 2.23606797749979 * r + 5.0 / 3.0 * r2) * exp(-2.23606797749979 * r);
  return o2 * (1.0 + 1.7320508075688772 * r) * exp(-1.7320508075688772 * r);
}

// U[j][i] = sum_k k(xs_j, xt_k) Linv[i][k]  (j < n candidates, i, k < m training points), fp64;
// xs / xt are already divided by the lengthscale.  The kernel entries are recomputed per output
// tile (m / 64 times), which is cheap next to the contraction for the paper's m (<= 100).
template <int KIND>
__global__ void __launch_bounds__(256) build_u_kernel(const float* __restrict__ xs, const float* __restrict__ xt,
                                                      int d, int64_t n, int m, double o2,
                                                      const double* __restrict__ linv, double* __restrict__ u,
                                                      float* __restrict__ uf) {
  __shared__ double ks[KB][TB + 1];
  __shared__ double ls[KB][TB + 1];
  const int64_t j0 = (int64_t)blockIdx.x * TB;
  const int i0 = blockIdx.y * TB;
  const int tid = threadIdx.x, tj = tid / 16, ti = tid % 16;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < m; k0 += KB) {
    __syncthreads();
    for (int e = tid; e < KB * TB; e += 256) {
      const int kk = e / TB, jj = e % TB;
      const int64_t j = j0 + jj;
      const int k = k0 + kk;
      double kv = 0.0;
      if (j < n && k < m) {
        double r2 = 0.0;
        for (int t = 0; t < d; ++t) {
          const double df = (double)xs[j * d + t] - (double)xt[(int64_t)k * d + t];
          r2 += df * df;
        }
        kv = kfun<KIND>(r2, o2);
      }
      ks[kk][jj] = kv;
      const int i = i0 + jj;
      ls[kk][jj] = (i < m && k < m) ? linv[(int64_t)i * m + k] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < KB; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) { a[x] = ks[kk][tj * 4 + x]; b[x] = ls[kk][ti * 4 + x]; }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
    }
  }
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int64_t j = j0 + tj * 4 + x;
    if (j >= n) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int i = i0 + ti * 4 + y;
      if (i < m) { u[j * m + i] = acc[x][y]; uf[j * m + i] = (float)acc[x][y]; }
    }
  }
}

// ---- the downdate of every COV* MVM: out = t - U (U^T v), fp32 (|U U^T| <= diag K**: no
// amplification, so fp32 storage and accumulation sit far below the tcgen05 K** MVM's error) ----
constexpr int DU_ROWS = 32;   // rows staged per step
constexpr int DU_K = 128;     // k tile (training points)
constexpr int DU_C = 64;      // column tile

// part[s][k][c] = sum_{i in split s} U[i][k] v[i][c]; thread: 4 k x 8 c
__global__ void __launch_bounds__(256) post_utv_kernel(const float* __restrict__ u, int m,
                                                       const float* __restrict__ v, int tp, int64_t rows, int nsplit,
                                                       float* __restrict__ part) {
  __shared__ __align__(16) float us[DU_ROWS][DU_K];
  __shared__ __align__(16) float vs[DU_ROWS][DU_C];
  const int sp = blockIdx.x, k0 = blockIdx.y * DU_K, c0 = blockIdx.z * DU_C;
  const int64_t i_begin = rows * sp / nsplit, i_end = rows * (sp + 1) / nsplit;
  const int tid = threadIdx.x, tk = tid / 8, tc = tid % 8;
  float acc[4][8] = {};
  // register prefetch of the next 32-row step while the current one is multiplied
  float ru[DU_ROWS * DU_K / 256], rv[DU_ROWS * DU_C / 256];
  auto gload = [&](int64_t i0) {
#pragma unroll
    for (int q = 0; q < DU_ROWS * DU_K / 256; ++q) {
      const int e = tid + q * 256, r = e / DU_K, k = e % DU_K;
      const int64_t i = i0 + r;
      ru[q] = (i < i_end && k0 + k < m) ? u[i * m + k0 + k] : 0.f;
    }
#pragma unroll
    for (int q = 0; q < DU_ROWS * DU_C / 256; ++q) {
      const int e = tid + q * 256, r = e / DU_C, cc = e % DU_C;
      const int64_t i = i0 + r;
      rv[q] = (i < i_end && c0 + cc < tp) ? v[i * tp + c0 + cc] : 0.f;
    }
  };
  if (i_begin < i_end) gload(i_begin);
  for (int64_t i0 = i_begin; i0 < i_end; i0 += DU_ROWS) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < DU_ROWS * DU_K / 256; ++q) { const int e = tid + q * 256; us[e / DU_K][e % DU_K] = ru[q]; }
#pragma unroll
    for (int q = 0; q < DU_ROWS * DU_C / 256; ++q) { const int e = tid + q * 256; vs[e / DU_C][e % DU_C] = rv[q]; }
    __syncthreads();
    if (i0 + DU_ROWS < i_end) gload(i0 + DU_ROWS);
#pragma unroll 4
    for (int r = 0; r < DU_ROWS; ++r) {
      const float4 a = *reinterpret_cast<const float4*>(&us[r][tk * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&vs[r][tc * 8]);
      const float4 b1 = *reinterpret_cast<const float4*>(&vs[r][tc * 8 + 4]);
      const float av[4] = {a.x, a.y, a.z, a.w};
      const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 8; ++y) acc[x][y] = fmaf(av[x], bv[y], acc[x][y]);
    }
  }
  // 8 consecutive columns per thread as two float4 (tp is a multiple of 16): the 8 lanes of one k
  // row write 256 contiguous bytes
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int k = k0 + tk * 4 + x;
    const int c = c0 + tc * 8;
    if (k >= m || c >= tp) continue;
    float4* dst = reinterpret_cast<float4*>(part + ((size_t)sp * m + k) * tp + c);
    dst[0] = make_float4(acc[x][0], acc[x][1], acc[x][2], acc[x][3]);
    dst[1] = make_float4(acc[x][4], acc[x][5], acc[x][6], acc[x][7]);
  }
}

// h[k][c] = sum_s part[s][k][c]: 64 entries per CTA, 8 thread groups over the splits, combined
// in a fixed order (deterministic)
__global__ void __launch_bounds__(512) post_reduce_kernel(const float* __restrict__ part, int nsplit, int64_t mt,
                                                          float* __restrict__ h) {
  __shared__ float red[8][64];
  const int64_t e = (int64_t)blockIdx.x * 64 + threadIdx.x % 64;
  const int g = threadIdx.x / 64;
  float s = 0.f;
  if (e < mt)
    for (int sp = g; sp < nsplit; sp += 8) s += part[(size_t)sp * mt + e];
  red[g][threadIdx.x % 64] = s;
  __syncthreads();
  if (g == 0 && e < mt) {
    const int l = threadIdx.x;
    h[e] = ((red[0][l] + red[1][l]) + (red[2][l] + red[3][l])) + ((red[4][l] + red[5][l]) + (red[6][l] + red[7][l]));
  }
}

// out[i][c] = t[i][c] - sum_k U[i][k] h[k][c];  bpart[blk][c] = sum_{i in blk} out[i][c] v[i][c]
// (fp64, fixed order; the alpha partials of the msMINRES step).  Thread: 4 rows x 4 columns.
constexpr int DA_ROWS = 64, DA_K = 64;
__global__ void __launch_bounds__(256) post_apply_kernel(const float* __restrict__ u, int m,
                                                         const float* __restrict__ h, const float* __restrict__ t,
                                                         int tp, int64_t rows, float* __restrict__ out,
                                                         const float* __restrict__ dotv, double* __restrict__ bpart) {
  __shared__ __align__(16) float us[DA_K][DA_ROWS + 4];
  __shared__ __align__(16) float hs[DA_K][64];
  __shared__ double red[16][64];
  const int64_t i0 = (int64_t)blockIdx.x * DA_ROWS;
  const int c0 = blockIdx.y * 64;
  const int tid = threadIdx.x, ti = tid / 16, tc = tid % 16;
  float acc[4][4] = {};
  float ru[DA_ROWS * DA_K / 256], rh[DA_K * 64 / 256];   // register prefetch of the next k chunk
  auto gload = [&](int k0) {
#pragma unroll
    for (int q = 0; q < DA_ROWS * DA_K / 256; ++q) {
      const int e = tid + q * 256, r = e / DA_K, kk = e % DA_K;
      const int64_t i = i0 + r;
      ru[q] = (i < rows && k0 + kk < m) ? u[i * m + k0 + kk] : 0.f;
    }
#pragma unroll
    for (int q = 0; q < DA_K * 64 / 256; ++q) {
      const int e = tid + q * 256, kk = e / 64, cc = e % 64;
      rh[q] = (k0 + kk < m && c0 + cc < tp) ? h[(size_t)(k0 + kk) * tp + c0 + cc] : 0.f;
    }
  };
  gload(0);
  for (int k0 = 0; k0 < m; k0 += DA_K) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < DA_ROWS * DA_K / 256; ++q) { const int e = tid + q * 256; us[e % DA_K][e / DA_K] = ru[q]; }
#pragma unroll
    for (int q = 0; q < DA_K * 64 / 256; ++q) { const int e = tid + q * 256; hs[e / 64][e % 64] = rh[q]; }
    __syncthreads();
    if (k0 + DA_K < m) gload(k0 + DA_K);
#pragma unroll 8
    for (int kk = 0; kk < DA_K; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&us[kk][ti * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&hs[kk][tc * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fmaf(av[x], bv[y], acc[x][y]);
    }
  }
  double pd[4] = {0, 0, 0, 0};
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int64_t i = i0 + ti * 4 + x;
    if (i >= rows) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int c = c0 + tc * 4 + y;
      if (c >= tp) continue;
      const float o = t[i * tp + c] - acc[x][y];
      out[i * tp + c] = o;
      if (dotv) pd[y] += (double)o * (double)dotv[i * tp + c];
    }
  }
  if (bpart != nullptr) {
#pragma unroll
    for (int y = 0; y < 4; ++y) red[ti][tc * 4 + y] = pd[y];
    __syncthreads();
    if (tid < 64) {
      double s = 0.0;
      for (int g = 0; g < 16; ++g) s += red[g][tid];
      if (c0 + tid < tp) bpart[(size_t)blockIdx.x * tp + c0 + tid] = s;
    }
  }
}

// mu[j] = sum_i U[j][i] z[i]  (z = L^{-1} y), fp64 accumulate, fp32 store
__global__ void post_mean_kernel(const double* __restrict__ u, const double* __restrict__ z, int64_t n, int m,
                                 float* __restrict__ mu) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double s = 0.0;
  for (int i = 0; i < m; ++i) s = fma(u[j * m + i], z[i], s);
  mu[j] = (float)s;
}

// samples[j][c] = out[j][c] + mu[j] (in place, ld = ld), and per-block column argmin partials:
// part_v[blk][c], part_i[blk][c] (lowest index among equal minima)
constexpr int AM_ROWS = 256;
__global__ void __launch_bounds__(256) add_mean_argmin_kernel(float* __restrict__ s, int64_t ld, int64_t n, int t,
                                                              const float* __restrict__ mu,
                                                              float* __restrict__ part_v, int64_t* __restrict__ part_i) {
  __shared__ float sv[256];
  __shared__ int64_t si[256];
  const int64_t r0 = (int64_t)blockIdx.x * AM_ROWS;
  const int64_t r1 = r0 + AM_ROWS < n ? r0 + AM_ROWS : n;
  for (int c0 = 0; c0 < t; c0 += 64) {
    const int c = c0 + threadIdx.x % 64, g = threadIdx.x / 64;   // 4 row groups x 64 columns
    float best = INFINITY;
    int64_t bi = -1;
    if (c < t) {
      for (int64_t r = r0 + g; r < r1; r += 4) {
        const float x = s[r * ld + c] + mu[r];
        s[r * ld + c] = x;
        if (x < best || bi < 0) { best = x; bi = r; }
      }
    }
    sv[threadIdx.x] = best;
    si[threadIdx.x] = bi;
    __syncthreads();
    if (g == 0 && c < t) {
      for (int h = 1; h < 4; ++h) {
        const float x = sv[h * 64 + threadIdx.x];
        const int64_t xi = si[h * 64 + threadIdx.x];
        if (xi >= 0 && (bi < 0 || x < best || (x == best && xi < bi))) { best = x; bi = xi; }
      }
      part_v[(int64_t)blockIdx.x * t + c] = best;
      part_i[(int64_t)blockIdx.x * t + c] = bi;
    }
    __syncthreads();
  }
}

// idx[c] = argmin over the blocks' partials, in block order (ties: lowest row index)
__global__ void argmin_final_kernel(const float* __restrict__ part_v, const int64_t* __restrict__ part_i, int nblk,
                                    int t, int64_t* __restrict__ idx) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= t) return;
  float best = INFINITY;
  int64_t bi = -1;
  for (int b = 0; b < nblk; ++b) {
    const float x = part_v[(int64_t)b * t + c];
    const int64_t xi = part_i[(int64_t)b * t + c];
    if (xi >= 0 && (bi < 0 || x < best)) { best = x; bi = xi; }
  }
  idx[c] = bi;
}

}  // namespace

cudaError_t launch_build_u(int kind, const float* xs, const float* xt, int d, int64_t n, int m, double o2,
                           const double* linv, double* u, float* uf, cudaStream_t s) {
  dim3 grid((unsigned)((n + TB - 1) / TB), (unsigned)((m + TB - 1) / TB));
  if (kind == 1) build_u_kernel<1><<<grid, 256, 0, s>>>(xs, xt, d, n, m, o2, linv, u, uf);
  else if (kind == 2) build_u_kernel<2><<<grid, 256, 0, s>>>(xs, xt, d, n, m, o2, linv, u, uf);
  else build_u_kernel<3><<<grid, 256, 0, s>>>(xs, xt, d, n, m, o2, linv, u, uf);
  return cudaGetLastError();
}

cudaError_t launch_post_mean(const double* u, const double* z, int64_t n, int m, float* mu, cudaStream_t s) {
  post_mean_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(u, z, n, m, mu);
  return cudaGetLastError();
}

int post_splits(int64_t rows) { return (int)std::min<int64_t>(2 * 148, std::max<int64_t>(1, rows / 64)); }
int post_apply_blocks(int64_t rows) { return (int)((rows + DA_ROWS - 1) / DA_ROWS); }

cudaError_t launch_post_downdate(const float* uf, int m, const float* v, const float* t, int tp, int64_t rows,
                                 float* part, float* h, float* out, double* bpart, cudaStream_t s) {
  const int ns = post_splits(rows);
  post_utv_kernel<<<dim3(ns, (m + DU_K - 1) / DU_K, (tp + DU_C - 1) / DU_C), 256, 0, s>>>(uf, m, v, tp, rows, ns, part);
  const int64_t mt = (int64_t)m * tp;
  post_reduce_kernel<<<(unsigned)((mt + 63) / 64), 512, 0, s>>>(part, ns, mt, h);
  post_apply_kernel<<<dim3(post_apply_blocks(rows), (tp + 63) / 64), 256, 0, s>>>(uf, m, h, t, tp, rows, out,
                                                                                   bpart ? v : nullptr, bpart);
  return cudaGetLastError();
}

int argmin_blocks(int64_t n) { return (int)((n + AM_ROWS - 1) / AM_ROWS); }

cudaError_t launch_add_mean_argmin(float* samples, int64_t ld, int64_t n, int t, const float* mu, float* part_v,
                                   int64_t* part_i, int64_t* idx, cudaStream_t s) {
  const int nb = argmin_blocks(n);
  add_mean_argmin_kernel<<<nb, 256, 0, s>>>(samples, ld, n, t, mu, part_v, part_i);
  argmin_final_kernel<<<(t + 63) / 64, 64, 0, s>>>(part_v, part_i, nb, t, idx);
  return cudaGetLastError();
}

}  // namespace ciq
