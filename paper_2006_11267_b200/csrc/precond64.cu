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
// P: rows x tp (TP).  On the FP64 tensor pipe: DMMA (mma.sync m8n8k4 f64; measured on this B200
// 37.2 TFLOP/s vs 33.9 for DFMA, scripts/ubench_dmma.cu), 64 x 64 output tile per CTA, 8 warps of
// 32 x 16 (4 x 2 DMMA tiles), contraction staged 16 at a time through a 3-stage cp.async ring
// (no staging registers: 3 CTAs per SM; C4's 79 x 16 tiles fill 2.85 waves of 444).  Shared
// layouts: A[m][k] with a 20-double row (k + 4 pad), B[k][c] with a 68-double row -- the fragment
// loads (lane -> m = lane / 4, k = lane % 4 for A; k = lane % 4, c = lane / 4 for B) hit 16
// distinct 2-bank pairs per half-warp.  apart[rb][c] = sum_{i in the tile} V[row0 + i][c] P[i][c]
// (fixed order).  The round-1/2 SIMT kernel (128 x 128 tiles, 8 x 8 DFMA per thread) ran C4's M MVM
// at 12 TFLOP/s (32% of the FP64 pipe: one CTA per SM, 2.16 waves).
constexpr int MB = 64, MBN = 64, MK = 16, MST = 3;
constexpr int SA = MK + 4;      // A row (doubles)
constexpr int SB = MBN + 4;     // B row (elements)

__device__ __forceinline__ void cp16(void* dst, const void* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int sz = ok ? 16 : 0;   // zero fill out of range
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(sz) : "memory");
}

template <class TV>
__device__ __forceinline__ double ldv(const TV* p) { return (double)*p; }

template <class TV, class TP>
__global__ void __launch_bounds__(256, 3) mvm64_kernel(const double* __restrict__ mtx, int64_t ldm, int64_t rows, int64_t n,
                                                       const TV* __restrict__ v, int tp, int64_t row0,
                                                       TP* __restrict__ p, double* __restrict__ apart,
                                                       const Ctrl* __restrict__ done) {
  if (done != nullptr && done->done) return;
  extern __shared__ __align__(16) uint8_t smem64[];
  double* As = reinterpret_cast<double*>(smem64);                       // [MST][MB][SA]
  TV* Bs = reinterpret_cast<TV*>(smem64 + (size_t)MST * MB * SA * 8);   // [MST][MK][SB]
  const int c0 = blockIdx.x * MBN;
  const int rb = blockIdx.y;
  const int64_t i0 = (int64_t)rb * MB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;        // warp tile rows wm*32.., cols wn*16..
  const int64_t nk = (n + MK - 1) / MK;
  // one stage: A 64 rows x 16 k = 128 x 16 B (thread: row tid / 4 ... two chunks), B 16 k x 64 cols
  auto issue = [&](int64_t kt, int st) {
    const int64_t k0 = kt * MK;
    double* a = As + (size_t)st * MB * SA;
#pragma unroll
    for (int e = tid; e < MB * (MK / 2); e += 256) {   // 512 chunks of 2 doubles
      const int r = e >> 3, kc = (e & 7) * 2;
      const int64_t i = i0 + r, k = k0 + kc;
      const bool ok = i < rows && k < ldm;
      cp16(a + r * SA + kc, ok ? (const void*)(mtx + i * ldm + k) : (const void*)mtx, ok);
    }
    TV* bsm = Bs + (size_t)st * MK * SB;
    constexpr int EPC = 16 / sizeof(TV);               // elements per 16-byte chunk
    constexpr int CPR = MBN / EPC;                     // chunks per k row
#pragma unroll
    for (int e = tid; e < MK * CPR; e += 256) {
      const int kr = e / CPR, cc = (e % CPR) * EPC;
      const int64_t k = k0 + kr;
      const int col = c0 + cc;
      const bool ok = k < n && col < tp;
      cp16(bsm + kr * SB + cc, ok ? (const void*)(v + k * tp + col) : (const void*)v, ok);
    }
  };
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
  for (int st = 0; st < MST - 1; ++st) {
    if (st < nk) issue(st, st);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const int fr = lane >> 2, fk = lane & 3;
  for (int64_t kt = 0; kt < nk; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(MST - 2) : "memory");
    __syncthreads();   // stage kt landed for every thread; stage kt - 1 is free for reuse
    if (kt + MST - 1 < nk) issue(kt + MST - 1, (int)((kt + MST - 1) % MST));
    asm volatile("cp.async.commit_group;" ::: "memory");
    const int st = (int)(kt % MST);
    const double* a = As + (size_t)st * MB * SA + (wm * 32 + fr) * SA + fk;
    const TV* bsm = Bs + (size_t)st * MK * SB + fk * SB + wn * 16 + fr;
#pragma unroll
    for (int kk = 0; kk < MK; kk += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int mb = 0; mb < 4; ++mb) af[mb] = a[mb * 8 * SA + kk];
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) bf[nb] = ldv<TV>(bsm + kk * SB + nb * 8);
#pragma unroll
      for (int mb = 0; mb < 4; ++mb)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(acc[mb][nb][0]), "+d"(acc[mb][nb][1])
                       : "d"(af[mb]), "d"(bf[nb]));
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  // epilogue: D fragment (row fr, columns 2 fk, 2 fk + 1 of each 8 x 8 tile); alpha partials in a
  // fixed order (m-blocks of the lane, then lanes of a column chunk, then the two warp rows)
  double cs[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int mb = 0; mb < 4; ++mb) {
    const int64_t i = i0 + wm * 32 + mb * 8 + fr;
    if (i >= rows) continue;
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      const int c = c0 + wn * 16 + nb * 8 + 2 * fk;
      if (c >= tp) continue;
      p[i * tp + c] = (TP)acc[mb][nb][0];
      p[i * tp + c + 1] = (TP)acc[mb][nb][1];
      if (apart != nullptr) {
        cs[nb][0] = fma(ldv<TV>(v + (row0 + i) * tp + c), acc[mb][nb][0], cs[nb][0]);
        cs[nb][1] = fma(ldv<TV>(v + (row0 + i) * tp + c + 1), acc[mb][nb][1], cs[nb][1]);
      }
    }
  }
  if (apart != nullptr) {
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int xo = 4; xo < 32; xo <<= 1) cs[nb][e] += __shfl_xor_sync(0xffffffffu, cs[nb][e], xo);
    __syncthreads();   // the ring is free: reuse it for the two warp rows' partials
    double* red = reinterpret_cast<double*>(smem64);   // [2][MBN]
    if (lane < 4) {
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int e = 0; e < 2; ++e) red[wm * MBN + wn * 16 + nb * 8 + 2 * lane + e] = cs[nb][e];
    }
    __syncthreads();
    if (tid < MBN && c0 + tid < tp) apart[(int64_t)rb * tp + c0 + tid] = red[tid] + red[MBN + tid];
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

template <class TV, class TP>
cudaError_t launch_mvm64_t(const double* m, int64_t ldm, int64_t rows, int64_t n, const TV* v, int tp, int64_t row0,
                           TP* p, double* apart, const Ctrl* done, cudaStream_t s) {
  const size_t smem = (size_t)MST * MB * SA * 8 + (size_t)MST * MK * SB * sizeof(TV);
  auto k = mvm64_kernel<TV, TP>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(nblk(tp, MBN), (unsigned)mvm64_blocks(rows));   // column tiles fastest: a row block's M stays in L2
  k<<<grid, 256, smem, s>>>(m, ldm, rows, n, v, tp, row0, p, apart, done);
  return cudaGetLastError();
}

cudaError_t launch_mvm64(const double* m, int64_t ldm, int64_t rows, int64_t n, const void* v, bool v_double, int tp,
                         int64_t row0, void* p, bool p_double, double* apart, const Ctrl* done, cudaStream_t s) {
  if (ldm % 2 != 0 || tp % 16 != 0) return cudaErrorInvalidValue;
  if (v_double && p_double)
    return launch_mvm64_t(m, ldm, rows, n, (const double*)v, tp, row0, (double*)p, apart, done, s);
  if (v_double) return launch_mvm64_t(m, ldm, rows, n, (const double*)v, tp, row0, (float*)p, apart, done, s);
  if (p_double) return launch_mvm64_t(m, ldm, rows, n, (const float*)v, tp, row0, (double*)p, apart, done, s);
  return launch_mvm64_t(m, ldm, rows, n, (const float*)v, tp, row0, (float*)p, apart, done, s);
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
