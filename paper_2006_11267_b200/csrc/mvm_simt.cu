// mvm_simt.cu -- fp32 CUDA-core reference MVM  P = K V + sigma^2 V.
//
// The matrix-free ("map-reduce") variant forms each 64x32 tile of K in shared memory from
// the scaled points (kernel forms of reading G11, distances from coordinate differences) and never
// writes K to HBM; the dense variant streams the given K.  The epilogue adds sigma^2 V and emits
// the per-CTA partials sum_i V[i][c] P[i][c] of the Lanczos coefficient alpha, so alpha
// needs no extra pass over P.  fp32 FMA accumulation, fixed order: deterministic.
//
// This is the correctness baseline and the fallback for shapes the tcgen05 kernel (mvm_tc.cu)
// does not cover; it is NOT the performance path for the matrix-free configs.
#include <cuda_runtime.h>

#include "internal.h"

namespace ciq {
namespace {

constexpr int BM = 64;    // rows per CTA
constexpr int BK = 32;    // K columns (j) per smem stage
constexpr int DMAX = 16;  // max point dimension

template <int KIND>
CIQ_DEVICE float kernel_of_r2(float r2, float o2) {
  if (KIND == 1) {  // RBF
    return o2 * expf(-0.5f * r2);
  } else if (KIND == 2) {  // Matern-5/2
    float r = sqrtf(r2);
    float s5 = 2.2360679774997896f * r;
    return o2 * (1.0f + s5 + s5 * s5 * (1.0f / 3.0f)) * expf(-s5);
  } else if (KIND == 3) {  // Matern-3/2
    float r = sqrtf(r2);
    float s3 = 1.7320508075688772f * r;
    return o2 * (1.0f + s3) * expf(-s3);
  } else if (KIND == 4) {  // d/dl of RBF (o2 = o^2 / l): r^2 exp(-r^2/2)
    return o2 * r2 * expf(-0.5f * r2);
  } else if (KIND == 5) {  // d/dl of Matern-5/2: a^2 (1 + a) exp(-a) / 3
    float a = 2.2360679774997896f * sqrtf(r2);
    return o2 * a * a * (1.0f + a) * (1.0f / 3.0f) * expf(-a);
  } else {  // d/dl of Matern-3/2: a^2 exp(-a)
    float a = 1.7320508075688772f * sqrtf(r2);
    return o2 * a * a * expf(-a);
  }
}

// grid: (ceil(rows/BM), tp/TN); block 256.  Thread (tr = tid/16, tc = tid%16) owns rows
// tr*4..tr*4+3 and columns tc*CW..tc*CW+CW-1 of the CTA's BM x TN output tile.
template <int KIND, int TN>
__global__ void __launch_bounds__(256) mvm_simt_kernel(OpDev op, const float* __restrict__ v, int tp,
                                                       int64_t row0, int64_t row1, float* __restrict__ p,
                                                       int ldp, double* __restrict__ apart,
                                                       const Ctrl* __restrict__ done) {
  if (done != nullptr && done->done) return;
  constexpr int CW = TN / 16;
  __shared__ float ks[BM][BK + 1];
  __shared__ float vs[BK][TN];
  __shared__ float xi[BM][DMAX];
  __shared__ float xj[BK][DMAX];
  __shared__ float red[16][TN];

  const int tid = threadIdx.x;
  const int tr = tid >> 4, tc = tid & 15;
  const int64_t i0 = row0 + (int64_t)blockIdx.x * BM;
  const int c0 = blockIdx.y * TN;
  const int64_t n = op.n;
  const int d = op.d;

  if (KIND != 0) {
    for (int e = tid; e < BM * d; e += 256) {
      int r = e / d, k = e % d;
      int64_t i = i0 + r;
      xi[r][k] = (i < row1) ? op.xs[i * d + k] : 0.f;
    }
  }
  float acc[4][CW];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < CW; ++b) acc[a][b] = 0.f;

  for (int64_t j0 = 0; j0 < n; j0 += BK) {
    __syncthreads();
    if (KIND != 0) {
      for (int e = tid; e < BK * d; e += 256) {
        int r = e / d, k = e % d;
        int64_t j = j0 + r;
        xj[r][k] = (j < n) ? op.xs[j * d + k] : 0.f;
      }
    }
    for (int e = tid; e < BK * TN; e += 256) {
      int r = e / TN, c = e % TN;
      int64_t j = j0 + r;
      vs[r][c] = (j < n) ? v[j * tp + c0 + c] : 0.f;
    }
    if (KIND == 0) {
      for (int e = tid; e < BM * BK; e += 256) {
        int r = e / BK, c = e % BK;
        int64_t i = i0 + r, j = j0 + c;
        ks[r][c] = (i < row1 && j < n) ? op.k[i * op.ldk + j] : 0.f;
      }
    }
    __syncthreads();
    if (KIND != 0) {
      for (int e = tid; e < BM * BK; e += 256) {
        int r = e / BK, c = e % BK;
        float r2 = 0.f;
        for (int k = 0; k < d; ++k) {
          float df = xi[r][k] - xj[c][k];
          r2 = fmaf(df, df, r2);
        }
        ks[r][c] = (j0 + c < n) ? kernel_of_r2<KIND>(r2, op.o2) : 0.f;
      }
      __syncthreads();
    }
#pragma unroll 8
    for (int k = 0; k < BK; ++k) {
      float a[4], b[CW];
#pragma unroll
      for (int aa = 0; aa < 4; ++aa) a[aa] = ks[tr * 4 + aa][k];
#pragma unroll
      for (int bb = 0; bb < CW; ++bb) b[bb] = vs[k][tc * CW + bb];
#pragma unroll
      for (int aa = 0; aa < 4; ++aa)
#pragma unroll
        for (int bb = 0; bb < CW; ++bb) acc[aa][bb] = fmaf(a[aa], b[bb], acc[aa][bb]);
    }
  }

  // epilogue: + sigma^2 V, store, alpha partials
  float part[CW];
#pragma unroll
  for (int bb = 0; bb < CW; ++bb) part[bb] = 0.f;
#pragma unroll
  for (int aa = 0; aa < 4; ++aa) {
    int64_t i = i0 + tr * 4 + aa;
    if (i < row1) {
#pragma unroll
      for (int bb = 0; bb < CW; ++bb) {
        int c = c0 + tc * CW + bb;
        float vi = v[i * tp + c];
        float out = fmaf(op.diag, vi, acc[aa][bb]);
        p[(i - row0) * ldp + c] = out;
        part[bb] = fmaf(vi, out, part[bb]);
      }
    }
  }
  if (apart != nullptr) {
#pragma unroll
    for (int bb = 0; bb < CW; ++bb) red[tr][tc * CW + bb] = part[bb];
    __syncthreads();
    for (int c = tid; c < TN; c += 256) {
      double s = 0.0;
      for (int r = 0; r < 16; ++r) s += (double)red[r][c];
      apart[(int64_t)blockIdx.x * tp + c0 + c] = s;
    }
  }
}

template <int KIND>
cudaError_t launch_kind(const OpDev& op, const float* v, int tp, int64_t row0, int64_t row1, float* p, int ldp,
                        double* apart, const Ctrl* done, cudaStream_t s) {
  int64_t rows = row1 - row0;
  dim3 block(256);
  if (tp % 64 == 0) {
    dim3 grid((unsigned)((rows + BM - 1) / BM), tp / 64);
    mvm_simt_kernel<KIND, 64><<<grid, block, 0, s>>>(op, v, tp, row0, row1, p, ldp, apart, done);
  } else if (tp % 32 == 0) {
    dim3 grid((unsigned)((rows + BM - 1) / BM), tp / 32);
    mvm_simt_kernel<KIND, 32><<<grid, block, 0, s>>>(op, v, tp, row0, row1, p, ldp, apart, done);
  } else {
    dim3 grid((unsigned)((rows + BM - 1) / BM), tp / 16);
    mvm_simt_kernel<KIND, 16><<<grid, block, 0, s>>>(op, v, tp, row0, row1, p, ldp, apart, done);
  }
  return cudaGetLastError();
}

// K[i - row0][j] = k(x_i, x_j) for rows [row0, row1) (fp32, no sigma^2): the materialised
// operator of the small-N / many-RHS regime (mvm_materialize, ciq_api.cu).  One thread per entry.
template <int KIND>
__global__ void materialize_kernel(OpDev op, int64_t row0, int64_t rows, float* __restrict__ k) {
  const int64_t n = op.n;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * n) return;
  const int64_t i = row0 + e / n, j = e % n;
  const float* xi = op.xs + i * op.d;
  const float* xj = op.xs + j * op.d;
  float r2 = 0.f;
  for (int t = 0; t < op.d; ++t) {
    const float dlt = xi[t] - xj[t];
    r2 = fmaf(dlt, dlt, r2);
  }
  k[e] = kernel_of_r2<KIND>(r2, op.o2);
}

}  // namespace

int mvm_simt_blocks(int64_t rows) { return (int)((rows + BM - 1) / BM); }

cudaError_t launch_mvm_simt(const OpDev& op, const float* v, int tp, int64_t row0, int64_t row1, float* p,
                            int ldp, double* apart, const Ctrl* done, cudaStream_t s) {
  if (op.kind == 4) return launch_spmm(op, v, tp, row0, row1, p, ldp, apart, done, s);   // CIQ_OP_SPARSE
  if (op.d > DMAX && op.kind != 0) return cudaErrorInvalidValue;
  if (tp % 16 != 0) return cudaErrorInvalidValue;
  switch (op.kind) {
    case 0: return launch_kind<0>(op, v, tp, row0, row1, p, ldp, apart, done, s);
    case 1: return launch_kind<1>(op, v, tp, row0, row1, p, ldp, apart, done, s);
    case 2: return launch_kind<2>(op, v, tp, row0, row1, p, ldp, apart, done, s);
    case 3: return launch_kind<3>(op, v, tp, row0, row1, p, ldp, apart, done, s);
    case 11: return launch_kind<4>(op, v, tp, row0, row1, p, ldp, apart, done, s);
    case 12: return launch_kind<5>(op, v, tp, row0, row1, p, ldp, apart, done, s);
    case 13: return launch_kind<6>(op, v, tp, row0, row1, p, ldp, apart, done, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ciq

namespace ciq {
cudaError_t launch_materialize(const OpDev& op, int64_t row0, int64_t rows, float* k, cudaStream_t s) {
  const int64_t total = rows * op.n;
  const unsigned grid = (unsigned)((total + 255) / 256);
  switch (op.kind) {
    case 1: materialize_kernel<1><<<grid, 256, 0, s>>>(op, row0, rows, k); break;
    case 2: materialize_kernel<2><<<grid, 256, 0, s>>>(op, row0, rows, k); break;
    case 3: materialize_kernel<3><<<grid, 256, 0, s>>>(op, row0, rows, k); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
}  // namespace ciq
