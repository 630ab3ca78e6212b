// mvm_sparse.cu -- P = A V + diag V for a sparse symmetric operator A given in CSR form (SURVEY
// §8(f) f4(iv): the stencil precision Lambda = g_obs A^T A + g_prior L^T L of the paper's Gibbs
// sampler, ~79 nonzeros per row at N = 160^2).  msMINRES-CIQ touches the operator only
// through MVMs, so the sparse path is this one kernel plus the shared recurrence.
//
// One warp per row, lanes over 32-column chunks of V (coalesced 128-byte rows of V[col][c]); the
// CSR indices / values of the row are read once per chunk (broadcast within the warp).  A block of
// 8 warps covers 64 consecutive rows and writes the fp64 partials sum_i V[i][c] P[i][c] of the
// Lanczos alpha in fixed order (same contract as mvm_simt.cu).  HBM / L2 bound: the operator
// (~8 B per nonzero) and the gathered rows of V.
#include <cuda_runtime.h>

#include "internal.h"

namespace ciq {
namespace {

constexpr int SP_ROWS = 64;   // rows per block (= mvm_simt_blocks granularity)
constexpr int SP_WARPS = 8;

// CPL: 32-column chunks a lane covers at once (2 when tp % 64 == 0: the row's CSR entries are
// fetched once for 64 columns).  The row's (index, value) pairs are loaded 32 at a time, coalesced,
// and broadcast with shuffles; the gathered V loads of successive nonzeros are independent, so the
// unrolled loop keeps several in flight (the SpMM is latency-bound on those L2 gathers).
template <int CPL>
__global__ void __launch_bounds__(256) spmm_kernel(OpDev op, const float* __restrict__ v, int tp, int64_t row0,
                                                    int64_t rows, float* __restrict__ p, int ldp,
                                                    double* __restrict__ apart, const Ctrl* __restrict__ done) {
  if (done != nullptr && done->done) return;
  __shared__ double red[SP_WARPS][32 * CPL];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b0 = (int64_t)blockIdx.x * SP_ROWS;
  for (int c0 = 0; c0 < tp; c0 += 32 * CPL) {
    double a[CPL];
#pragma unroll
    for (int u = 0; u < CPL; ++u) a[u] = 0.0;
    for (int r = warp; r < SP_ROWS; r += SP_WARPS) {
      const int64_t il = b0 + r;
      if (il >= rows) break;
      const int64_t k0 = op.rp[il], k1 = op.rp[il + 1];
      float acc[CPL][2];
#pragma unroll
      for (int u = 0; u < CPL; ++u) acc[u][0] = acc[u][1] = 0.f;
      for (int64_t kb = k0; kb < k1; kb += 32) {
        const int64_t kk = kb + lane;
        int col = 0;
        float val = 0.f;
        if (kk < k1) { col = op.ci[kk]; val = op.cv[kk]; }
        const int cnt = (int)min((int64_t)32, k1 - kb);
#pragma unroll 4
        for (int e = 0; e < cnt; ++e) {
          const int ce = __shfl_sync(0xffffffffu, col, e);
          const float ve = __shfl_sync(0xffffffffu, val, e);
          const float* vr = v + (int64_t)ce * tp + c0 + lane;
#pragma unroll
          for (int u = 0; u < CPL; ++u)
            if (c0 + lane + 32 * u < tp) acc[u][e & 1] = fmaf(ve, vr[32 * u], acc[u][e & 1]);
        }
      }
#pragma unroll
      for (int u = 0; u < CPL; ++u) {
        const int c = c0 + lane + 32 * u;
        if (c < tp) {
          const float vi = v[(row0 + il) * tp + c];
          const float res = fmaf(op.diag, vi, acc[u][0] + acc[u][1]);
          p[il * ldp + c] = res;
          a[u] += (double)vi * (double)res;
        }
      }
    }
    if (apart != nullptr) {
#pragma unroll
      for (int u = 0; u < CPL; ++u) red[warp][lane + 32 * u] = a[u];
      __syncthreads();
      if (warp == 0) {
#pragma unroll
        for (int u = 0; u < CPL; ++u) {
          const int c = c0 + lane + 32 * u;
          double sum = 0.0;
          for (int w = 0; w < SP_WARPS; ++w) sum += red[w][lane + 32 * u];
          if (c < tp) apart[(int64_t)blockIdx.x * tp + c] = sum;
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace

cudaError_t launch_spmm(const OpDev& op, const float* v, int tp, int64_t row0, int64_t row1, float* p, int ldp,
                        double* alpha_part, const Ctrl* done, cudaStream_t s) {
  const int64_t rows = row1 - row0;
  const unsigned grid = (unsigned)((rows + SP_ROWS - 1) / SP_ROWS);
  if (tp % 64 == 0) spmm_kernel<2><<<grid, SP_WARPS * 32, 0, s>>>(op, v, tp, row0, rows, p, ldp, alpha_part, done);
  else spmm_kernel<1><<<grid, SP_WARPS * 32, 0, s>>>(op, v, tp, row0, rows, p, ldp, alpha_part, done);
  return cudaGetLastError();
}

}  // namespace ciq
