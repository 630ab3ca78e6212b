// common.cuh -- shared device helpers of libciq (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define CIQ_DEVICE __device__ __forceinline__

namespace ciq {

constexpr int kWarp = 32;

CIQ_DEVICE float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
CIQ_DEVICE double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// Transposed warp reduction: lane l holds v[0..W) (one value per column, W | 32); returns to lane
// l the sum over the 32 lanes of column l % W.  W - 1 + log2(32 / W) shuffles instead of W x 5.
template <int W>
CIQ_DEVICE float warp_sum_transpose(float (&v)[W], int lane) {
#pragma unroll
  for (int s = W / 2; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int k = 0; k < s; ++k) {
      const float send = up ? v[k] : v[k + s];
      const float keep = up ? v[k + s] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  float r = v[0];
#pragma unroll
  for (int o = W; o < 32; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}
CIQ_DEVICE double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Control block of one solve (device memory).  Kernels of an iteration return immediately once
// `done` is set, so iterations launched past convergence are no-ops.
struct Ctrl {
  int done;        // 1 once the stopping rule fired (or max_iters reached)
  int iters;       // msMINRES steps whose Givens coefficients have been computed (J so far)
  int pending;     // 1 if the descent update of step `iters` has not been applied yet
  int breakdown;   // columns frozen on an invariant subspace
  int max_iters;
  int nq;
  int tp;          // padded number of columns
  unsigned int arrive;  // column-CTAs of the current givens launch that have finished (last one decides)
  double tol;
  double bd_tol;
  double max_relres;
  int nonfinite;   // 1 once a residual or beta_{j+1} came out NaN / inf (the solve stops; CIQ_NOT_CONVERGED)
  int relaxed;     // params.mvm_relax: 1 once max_relres <= relax_thr (long accumulation chains),
                   // 2 once max_relres <= relax_thr2 (also k_hi only)
  int relaxed_from;   // the first msMINRES step run at level 1 (0: none)
  int relaxed2_from;  // ... at level 2
  double relax_thr;   // 0: never
  double relax_thr2;
};

}  // namespace ciq
