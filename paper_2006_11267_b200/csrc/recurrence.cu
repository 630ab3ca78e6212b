// recurrence.cu -- the msMINRES recurrence around the MVM.
//
// Per iteration j ("a single MVM ... all subsequent operations are O(N)"; the shifted
// QR of eq. minres_qr_shifted; vectorised over shifts as P:1379 suggests):
//
//   MVM_j      P = K W_cur                       (W_cur = nrm_j v_j: Lanczos vectors are kept
//                                                 UNnormalised, the 1/nrm_j is folded in below)
//   alpha_j    alpha = (sum_blocks W_cur.P) / nrm_j^2                         [1 CTA]
//   update_j   w_j = P/nrm_j - alpha v_j - (beta_j/nrm_{j-1}) W_prev ; beta_{j+1}^2 partials
//              + the descent update of step j-1 for every shift q:
//                d_q = (v_{j-1} - delta d1_q - eps d2_q)/gamma ;  Y += w_q phi_q d_q      [stream]
//   givens_j   beta_{j+1}; per (q, column) Givens rotation of [T_j + t_q I; beta_{j+1} e_j^T];
//              coefficients of step j's update; stopping rule; invariant-subspace freeze  [1 CTA]
//
// so one streaming pass over N x T x (3Q + 6) words per iteration carries both the Lanczos step
// and all Q shifted solution updates (eq. minres_descent), and Y = sum_q w_q x_q is
// accumulated in place (eq. contour_integral_quad) -- the x_q are never stored.
// All reductions are fixed-order (fp64 across CTAs): deterministic.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "internal.h"

namespace ciq {
namespace {

constexpr int kRowsPerCta = 64;   // rows covered by one CTA of the streaming kernels
constexpr int kThreads = 256;
constexpr int kChunk = 256;       // columns per CTA (grid.y covers the rest: wide T -> more CTAs)

// Geometry of a streaming CTA: tpr threads per row (one float4 column quad each), rpp rows per pass.
struct Geo {
  int cc, tpr, rpp;
  CIQ_DEVICE Geo(int tp) {
    int c0 = blockIdx.y * kChunk;
    cc = min(kChunk, tp - c0);
    tpr = cc / 4;
    rpp = kThreads / tpr;
  }
};

// Fixed-order sum over a 256-thread CTA (warp shuffles, then warp 0 over the 8 warp sums).
CIQ_DEVICE double block_sum256(double v) {
  __shared__ double ws[8];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = (threadIdx.x < 8) ? ws[threadIdx.x] : 0.0;
  if (threadIdx.x < 32) t = warp_sum(t);
  __syncthreads();
  return t;  // valid in thread 0
}

// Fixed-order CTA reduction of per-thread column-quad partials into part[blockIdx.x][c].
CIQ_DEVICE void cta_col_reduce(const Geo& g, int tp, const double (&acc)[4], double* part) {
  __shared__ double sums[kChunk];   // rpp * tpr * 4 <= 1024
  const int tid = threadIdx.x;
  const int lane_row = tid / g.tpr, quad = tid % g.tpr;
  __syncthreads();
  for (int r = 0; r < g.rpp; ++r) {
    if (lane_row == r && lane_row < g.rpp) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        double prev = (r == 0) ? 0.0 : sums[quad * 4 + k];
        sums[quad * 4 + k] = prev + acc[k];
      }
    }
    __syncthreads();
  }
  const int c0 = blockIdx.y * kChunk;
  for (int c = tid; c < g.cc; c += kThreads) part[(int64_t)blockIdx.x * tp + c0 + c] = sums[c];
}

template <class T> struct Vec4 { T x, y, z, w; };
template <class T> CIQ_DEVICE Vec4<T> ld4(const T* p);
template <> CIQ_DEVICE Vec4<float> ld4<float>(const float* p) {
  const float4 f = *reinterpret_cast<const float4*>(p);
  return {f.x, f.y, f.z, f.w};
}
template <> CIQ_DEVICE Vec4<double> ld4<double>(const double* p) {
  const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
  return {a.x, a.y, b.x, b.y};
}
template <class T> CIQ_DEVICE void st4(T* p, const Vec4<T>& v);
template <> CIQ_DEVICE void st4<float>(float* p, const Vec4<float>& v) {
  *reinterpret_cast<float4*>(p) = make_float4(v.x, v.y, v.z, v.w);
}
template <> CIQ_DEVICE void st4<double>(double* p, const Vec4<double>& v) {
  reinterpret_cast<double2*>(p)[0] = make_double2(v.x, v.y);
  reinterpret_cast<double2*>(p)[1] = make_double2(v.z, v.w);
}

template <class T>
__global__ void __launch_bounds__(kThreads) colsq_kernel(const T* __restrict__ v, int64_t rows, int tp,
                                                         double* __restrict__ part) {
  Geo g(tp);
  const int tid = threadIdx.x;
  const int lane_row = tid / g.tpr, quad = tid % g.tpr;
  const int c = blockIdx.y * kChunk + quad * 4;
  double acc[4] = {0, 0, 0, 0};
  if (lane_row < g.rpp) {
    int64_t r0 = (int64_t)blockIdx.x * kRowsPerCta;
    for (int64_t i = r0 + lane_row; i < min(rows, r0 + kRowsPerCta); i += g.rpp) {
      const Vec4<T> x = ld4<T>(v + i * tp + c);
      acc[0] += (double)x.x * x.x; acc[1] += (double)x.y * x.y;
      acc[2] += (double)x.z * x.z; acc[3] += (double)x.w * x.w;
    }
  }
  cta_col_reduce(g, tp, acc, part);
}

// out[c] = sum_b part[b][c] in fixed order; one warp per column.  op_sqrt: out = sqrt(sum).
__global__ void reduce_cols_kernel(const double* __restrict__ part, int nblk, int m, double* __restrict__ out,
                                   int op_sqrt) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
  if (warp >= m) return;
  double s = 0.0;
  for (int b = lane; b < nblk; b += 32) s += part[(int64_t)b * m + warp];
  s = warp_sum(s);
  if (lane == 0) out[warp] = op_sqrt ? sqrt(s) : s;
}

__global__ void load_block_kernel(const float* __restrict__ src, int64_t ld, int64_t rows, int cols,
                                  float* __restrict__ dst, int tp) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * tp) return;
  int64_t i = e / tp;
  int c = (int)(e % tp);
  dst[e] = (c < cols) ? src[i * ld + c] : 0.f;
}

__global__ void store_block_kernel(const float* __restrict__ src, int tp, int64_t rows, int cols,
                                   float* __restrict__ dst, int64_t ld) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * cols) return;
  int64_t i = e / cols;
  int c = (int)(e % cols);
  dst[i * ld + c] = src[i * tp + c];
}

CIQ_DEVICE uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Counter-based N(0,1): element (global row, column) -> Box-Muller of two 53-bit uniforms.
__global__ void randn_kernel(float* __restrict__ dst, int64_t rows, int cols, int tp, int64_t row_offset,
                             uint64_t seed) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * tp) return;
  int64_t i = e / tp;
  int c = (int)(e % tp);
  if (c >= cols) { dst[e] = 0.f; return; }
  uint64_t key = seed * 0x100000001B3ull ^ ((uint64_t)(i + row_offset) << 20) ^ (uint64_t)c;
  uint64_t a = splitmix64(key), b = splitmix64(key ^ 0xD1B54A32D192ED03ull);
  double u1 = ((a >> 11) + 1.0) * (1.0 / 9007199254740993.0);
  double u2 = (b >> 11) * (1.0 / 9007199254740992.0);
  dst[e] = (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
}

__global__ void sqrt_inplace_kernel(double* __restrict__ v, int m) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) v[k] = sqrt(v[k]);
}

__global__ void scale_cols_kernel(float* __restrict__ v, int64_t rows, int tp, const double* __restrict__ nrm) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * tp) return;
  double s = nrm[e % tp];
  v[e] = (s > 0) ? (float)(v[e] / s) : 0.f;
}

__global__ void scale_cols_by_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t rows, int tp,
                                     const double* __restrict__ inv) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * tp) return;
  dst[e] = (float)(src[e] * inv[e % tp]);
}

// Initial state of a solve from colsq[c] = ||b_c||^2.
__global__ void init_state_kernel(Scal sc, int nq, int tp, const double* __restrict__ colsq) {
  for (int c = threadIdx.x; c < tp; c += blockDim.x) {
    double b1 = sqrt(colsq[c]);
    sc.beta1[c] = b1;
    sc.nrm_cur[c] = (b1 > 0) ? b1 : 1.0;
    sc.nrm_prev[c] = 1.0;
    sc.tb_cur[c] = 0.0;
    sc.alpha[c] = 0.0;
    sc.frozen[c] = (b1 > 0) ? 0 : 1;
    for (int q = 0; q < nq; ++q) {
      int k = q * tp + c;
      sc.c1[k] = 1.0; sc.s1[k] = 0.0; sc.c2[k] = 1.0; sc.s2[k] = 0.0;
      sc.phibar[k] = b1;
      sc.ca[k] = 0.f; sc.cb[k] = 0.f; sc.ce[k] = 0.f; sc.cf[k] = 0.f; sc.cphi[k] = 0.f;
      sc.da[k] = 0.0; sc.db[k] = 0.0; sc.de[k] = 0.0; sc.df[k] = 0.0;
    }
  }
  if (threadIdx.x == 0) {
    sc.ctrl->done = 0;
    sc.ctrl->iters = 0;
    sc.ctrl->pending = 0;
    sc.ctrl->breakdown = 0;
    sc.ctrl->max_relres = 0.0;
    sc.ctrl->arrive = 0;
    sc.ctrl->nonfinite = 0;
  }
}

// alpha_j = (sum_b W_cur.P partials) / nrm_j^2.  One warp per column, fixed order.
// One CTA per column c (256 threads): fixed-order reduction of the nblk partials.
__global__ void __launch_bounds__(256) alpha_kernel(Scal sc, const double* __restrict__ apart, int nblk, int tp) {
  if (sc.ctrl->done) return;
  const int c = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += 256) s += apart[(int64_t)b * tp + c];
  s = block_sum256(s);
  if (threadIdx.x == 0) {
    const double nr = sc.nrm_cur[c];
    sc.alpha[c] = sc.frozen[c] ? 0.0 : s / (nr * nr);
  }
}

// Row-sharded variant: alpha_j from the already globally summed W_cur.P (one value per column).
__global__ void alpha_from_sum_kernel(Scal sc, const double* __restrict__ sums, int tp) {
  if (sc.ctrl->done) return;
  for (int c = threadIdx.x; c < tp; c += blockDim.x) {
    const double nr = sc.nrm_cur[c];
    sc.alpha[c] = sc.frozen[c] ? 0.0 : sums[c] / (nr * nr);
  }
}

// out[k] = sum_r g[r][k] in rank order (cross-rank fixed-order sum after an allgather).
__global__ void sum_ranks_kernel(const double* __restrict__ g, int world, int m, double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  double s = 0.0;
  for (int r = 0; r < world; ++r) s += g[(size_t)r * m + k];
  out[k] = s;
}

// Split-fp16 operand planes of the next MVM, written by the streaming pass (world == 1): W_{j+1}
// scaled per column by 2^e, e = round(log2(sqrt(n) / nrm_j)) -- the norm of the CURRENT block
// stands in for beta_{j+1}, which is not known yet (any power of two that keeps both fp16 halves
// in range gives the same product: scaling by 2^e is exact).  Layout as pack_v (mvm_tc.cu):
// [chunk][hi|lo][npad/8][tn/8][8][8].
// Stored-basis output of the streaming / Givens passes (params.stored_basis): W_{j+1} to slot j of
// basis (stride elements per slot), and the step's scalars to hist = [alpha | beta_{j+1} | nrm_{j+1} |
// frozen] x [hlen][tp] at slot j - 1.  basis / hist null: not stored.
struct BasisOut {
  float* basis;
  size_t stride;
  double* hist;
  int hlen;
};

struct PackOut {
  __half* planes;      // null: no packing
  float* inv_scale;
  int64_t npad;        // plane rows
  int tn;
  double sqrt_n;
  int64_t row0;        // global row of local row 0 (row-sharded: each rank packs its rows)
};

CIQ_DEVICE float pack_scale(double nrm, double sqrt_n, float* inv) {
  int ex = 0;
  if (nrm > 0 && isfinite(nrm)) ex = (int)lrint(log2(sqrt_n / nrm));
  ex = max(-60, min(60, ex));
  *inv = ldexpf(1.f, -ex);
  return ldexpf(1.f, ex);
}

// The streaming pass (see file header).  final_only: apply the pending update of the last step
// only (wprev = the buffer holding nrm_J v_J).  Shifts are processed in batches of QB so that the
// 2 QB direction loads of a row are in flight together (the loop over shifts otherwise
// serialises on the stores to d2, which the compiler cannot reorder).
#ifndef CIQ_UPD_QB
#define CIQ_UPD_QB 2        // shifts whose d-vector loads are in flight together
#endif
#ifndef CIQ_UPD_SG
#define CIQ_UPD_SG 1        // partial-product loads grouped per iteration (A/B: scripts/ab_update_sg.sh)
#endif
#ifndef CIQ_UPD_MINB
#define CIQ_UPD_MINB 3      // resident CTAs per SM the register budget is sized for
#endif
template <class T> CIQ_DEVICE const T* coef_sel(const float* f, const double* d);
template <> CIQ_DEVICE const float* coef_sel<float>(const float* f, const double*) { return f; }
template <> CIQ_DEVICE const double* coef_sel<double>(const float*, const double* d) { return d; }

template <class T>
__global__ void __launch_bounds__(kThreads, sizeof(T) == 4 ? CIQ_UPD_MINB : 2) lanczos_update_kernel(
    Scal sc, const T* __restrict__ p, int nsplit, size_t split_stride, const T* __restrict__ wcur, const T* __restrict__ wprev,
    T* __restrict__ wnew, const T* __restrict__ d1base, T* __restrict__ d2base, int64_t qstride,
    T* __restrict__ y, int nq, int64_t rows, int tp, double* __restrict__ bpart, int final_only, PackOut pk,
    float* __restrict__ xq, BasisOut bo, int nsplit_relaxed) {
  constexpr int QB = CIQ_UPD_QB;
  constexpr bool kF32 = sizeof(T) == 4;
  const T* CA = coef_sel<T>(sc.ca, sc.da);
  const T* CB = coef_sel<T>(sc.cb, sc.db);
  const T* CE = coef_sel<T>(sc.ce, sc.de);
  const T* CF = coef_sel<T>(sc.cf, sc.df);
  const Ctrl* ctrl = sc.ctrl;
  if (!final_only && ctrl->done) return;
  const int pending = ctrl->pending;
  if (nsplit_relaxed > 0 && ctrl->relaxed) nsplit = nsplit_relaxed;   // the relaxed MVM's partial products
  // stored-basis variant: W_{j+1} also goes to basis slot j (= Givens steps done + 1; the Givens
  // pass of step j runs after this one), so no separate copy pass (store_basis) per iteration
  T* bslot = nullptr;
  if (bo.basis != nullptr && !final_only) {
    const int j = ctrl->iters + 1;
    if (j >= 1 && j < bo.hlen) bslot = reinterpret_cast<T*>(bo.basis) + (size_t)j * bo.stride;
  }
  Geo g(tp);
  const int tid = threadIdx.x;
  const int lane_row = tid / g.tpr, quad = tid % g.tpr;
  const int c = blockIdx.y * kChunk + quad * 4;
  double acc[4] = {0, 0, 0, 0};
  if (lane_row < g.rpp) {
    T inv_nrm[4], alpha[4], cprev[4];
    float psc[4];
    if (!final_only) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        int cc = c + k;
        bool fr = sc.frozen[cc] != 0;
        inv_nrm[k] = fr ? T(0) : (T)(1.0 / sc.nrm_cur[cc]);
        alpha[k] = fr ? T(0) : (T)sc.alpha[cc];
        cprev[k] = fr ? T(0) : (T)(sc.tb_cur[cc] / sc.nrm_prev[cc]);
        // scale proxy for ||W_{j+1}|| = beta_{j+1} (not known until this pass ends): beta_j for
        // j >= 2; at j = 1 (T off-diagonal beta_1 = 0) nrm_1 = ||b|| is the caller's scale, not the
        // operator's, so alpha_1 = v_1^T K v_1 stands in (beta_2^2 <= alpha_1 (lambda_max - alpha_1)
        // for PSD K, so beta_2 / alpha_1 <= sqrt(kappa): both fp16 planes stay in range)
        const double a1 = fabs(sc.alpha[cc]);
        const double proxy = (sc.tb_cur[cc] == 0.0 && a1 > 0.0) ? a1 : sc.nrm_cur[cc];
        float inv;
        psc[k] = pack_scale(proxy, pk.sqrt_n, &inv);
        if (kF32 && pk.planes != nullptr && blockIdx.x == 0 && lane_row == 0) pk.inv_scale[cc] = inv;
      }
    }
    // grid-stride over 64-row blocks: the grid is sized to the resident CTAs (update_blocks), so
    // the pass has no partial last wave; each CTA's beta^2 partials cover its fixed set of blocks
    const int64_t nrb = (rows + kRowsPerCta - 1) / kRowsPerCta;
    for (int64_t rb = blockIdx.x; rb < nrb; rb += gridDim.x) {
    const int64_t r0 = rb * kRowsPerCta;
    const int64_t r1 = min(rows, r0 + kRowsPerCta);
    for (int64_t i = r0 + lane_row; i < r1; i += g.rpp) {
      const int64_t off = i * tp + c;
      const Vec4<T> wp = ld4<T>(wprev + off);
      if (!final_only) {
        Vec4<T> pp = ld4<T>(p + off);
        // the MVM's column-split partial products, summed in split order, CIQ_UPD_SG loads in flight
        for (int sp = 1; sp < nsplit; sp += CIQ_UPD_SG) {
          Vec4<T> q4[CIQ_UPD_SG];
#pragma unroll
          for (int u = 0; u < CIQ_UPD_SG; ++u)
            if (sp + u < nsplit) q4[u] = ld4<T>(p + (sp + u) * split_stride + off);
#pragma unroll
          for (int u = 0; u < CIQ_UPD_SG; ++u)
            if (sp + u < nsplit) { pp.x += q4[u].x; pp.y += q4[u].y; pp.z += q4[u].z; pp.w += q4[u].w; }
        }
        const Vec4<T> wc = ld4<T>(wcur + off);
        Vec4<T> w;
        w.x = fma(-cprev[0], wp.x, (pp.x - alpha[0] * wc.x) * inv_nrm[0]);
        w.y = fma(-cprev[1], wp.y, (pp.y - alpha[1] * wc.y) * inv_nrm[1]);
        w.z = fma(-cprev[2], wp.z, (pp.z - alpha[2] * wc.z) * inv_nrm[2]);
        w.w = fma(-cprev[3], wp.w, (pp.w - alpha[3] * wc.w) * inv_nrm[3]);
        st4<T>(wnew + off, w);
        if (bslot != nullptr) st4<T>(bslot + off, w);
        acc[0] += (double)w.x * w.x; acc[1] += (double)w.y * w.y;
        acc[2] += (double)w.z * w.z; acc[3] += (double)w.w * w.w;
        if (kF32 && pk.planes != nullptr) {
          const float x[4] = {(float)w.x * psc[0], (float)w.y * psc[1], (float)w.z * psc[2], (float)w.w * psc[3]};
          uint32_t hw[2], lw[2];
#pragma unroll
          for (int k = 0; k < 4; k += 2) {
            const __half2 hh = __floats2half2_rn(x[k], x[k + 1]);
            const float2 hf = __half22float2(hh);
            const __half2 ll = __floats2half2_rn(x[k] - hf.x, x[k + 1] - hf.y);
            hw[k / 2] = *reinterpret_cast<const uint32_t*>(&hh);
            lw[k / 2] = *reinterpret_cast<const uint32_t*>(&ll);
          }
          const int chunk = c / pk.tn, cl = c % pk.tn;
          const size_t plane = (size_t)pk.npad * pk.tn;
          const int64_t ig = i + pk.row0;
          const size_t po = (size_t)chunk * 2 * plane + ((size_t)((ig / 8) * (pk.tn / 8) + cl / 8) * 64 + (ig % 8) * 8 + cl % 8);
          *reinterpret_cast<uint2*>(pk.planes + po) = make_uint2(hw[0], hw[1]);
          *reinterpret_cast<uint2*>(pk.planes + po + plane) = make_uint2(lw[0], lw[1]);
        }
      }
      if (pending && nq > 0) {
        Vec4<T> yy = ld4<T>(y + off);
        for (int q0 = 0; q0 < nq; q0 += QB) {
          Vec4<T> x1[QB], x2[QB];
#pragma unroll
          for (int u = 0; u < QB; ++u) {
            if (q0 + u < nq) {
              x1[u] = ld4<T>(d1base + (q0 + u) * qstride + off);
              x2[u] = ld4<T>(d2base + (q0 + u) * qstride + off);
            }
          }
#pragma unroll
          for (int u = 0; u < QB; ++u) {
            if (q0 + u < nq) {
              const int k = (q0 + u) * tp + c;
              const Vec4<T> a = ld4<T>(CA + k);
              const Vec4<T> bq = ld4<T>(CB + k);
              const Vec4<T> e = ld4<T>(CE + k);
              const Vec4<T> f = ld4<T>(CF + k);
              Vec4<T> dn;
              dn.x = fma(a.x, wp.x, fma(bq.x, x1[u].x, e.x * x2[u].x));
              dn.y = fma(a.y, wp.y, fma(bq.y, x1[u].y, e.y * x2[u].y));
              dn.z = fma(a.z, wp.z, fma(bq.z, x1[u].z, e.z * x2[u].z));
              dn.w = fma(a.w, wp.w, fma(bq.w, x1[u].w, e.w * x2[u].w));
              st4<T>(d2base + (q0 + u) * qstride + off, dn);
              if (kF32 && xq != nullptr) {   // kept per-shift solutions (backward pass)
                const Vec4<float> ph = ld4<float>(sc.cphi + k);
                Vec4<float> xx = ld4<float>(xq + (q0 + u) * qstride + off);
                xx.x = fmaf(ph.x, (float)dn.x, xx.x); xx.y = fmaf(ph.y, (float)dn.y, xx.y);
                xx.z = fmaf(ph.z, (float)dn.z, xx.z); xx.w = fmaf(ph.w, (float)dn.w, xx.w);
                st4<float>(xq + (q0 + u) * qstride + off, xx);
              }
              yy.x = fma(f.x, dn.x, yy.x); yy.y = fma(f.y, dn.y, yy.y);
              yy.z = fma(f.z, dn.z, yy.z); yy.w = fma(f.w, dn.w, yy.w);
            }
          }
        }
        st4<T>(y + off, yy);
      }
    }
    }
  }
  if (!final_only) cta_col_reduce(g, tp, acc, bpart);
}

// beta_{j+1}, Givens rotations of step j for every (shift, column), coefficients of step j's
// descent update, stopping rule.  One CTA per column (threads over shifts); per-column results
// go to col_rel / col_state and the last CTA to finish (atomic arrival count) takes the global
// decision -- max and counts are order-independent, so the outcome is deterministic.
__global__ void __launch_bounds__(256) givens_kernel(Scal sc, const double* __restrict__ bpart, int nblk, int nq,
                                                     int tp, double* __restrict__ col_rel, int* __restrict__ col_state,
                                                     BasisOut bo) {
  Ctrl* ctrl = sc.ctrl;
  if (ctrl->done) return;
  const int c = blockIdx.x;
  const int jstep = ctrl->iters + 1;   // this step (the last CTA increments ctrl->iters after every CTA read it)
  double s = 0.0;
  for (int b = threadIdx.x; b < nblk; b += 256) s += bpart[(int64_t)b * tp + c];
  s = block_sum256(s);
  __shared__ double s_tbn;
  __shared__ double s_rel[8];
  __shared__ bool s_last;
  if (threadIdx.x == 0) s_tbn = sqrt(s);
  __syncthreads();
  const double tbn = s_tbn;                      // beta_{j+1}
  const bool frozen = sc.frozen[c] != 0;
  const double a_j = sc.alpha[c], tb = sc.tb_cur[c], nrm = sc.nrm_cur[c], b1 = sc.beta1[c];
  double rel = 0.0;
  for (int q = threadIdx.x; q < nq; q += 256) {
    const int k = q * tp + c;
    if (frozen) {
      sc.ca[k] = 0.f; sc.cb[k] = 0.f; sc.ce[k] = 0.f; sc.cf[k] = 0.f; sc.cphi[k] = 0.f;
      sc.da[k] = 0.0; sc.db[k] = 0.0; sc.de[k] = 0.0; sc.df[k] = 0.0;
      continue;
    }
    const double a = a_j + sc.shifts[q];
    const double c1 = sc.c1[k], s1 = sc.s1[k], c2 = sc.c2[k], s2 = sc.s2[k];
    const double eps = s2 * tb;
    const double dp = c2 * tb;
    const double delta = c1 * dp + s1 * a;
    const double gbar = -s1 * dp + c1 * a;
    const double gamma = hypot(gbar, tbn);
    const double cs = gbar / gamma, sn = tbn / gamma;
    const double phib = sc.phibar[k];
    const double phi = cs * phib;
    const double phib_new = -sn * phib;
    sc.phibar[k] = phib_new;
    sc.ca[k] = (float)(1.0 / (gamma * nrm));   // d = (v_j - delta d1 - eps d2)/gamma, v_j = W/nrm
    sc.cb[k] = (float)(-delta / gamma);
    sc.ce[k] = (float)(-eps / gamma);
    sc.cf[k] = (float)(sc.weights[q] * phi);   // Y += w_q phi d
    sc.cphi[k] = (float)phi;                    // x_q += phi d (kept solutions)
    sc.da[k] = 1.0 / (gamma * nrm); sc.db[k] = -delta / gamma; sc.de[k] = -eps / gamma;
    sc.df[k] = sc.weights[q] * phi;
    sc.c2[k] = c1; sc.s2[k] = s1; sc.c1[k] = cs; sc.s1[k] = sn;
    const double r = fabs(phib_new) / b1;
    rel = (r <= 1e300) ? fmax(rel, r) : INFINITY;   // NaN / inf residual -> +inf (never "converged")
  }
  rel = warp_max(rel);
  if ((threadIdx.x & 31) == 0) s_rel[threadIdx.x >> 5] = rel;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) rel = fmax(rel, s_rel[w]);
    int state = 0;  // 0 frozen before, 1 active, 2 broke now
    if (!frozen) {
      const bool broke = tbn <= ctrl->bd_tol * (fabs(a_j) + tb);
      if (broke) sc.frozen[c] = 1;
      state = broke ? 2 : 1;
      sc.nrm_prev[c] = nrm;
      sc.nrm_cur[c] = broke ? 1.0 : tbn;
      sc.tb_cur[c] = tbn;
    }
    if (bo.hist != nullptr && jstep < bo.hlen) {   // stored basis: the step's scalars (slot j - 1)
      double* ha = bo.hist;                          // alpha_j
      double* hb = ha + (size_t)bo.hlen * tp;        // beta_{j+1}
      double* hn = hb + (size_t)bo.hlen * tp;        // nrm_{j+1}
      double* hf = hn + (size_t)bo.hlen * tp;        // frozen after step j
      const size_t o = (size_t)(jstep - 1) * tp + c;
      ha[o] = a_j;
      hb[o] = sc.tb_cur[c];
      hn[o] = sc.nrm_cur[c];
      hf[o] = (double)sc.frozen[c];
    }
    col_rel[c] = (state == 1) ? rel : 0.0;
    col_state[c] = state;
    __threadfence();
    s_last = atomicAdd(&ctrl->arrive, 1u) == (unsigned)tp - 1;
  }
  __syncthreads();
  if (s_last) {   // last column CTA: global decision (max / counts: order-independent), all threads
    __threadfence();
    double mx = 0.0;
    int act = 0, brk = 0;
    for (int cc = threadIdx.x; cc < tp; cc += 256) {
      const int st = ((volatile int*)col_state)[cc];
      if (st == 1) { ++act; mx = fmax(mx, ((volatile double*)col_rel)[cc]); }
      if (st == 2) ++brk;
    }
    mx = warp_max(mx);
    act = __reduce_add_sync(0xffffffffu, act);
    brk = __reduce_add_sync(0xffffffffu, brk);
    __shared__ double s_mx[8];
    __shared__ int s_act[8], s_brk[8];
    if ((threadIdx.x & 31) == 0) { s_mx[threadIdx.x >> 5] = mx; s_act[threadIdx.x >> 5] = act; s_brk[threadIdx.x >> 5] = brk; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < 8; ++w) { mx = fmax(mx, s_mx[w]); act += s_act[w]; brk += s_brk[w]; }
      const int j = ctrl->iters + 1;
      ctrl->iters = j;
      ctrl->pending = 1;
      ctrl->breakdown += brk;
      ctrl->max_relres = mx;
      ctrl->arrive = 0;
      if (!(mx <= 1e300)) ctrl->nonfinite = 1;   // stop: a NaN / inf never recovers
      // relaxed inexact Krylov (params.mvm_relax): from here on the cheaper MVM variant runs
      if (nq > 0 && ctrl->relax_thr > 0 && mx <= ctrl->relax_thr && ctrl->relaxed == 0) {
        ctrl->relaxed = 1;
        ctrl->relaxed_from = j + 1;
      }
      if (nq > 0 && ctrl->relax_thr2 > 0 && mx <= ctrl->relax_thr2 && ctrl->relaxed < 2) {
        ctrl->relaxed = 2;
        ctrl->relaxed2_from = j + 1;
      }
      if (act == 0 || (ctrl->tol > 0 && mx <= ctrl->tol) || j >= ctrl->max_iters || ctrl->nonfinite) ctrl->done = 1;
    }
  }
}

// ---- lambda-estimation Lanczos with full re-orthogonalisation ----

// part[b][k][c] = sum_{i in block b} basis_k[i][c] p[i][c],  k < nb.  basis_k = basis + k bstride.
__global__ void __launch_bounds__(kThreads) basis_dots_kernel(const float* __restrict__ basis, int64_t bstride,
                                                              int nb, int64_t rows, int tp,
                                                              const float* __restrict__ p, double* __restrict__ part) {
  // tp is small here (lanczos_cols <= 64): one thread per (row-lane, column)
  __shared__ double sh[kThreads];
  const int tid = threadIdx.x;
  const int rl = tid / tp, c = tid % tp, rpp = kThreads / tp;
  int64_t r0 = (int64_t)blockIdx.x * kRowsPerCta;
  int64_t r1 = min(rows, r0 + kRowsPerCta);
  for (int k = 0; k < nb; ++k) {
    double acc = 0.0;
    if (rl < rpp)
      for (int64_t i = r0 + rl; i < r1; i += rpp)
        acc += (double)basis[(int64_t)k * bstride + i * tp + c] * p[i * tp + c];
    sh[tid] = acc;
    __syncthreads();
    if (tid < tp) {
      double s = 0.0;
      for (int r = 0; r < rpp; ++r) s += sh[r * tp + tid];
      part[((int64_t)blockIdx.x * nb + k) * tp + tid] = s;
    }
    __syncthreads();
  }
}

__global__ void basis_axpy_kernel(const float* __restrict__ basis, int64_t bstride, int nb, int64_t rows, int tp,
                                  const double* __restrict__ h, float* __restrict__ p) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * tp) return;
  int c = (int)(e % tp);
  double s = 0.0;
  for (int k = 0; k < nb; ++k) s += h[k * tp + c] * (double)basis[(int64_t)k * bstride + e];
  p[e] = (float)(p[e] - s);
}

// alpha_j = h1[j] + h2[j] (CGS twice), beta = ||w||, breakdown per column, 1/beta for the scale.
__global__ void lanczos_coeffs_kernel(const double* __restrict__ h1, const double* __restrict__ h2,
                                      const double* __restrict__ bsq, int j, int tp, double bd_tol,
                                      double* __restrict__ alphas, double* __restrict__ betas, int* __restrict__ len,
                                      double* __restrict__ inv_beta) {
  for (int c = threadIdx.x; c < tp; c += blockDim.x) {
    double inv = 0.0;
    if (len[c] == j) {  // column still active
      double a = h1[j * tp + c] + h2[j * tp + c];
      double b = sqrt(bsq[c]);
      alphas[j * tp + c] = a;
      len[c] = j + 1;
      double bprev = (j > 0) ? betas[(j - 1) * tp + c] : 0.0;
      if (b > bd_tol * (fabs(a) + bprev)) {
        betas[j * tp + c] = b;
        inv = 1.0 / b;
      } else {
        betas[j * tp + c] = 0.0;
        len[c] = -(j + 1);   // stopped: T_J has j+1 rows
      }
    }
    inv_beta[c] = inv;
  }
}

// out = sum_s parts[s] (fixed order), float4 vectorised.
__global__ void sum_splits_kernel(const float* __restrict__ parts, int nsplit, size_t stride, int64_t n4,
                                  float* __restrict__ out, const int* __restrict__ relaxed, int nsplit_relaxed) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n4) return;
  if (relaxed != nullptr && *relaxed) nsplit = nsplit_relaxed;   // the relaxed MVM schedule's split count
  float4 acc = reinterpret_cast<const float4*>(parts)[e];
  for (int s = 1; s < nsplit; s += 4) {   // split order; 4 loads in flight
    float4 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (s + u < nsplit) q[u] = reinterpret_cast<const float4*>(parts + (s + u) * stride)[e];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (s + u < nsplit) { acc.x += q[u].x; acc.y += q[u].y; acc.z += q[u].z; acc.w += q[u].w; }
  }
  reinterpret_cast<float4*>(out)[e] = acc;
}


// ---- backward pass ----
// G[i][j] = -1/2 sum_q w_q sum_c (xv[q][i][c] xb[q][j][c] + xb[q][i][c] xv[q][j][c]): a 128 x 128
// output tile per CTA, 8 x 8 per thread (4 FMAs per shared-memory load), contraction over (q, c)
// staged through shared memory 16 columns at a time; fp32, fixed summation order (deterministic).
#ifndef CIQ_VJP_MINB
#define CIQ_VJP_MINB 2   // 2 CTAs per SM (128 registers): 2.87 -> 2.67 ms on C2 (A/B, ncu)
#endif
__global__ void __launch_bounds__(256, CIQ_VJP_MINB) vjp_dense_kernel(const float* __restrict__ xb, const float* __restrict__ xv,
                                                        const double* __restrict__ w, int nq, int64_t n, int tp,
                                                        int cols, float* __restrict__ g, int64_t ldg) {
  constexpr int TBV = 128, KS = 16;
  __shared__ float av[KS][TBV + 4], ab[KS][TBV + 4], bb[KS][TBV + 4], bv[KS][TBV + 4];
  const int64_t i0 = (int64_t)blockIdx.y * TBV, j0 = (int64_t)blockIdx.x * TBV;
  const int tid = threadIdx.x, ti = tid / 16, tj = tid % 16;
  float acc[8][8] = {};
  for (int q = 0; q < nq; ++q) {
    const float wq = (float)w[q];
    const size_t qo = (size_t)q * n * tp;
    for (int c0 = 0; c0 < cols; c0 += KS) {
      __syncthreads();
      for (int e = tid; e < KS * TBV; e += 256) {
        const int r = e / KS, cc = e % KS;   // consecutive threads read consecutive columns of a row
        const bool okc = c0 + cc < cols;
        const int64_t ii = i0 + r, jj = j0 + r;
        av[cc][r] = (okc && ii < n) ? wq * xv[qo + ii * tp + c0 + cc] : 0.f;
        ab[cc][r] = (okc && ii < n) ? wq * xb[qo + ii * tp + c0 + cc] : 0.f;
        bb[cc][r] = (okc && jj < n) ? xb[qo + jj * tp + c0 + cc] : 0.f;
        bv[cc][r] = (okc && jj < n) ? xv[qo + jj * tp + c0 + cc] : 0.f;
      }
      __syncthreads();
#pragma unroll 4
      for (int cc = 0; cc < KS; ++cc) {
        float a1[8], a2[8], b1[8], b2[8];
#pragma unroll
        for (int x = 0; x < 8; x += 4) {
          *reinterpret_cast<float4*>(&a1[x]) = *reinterpret_cast<const float4*>(&av[cc][ti * 4 + x * 16]);
          *reinterpret_cast<float4*>(&a2[x]) = *reinterpret_cast<const float4*>(&ab[cc][ti * 4 + x * 16]);
          *reinterpret_cast<float4*>(&b1[x]) = *reinterpret_cast<const float4*>(&bb[cc][tj * 4 + x * 16]);
          *reinterpret_cast<float4*>(&b2[x]) = *reinterpret_cast<const float4*>(&bv[cc][tj * 4 + x * 16]);
        }
#pragma unroll
        for (int x = 0; x < 8; ++x)
#pragma unroll
          for (int y2 = 0; y2 < 8; ++y2) acc[x][y2] = fmaf(a1[x], b1[y2], fmaf(a2[x], b2[y2], acc[x][y2]));
      }
    }
  }
  // thread (ti, tj) owns rows ti*4 + {0..3} and ti*4 + 64 + {0..3}, likewise columns
#pragma unroll
  for (int x = 0; x < 8; ++x) {
    const int64_t i = i0 + ti * 4 + (x & 3) + (x >> 2) * 64;
    if (i >= n) continue;
#pragma unroll
    for (int y2 = 0; y2 < 8; ++y2) {
      const int64_t j = j0 + tj * 4 + (y2 & 3) + (y2 >> 2) * 64;
      if (j < n) g[i * ldg + j] = -0.5f * acc[x][y2];
    }
  }
}

inline unsigned nb_elem(int64_t e, int bs) { return (unsigned)((e + bs - 1) / bs); }

}  // namespace

int rowblocks(int64_t rows, int /*tp*/) { return (int)((rows + kRowsPerCta - 1) / kRowsPerCta); }

static int sm_count_cached() {
  static const int nsm = [] {
    int v = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return nsm;
}

int update_blocks(int64_t rows) {
  const int resident = CIQ_UPD_MINB * sm_count_cached();   // __launch_bounds__(kThreads, CIQ_UPD_MINB)
  const int nrb = rowblocks(rows, 0);
  return nrb < resident ? nrb : resident;
}

int update_blocks64(int64_t rows) {
  const int resident = 2 * sm_count_cached();   // fp64 instance: __launch_bounds__(kThreads, 2)
  const int nrb = rowblocks(rows, 0);
  return nrb < resident ? nrb : resident;
}

static dim3 stream_grid(int64_t rows, int tp) {
  return dim3((unsigned)((rows + kRowsPerCta - 1) / kRowsPerCta), (unsigned)((tp + kChunk - 1) / kChunk));
}

cudaError_t launch_sum_splits(const float* parts, int nsplit, size_t stride, int64_t elems, float* out,
                              cudaStream_t s, const int* relaxed, int nsplit_relaxed) {
  const int64_t n4 = elems / 4;
  sum_splits_kernel<<<nb_elem(n4, 256), 256, 0, s>>>(parts, nsplit, stride, n4, out, relaxed, nsplit_relaxed);
  return cudaGetLastError();
}
cudaError_t launch_load_block(const float* src, int64_t ld_src, int64_t rows, int cols, float* dst, int tp,
                              cudaStream_t s) {
  load_block_kernel<<<nb_elem(rows * tp, 256), 256, 0, s>>>(src, ld_src, rows, cols, dst, tp);
  return cudaGetLastError();
}
cudaError_t launch_store_block(const float* src, int tp, int64_t rows, int cols, float* dst, int64_t ld_dst,
                               cudaStream_t s) {
  store_block_kernel<<<nb_elem(rows * cols, 256), 256, 0, s>>>(src, tp, rows, cols, dst, ld_dst);
  return cudaGetLastError();
}
cudaError_t launch_randn_fill(float* dst, int64_t rows, int cols, int tp, int64_t row_offset, uint64_t seed,
                              cudaStream_t s) {
  randn_kernel<<<nb_elem(rows * tp, 256), 256, 0, s>>>(dst, rows, cols, tp, row_offset, seed);
  return cudaGetLastError();
}
// part[blockIdx.x] = sum over this block's fixed rows (grid-stride) of sum_{c < cols} a[i][c] b[i][c],
// fp64, fixed order (the bilinear forms of the hyper-parameter gradient, ciq_hyper_grad).
__global__ void __launch_bounds__(256) dot_rows_kernel(const float* __restrict__ a, int64_t lda,
                                                       const float* __restrict__ b, int64_t ldb, int64_t rows,
                                                       int cols, double* __restrict__ part) {
  double acc = 0.0;
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * 256 + threadIdx.x; e < total; e += (int64_t)gridDim.x * 256) {
    const int64_t i = e / cols, c = e % cols;
    acc = fma((double)a[i * lda + c], (double)b[i * ldb + c], acc);
  }
  acc = block_sum256(acc);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}
int dot_rows_blocks() { return 296; }
cudaError_t launch_dot_rows(const float* a, int64_t lda, const float* b, int64_t ldb, int64_t rows, int cols,
                            double* part, cudaStream_t s) {
  dot_rows_kernel<<<dot_rows_blocks(), 256, 0, s>>>(a, lda, b, ldb, rows, cols, part);
  return cudaGetLastError();
}

cudaError_t launch_colsq_partials(const float* v, int64_t rows, int tp, double* part, cudaStream_t s) {
  colsq_kernel<float><<<stream_grid(rows, tp), kThreads, 0, s>>>(v, rows, tp, part);
  return cudaGetLastError();
}
cudaError_t launch_reduce_cols(const double* part, int nblk, int m, double* out, int op_sqrt, cudaStream_t s) {
  reduce_cols_kernel<<<nb_elem((int64_t)m * 32, 256), 256, 0, s>>>(part, nblk, m, out, op_sqrt);
  return cudaGetLastError();
}
cudaError_t launch_sqrt_inplace(double* v, int m, cudaStream_t s) {
  sqrt_inplace_kernel<<<nb_elem(m, 256), 256, 0, s>>>(v, m);
  return cudaGetLastError();
}
cudaError_t launch_scale_cols(float* v, int64_t rows, int tp, const double* nrm, cudaStream_t s) {
  scale_cols_kernel<<<nb_elem(rows * tp, 256), 256, 0, s>>>(v, rows, tp, nrm);
  return cudaGetLastError();
}
cudaError_t launch_scale_cols_by(const float* src, float* dst, int64_t rows, int tp, const double* inv,
                                 cudaStream_t s) {
  scale_cols_by_kernel<<<nb_elem(rows * tp, 256), 256, 0, s>>>(src, dst, rows, tp, inv);
  return cudaGetLastError();
}
cudaError_t launch_init_state(const Scal& sc, int nq, int tp, const double* colsq, cudaStream_t s) {
  init_state_kernel<<<1, 256, 0, s>>>(sc, nq, tp, colsq);
  return cudaGetLastError();
}
cudaError_t launch_alpha(const Scal& sc, const double* apart, int nblk, int tp, cudaStream_t s) {
  alpha_kernel<<<tp, 256, 0, s>>>(sc, apart, nblk, tp);
  return cudaGetLastError();
}
cudaError_t launch_lanczos_update(const Scal& sc, const float* p, int nsplit, size_t split_stride, const float* wcur, const float* wprev,
                                  float* wnew, float* const* d1, float* const* d2, float* y, int nq,
                                  int64_t rows, int tp, double* bpart, int final_only, cudaStream_t s,
                                  __half* planes, float* inv_scale, int64_t npad, int tn, int64_t n, float* xq,
                                  int64_t plane_row0, float* basis, size_t basis_stride, int hlen, int nsplit_relaxed) {
  const int64_t qstride = rows * tp;
  PackOut pk{planes, inv_scale, npad, tn, sqrt((double)n), plane_row0};
  dim3 grid = stream_grid(rows, tp);
  grid.x = (unsigned)update_blocks(rows);
  lanczos_update_kernel<float><<<grid, kThreads, 0, s>>>(sc, p, nsplit, split_stride, wcur, wprev, wnew, d1[0], d2[0],
                                                         qstride, y, nq, rows, tp, bpart, final_only, pk, xq,
                                                         BasisOut{basis, basis_stride, nullptr, hlen}, nsplit_relaxed);
  return cudaGetLastError();
}
cudaError_t launch_lanczos_update64(const Scal& sc, const double* p, const double* wcur, const double* wprev,
                                    double* wnew, double* const* d1, double* const* d2, double* y, int nq,
                                    int64_t rows, int tp, double* bpart, int final_only, cudaStream_t s) {
  const int64_t qstride = rows * tp;
  PackOut pk{nullptr, nullptr, 0, 0, 1.0, 0};
  dim3 grid = stream_grid(rows, tp);
  grid.x = (unsigned)update_blocks64(rows);
  lanczos_update_kernel<double><<<grid, kThreads, 0, s>>>(sc, p, 1, 0, wcur, wprev, wnew, d1[0], d2[0], qstride, y, nq,
                                                          rows, tp, bpart, final_only, pk, nullptr,
                                                          BasisOut{nullptr, 0, nullptr, 0}, 0);
  return cudaGetLastError();
}
cudaError_t launch_colsq_partials64(const double* v, int64_t rows, int tp, double* part, cudaStream_t s) {
  colsq_kernel<double><<<stream_grid(rows, tp), kThreads, 0, s>>>(v, rows, tp, part);
  return cudaGetLastError();
}
cudaError_t launch_alpha_from_sum(const Scal& sc, const double* sums, int tp, cudaStream_t s) {
  alpha_from_sum_kernel<<<1, 256, 0, s>>>(sc, sums, tp);
  return cudaGetLastError();
}
cudaError_t launch_sum_ranks(const double* g, int world, int m, double* out, cudaStream_t s) {
  sum_ranks_kernel<<<nb_elem(m, 256), 256, 0, s>>>(g, world, m, out);
  return cudaGetLastError();
}
// Stored-basis variant (x_J = Q_J y_J with the Lanczos basis
// kept): after step j's givens (ctrl->iters = j) W_{j+1} (this rank's rows) goes to basis slot j
// and the step's scalars alpha_j, beta_{j+1}, nrm_{j+1}, frozen to the history at index j - 1.
// Reads the slot from ctrl, so a captured block of iterations replays correctly.
// Y[i][c] = sum_{k < nb} coef[k][c] basis_k[i][c]  (the stored-basis solution, fp32 accumulate in
// step order like the streaming Y += w phi d)
__global__ void combine_basis_kernel(const float* __restrict__ basis, size_t stride, int nb, const float* __restrict__ coef,
                                     int64_t elems, int tp, float* __restrict__ y) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < elems; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e % tp);
    float acc = 0.f;
    for (int k = 0; k < nb; ++k) acc = fmaf(coef[(size_t)k * tp + c], basis[(size_t)k * stride + e], acc);
    y[e] = acc;
  }
}

__global__ void int_to_double_kernel(const int* __restrict__ a, int m, double* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) out[i] = (double)a[i];
}
cudaError_t launch_int_to_double(const int* a, int m, double* out, cudaStream_t s) {
  int_to_double_kernel<<<(m + 255) / 256, 256, 0, s>>>(a, m, out);
  return cudaGetLastError();
}
cudaError_t launch_combine_basis(const float* basis, size_t stride, int nb, const float* coef, int64_t elems, int tp,
                                 float* y, cudaStream_t s) {
  combine_basis_kernel<<<1184, 256, 0, s>>>(basis, stride, nb, coef, elems, tp, y);
  return cudaGetLastError();
}

cudaError_t launch_givens(const Scal& sc, const double* bpart, int nblk, int nq, int tp, cudaStream_t s, double* hist,
                          int hlen) {
  givens_kernel<<<tp, 256, 0, s>>>(sc, bpart, nblk, nq, tp, sc.col_rel, sc.col_state, BasisOut{nullptr, 0, hist, hlen});
  return cudaGetLastError();
}
cudaError_t launch_basis_dots(const float* basis, int64_t bstride, int nb, int64_t rows, int tp, const float* p,
                              double* part, cudaStream_t s) {
  if (tp > kThreads) return cudaErrorInvalidValue;
  basis_dots_kernel<<<(unsigned)((rows + kRowsPerCta - 1) / kRowsPerCta), kThreads, 0, s>>>(basis, bstride, nb,
                                                                                             rows, tp, p, part);
  return cudaGetLastError();
}
cudaError_t launch_basis_axpy(const float* basis, int64_t bstride, int nb, int64_t rows, int tp, const double* h,
                              float* p, cudaStream_t s) {
  basis_axpy_kernel<<<nb_elem(rows * tp, 256), 256, 0, s>>>(basis, bstride, nb, rows, tp, h, p);
  return cudaGetLastError();
}
cudaError_t launch_lanczos_coeffs(const double* h1, const double* h2, const double* bsq, int j, int /*nb_total*/,
                                  int tp, double bd_tol, double* alphas, double* betas, int* len, double* inv_beta,
                                  cudaStream_t s) {
  lanczos_coeffs_kernel<<<1, 256, 0, s>>>(h1, h2, bsq, j, tp, bd_tol, alphas, betas, len, inv_beta);
  return cudaGetLastError();
}

cudaError_t launch_vjp_dense(const float* xb, const float* xv, const double* w, int nq, int64_t n, int tp, int cols,
                             float* g, int64_t ldg, cudaStream_t s) {
  dim3 grid((unsigned)((n + 127) / 128), (unsigned)((n + 127) / 128));
  vjp_dense_kernel<<<grid, 256, 0, s>>>(xb, xv, w, nq, n, tp, cols, g, ldg);
  return cudaGetLastError();
}

}  // namespace ciq
