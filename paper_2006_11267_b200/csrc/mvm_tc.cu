// mvm_tc.cu -- the fused matrix-free kernel MVM on the 5th-generation tensor cores (SURVEY K1,
// §8(a) row a4):  P = K(X, X) V + sigma^2 V  with K never materialised in HBM.
//
// Per CTA: a 128-row block I of K and a TN-column chunk of V; it streams 128-column tiles J:
//
//   (1) S = A_I . B_J^T on tcgen05 (kind::f16, SS): augmented split-fp16 point features, so that
//       S_ij = y_i.y_j - h_i - h_j = -(log2 e / 2) ||x_i - x_j||^2 / l^2 directly (fp16x3:
//       hi.hi + lo.hi + hi.lo in one K=32 contraction; fp32 accumulate in TMEM);
//   (2) epilogue warps: tcgen05.ld S -> k = ex2(S) (RBF) or the Matern forms, masked past N ->
//       split k = k_hi + k_lo (two fp16 planes) -> tcgen05.st into a TMEM A-operand buffer;
//   (3) O += K_tile . V_J on tcgen05 (kind::f16, TS: A from TMEM, B = V_J from smem, MN-major),
//       three products k_hi.v_hi + k_hi.v_lo + k_lo.v_hi (fp32-equivalent).
//
// Warp roles (384 threads): warp 0 = bulk-copy producer (cp.async.bulk into a 4-stage ring),
// warp 1 = TMEM allocator + single-thread MMA issuer, warps 4..11 = epilogue (TMEM lane quarter
// = warp % 4, column half = (warp - 4) / 4).  Pipelining: S single-buffered (released as soon as
// it is loaded), K double-buffered, so the tensor pipe runs S(J+1) and K(J).V(J) while the
// epilogue exponentiates tile J.  TMEM: S 128 | K0 128 | K1 128 | O TN  (<= 512 columns).
//
// Operand layouts (SWIZZLE_NONE canonical core matrices, 8 rows x 16 B = 128 B contiguous):
//   features  [N/8][KF/8][8][8] fp16, K-major: LBO = 128 B (K-adjacent), SBO = KF/8 * 128 B
//   V planes  [N/8][TN/8][8][8] fp16, MN-major: SBO = 128 B (N-adjacent), LBO = TN/8 * 128 B
// so every 128-row tile is one contiguous block, fetched with one bulk copy.  V is pre-split by
// pack_v_kernel with a per-column power-of-two scale (exact) so that both halves stay normal.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "tc_util.cuh"

namespace ciq {
namespace {

using namespace tc;

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int KF = 32;           // feature contraction (3 * (d + 2) <= 32, padded)
constexpr int NUM_THREADS = 384;
constexpr int EPI_WARP0 = 4;
constexpr int TM_S = 0, TM_K0 = 128, TM_K1 = 256, TM_O = 384;

template <int TN>
struct Cfg {
  static constexpr int STAGES = (TN >= 128) ? 3 : 4;
  static constexpr int FEAT_BYTES = BN * KF * 2;     // 8 KB
  static constexpr int V_BYTES = BN * TN * 2;        // one plane of one tile
  static constexpr int STAGE_BYTES = FEAT_BYTES + 2 * V_BYTES;
  static constexpr int SMEM = 1024 + FEAT_BYTES /*A rows*/ + STAGES * STAGE_BYTES + 4096 /*misc*/;
};

struct Bars {
  uint64_t full[4], empty[4];
  uint64_t s_full, s_empty, k_full[2], k_empty[2], o_full, a_full;
  uint32_t tmem_base;
};

template <int KIND>
__device__ __forceinline__ float kernel_from_s(float s) {
  // s = -(log2 e / 2) r^2
  if (KIND == 1) return ex2_approx(s);
  const float r = sqrtf(fmaxf(0.f, -1.3862943611198906f * s));  // r^2 = -2 ln2 s
  if (KIND == 2) {
    const float a = 2.2360679774997896f * r;
    return (1.f + a + a * a * (1.f / 3.f)) * ex2_approx(-1.4426950408889634f * a);
  }
  const float a = 1.7320508075688772f * r;
  return (1.f + a) * ex2_approx(-1.4426950408889634f * a);
}

template <int KIND, int TN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    mvm_tc_kernel(TcArgs args) {
  using C = Cfg<TN>;
  if (args.done != nullptr && args.done->done) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a_feat = smem;
  uint8_t* stages = smem + C::FEAT_BYTES;
  Bars* bars = reinterpret_cast<Bars*>(stages + C::STAGES * C::STAGE_BYTES);
  float* red = reinterpret_cast<float*>(bars + 1);  // [4][TN] alpha partial staging

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nsplit = args.nsplit;
  const int rt = blockIdx.x / nsplit, split = blockIdx.x % nsplit;
  const int chunk = blockIdx.y;
  const int64_t n = args.n;
  const int64_t i0 = args.row0 + (int64_t)rt * BM;  // global row of the tile
  const int ntiles = (int)((n + BN - 1) / BN);
  const int jt0 = (int)((int64_t)ntiles * split / nsplit), jt1 = (int)((int64_t)ntiles * (split + 1) / nsplit);
  const int njt = jt1 - jt0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&bars->full[s], 1); mbar_init(&bars->empty[s], 1); }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->s_empty, 8);
    for (int b = 0; b < 2; ++b) { mbar_init(&bars->k_full[b], 8); mbar_init(&bars->k_empty[b], 1); }
    mbar_init(&bars->o_full, 1);
    mbar_init(&bars->a_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = bars->tmem_base;

  const size_t plane_elems = (size_t)args.npad * TN;  // one plane of one chunk
  const __half* vh = args.vplanes + (size_t)chunk * 2 * plane_elems;
  const __half* vl = vh + plane_elems;

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars->a_full, C::FEAT_BYTES);
      bulk_g2s(a_feat, args.feat_a + (size_t)(i0 / BM) * BM * KF, C::FEAT_BYTES, &bars->a_full);
      for (int jj = 0; jj < njt; ++jj) {
        const int st = jj % C::STAGES;
        const uint32_t use = jj / C::STAGES;
        mbar_wait(&bars->empty[st], (use & 1) ^ 1);
        uint8_t* sb = stages + st * C::STAGE_BYTES;
        const int jt = jt0 + jj;
        mbar_arrive_expect_tx(&bars->full[st], C::STAGE_BYTES);
        bulk_g2s(sb, args.feat_b + (size_t)jt * BN * KF, C::FEAT_BYTES, &bars->full[st]);
        bulk_g2s(sb + C::FEAT_BYTES, vh + (size_t)jt * BN * TN, C::V_BYTES, &bars->full[st]);
        bulk_g2s(sb + C::FEAT_BYTES + C::V_BYTES, vl + (size_t)jt * BN * TN, C::V_BYTES, &bars->full[st]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_f16(128, BN, 0, 0);   // A K-major, B K-major, N = 128
      constexpr uint32_t idesc_o = idesc_f16(128, TN, 0, 1);   // A (TMEM) K-major, B MN-major
      const uint32_t a_base = smem_u32(a_feat);
      mbar_wait(&bars->a_full, 0);
      auto issue_kv = [&](int jj) {
        const int b = jj & 1;
        mbar_wait(&bars->k_full[b], (jj >> 1) & 1);
        fence_after_sync();
        const int st = jj % C::STAGES;
        const uint32_t vh_s = smem_u32(stages + st * C::STAGE_BYTES + C::FEAT_BYTES);
        const uint32_t vl_s = vh_s + C::V_BYTES;
        const uint32_t kh = tbase + (b ? TM_K1 : TM_K0), kl = kh + 64;
        const uint32_t o = tbase + TM_O;
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          // K-step of 16 rows j = 2 core-matrix rows along K: LBO = TN/8*128 B, SBO = 128 B
          const uint32_t koff = kk * 2 * (TN / 8) * 128;
          const uint64_t dvh = smem_desc(vh_s + koff, (TN / 8) * 128, 128);
          const uint64_t dvl = smem_desc(vl_s + koff, (TN / 8) * 128, 128);
          mma_ts(o, kh + kk * 8, dvh, idesc_o, (jj > 0 || kk > 0) ? 1u : 0u);
          mma_ts(o, kh + kk * 8, dvl, idesc_o, 1u);
          mma_ts(o, kl + kk * 8, dvh, idesc_o, 1u);
        }
        mma_commit(&bars->k_empty[b]);
        mma_commit(&bars->empty[st]);
      };
      for (int jj = 0; jj < njt; ++jj) {
        const int st = jj % C::STAGES;
        mbar_wait(&bars->full[st], (jj / C::STAGES) & 1);
        mbar_wait(&bars->s_empty, (jj & 1) ^ 1);
        fence_after_sync();
        const uint32_t bf = smem_u32(stages + st * C::STAGE_BYTES);
#pragma unroll
        for (int kk = 0; kk < KF / 16; ++kk) {
          // K-major features: LBO = 128 B (K-adjacent core), SBO = KF/8*128 B (8-row groups)
          const uint64_t da = smem_desc(a_base + kk * 256, 128, (KF / 8) * 128);
          const uint64_t db = smem_desc(bf + kk * 256, 128, (KF / 8) * 128);
          mma_ss(tbase + TM_S, da, db, idesc_s, kk > 0 ? 1u : 0u);
        }
        mma_commit(&bars->s_full);
        if (jj > 0) issue_kv(jj - 1);
      }
      if (njt > 0) issue_kv(njt - 1);
      mma_commit(&bars->o_full);
    }
  } else if (warp >= EPI_WARP0) {
    // ---------------- epilogue ----------------
    const int q = warp % 4;               // TMEM lane quarter -> rows 32q .. 32q+31
    const int hsel = (warp - EPI_WARP0) / 4;  // column half of S
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    for (int jj = 0; jj < njt; ++jj) {
      const int b = jj & 1;
      const int64_t jcol0 = (int64_t)(jt0 + jj) * BN + hsel * 64;
      mbar_wait(&bars->s_full, jj & 1);
      fence_after_sync();
      uint32_t s0[32], s1[32];
      tmem_ld32(tbase + TM_S + lane_base + hsel * 64, s0);
      tmem_ld32(tbase + TM_S + lane_base + hsel * 64 + 32, s1);
      tmem_ld_wait();
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->s_empty);
      mbar_wait(&bars->k_empty[b], ((jj >> 1) & 1) ^ 1);
      fence_after_sync();
      const uint32_t kh = tbase + (b ? TM_K1 : TM_K0) + lane_base + hsel * 32;
      const uint32_t kl = kh + 64;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t* sv = half ? s1 : s0;
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          const int64_t j = jcol0 + half * 32 + c;
          float k0 = kernel_from_s<KIND>(__uint_as_float(sv[c]));
          float k1 = kernel_from_s<KIND>(__uint_as_float(sv[c + 1]));
          k0 = (j < n) ? k0 : 0.f;
          k1 = (j + 1 < n) ? k1 : 0.f;
          const uint32_t h = pack_half2(k0, k1);
          const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h));
          hi[c / 2] = h;
          lo[c / 2] = pack_half2(k0 - hf.x, k1 - hf.y);
        }
        tmem_st16(kh + half * 16, hi);
        tmem_st16(kl + half * 16, lo);
      }
      tmem_st_wait();
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->k_full[b]);
    }
    // ---- output: P_split = o2 * O / scale (+ diag V on split 0), alpha partials ----
    mbar_wait(&bars->o_full, 0);
    fence_after_sync();
    const int64_t i = i0 + q * 32 + lane;
    const bool row_ok = i < args.row1;
    const int cpw = TN / 2;  // columns per warp half
    const int c_begin = hsel * cpw;
    float* pout = args.p + (size_t)split * args.p_split_stride;
    const int cglob0 = chunk * TN;
    for (int cb = 0; cb < cpw; cb += 16) {
      uint32_t o16[16];
      if (cpw >= 16) {
        tmem_ld16(tbase + TM_O + lane_base + c_begin + cb, o16);
      } else {  // TN = 16: column half of 8 -> read 16 and keep own 8
        tmem_ld16(tbase + TM_O + lane_base + 0, o16);
      }
      tmem_ld_wait();
      const int ncols = cpw >= 16 ? 16 : cpw;
      const int coff = cpw >= 16 ? 0 : c_begin;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        if (c >= ncols) break;
        const int col = cglob0 + c_begin + cb + c;
        const float ov = __uint_as_float(o16[coff + c]);
        float v = 0.f, out = 0.f;
        if (row_ok) {
          v = args.v[(size_t)i * args.tp + col];
          out = args.o2 * ov * args.inv_scale[col];
          if (split == 0) out = fmaf(args.diag, v, out);
          pout[(size_t)(i - args.row0) * args.tp + col] = out;
        }
        float part = v * out;
        part = warp_sum(part);
        if (lane == 0) red[q * TN + c_begin + cb + c] = part;
      }
    }
  }
  fence_before_sync();
  __syncthreads();
  if (args.apart != nullptr) {
    for (int c = threadIdx.x; c < TN; c += NUM_THREADS) {
      double s = 0.0;
      for (int qq = 0; qq < 4; ++qq) s += (double)red[qq * TN + c];
      args.apart[(size_t)blockIdx.x * args.tp + chunk * TN + c] = s;
    }
  }
  if (warp == 1) {
    fence_after_sync();
    tmem_dealloc<512>(tbase);
  }
}

// ---- operand preparation ----

// V (rows x tp fp32, global rows [0, n)) -> per-chunk split planes [chunk][hi|lo][npad/8][TN/8][8][8]
// scaled per column by 2^e_c (e_c = round(log2(sqrt(n)/nrm_c))); inv_scale[c] = 2^-e_c.
__global__ void pack_v_kernel(const float* __restrict__ v, int64_t n, int64_t npad, int tp, int tn,
                              const double* __restrict__ nrm, __half* __restrict__ planes, float* __restrict__ inv_scale) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one thread per (row, 8 columns)
  const int groups = tp / 8;
  if (e >= npad * groups) return;
  const int64_t j = e / groups;
  const int g = (int)(e % groups);
  const int chunk = (g * 8) / tn;
  const int ng = (g * 8 % tn) / 8;
  float sc[8];
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int c = g * 8 + k;
    const double nr = nrm ? nrm[c] : 1.0;
    int ex = 0;
    if (nr > 0 && isfinite(nr)) ex = (int)lrint(log2(sqrt((double)n) / nr));
    ex = max(-60, min(60, ex));
    sc[k] = ldexpf(1.f, ex);
    x[k] = (j < n) ? v[j * tp + c] * sc[k] : 0.f;
    if (j == 0) inv_scale[c] = ldexpf(1.f, -ex);
  }
  uint32_t hw[4], lw[4];
#pragma unroll
  for (int k = 0; k < 8; k += 2) {
    const uint32_t h = tc::pack_half2(x[k], x[k + 1]);
    const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h));
    hw[k / 2] = h;
    lw[k / 2] = tc::pack_half2(x[k] - hf.x, x[k + 1] - hf.y);
  }
  const size_t plane = (size_t)npad * tn;
  const int64_t kc = j / 8, kk = j % 8;
  const size_t off = (size_t)chunk * 2 * plane + ((size_t)(kc * (tn / 8) + ng) * 64 + kk * 8);
  *reinterpret_cast<uint4*>(planes + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
  *reinterpret_cast<uint4*>(planes + off + plane) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
}

template <int KIND>
cudaError_t launch_kind(const TcArgs& a, int tn, cudaStream_t s) {
  dim3 grid(a.nblk_x, a.tp / tn);
  switch (tn) {
#define CIQ_TC_CASE(TNV)                                                                                   \
  case TNV: {                                                                                              \
    auto k = mvm_tc_kernel<KIND, TNV>;                                                                     \
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<TNV>::SMEM);   \
    if (e != cudaSuccess) return e;                                                                        \
    k<<<grid, NUM_THREADS, Cfg<TNV>::SMEM, s>>>(a);                                                         \
    return cudaGetLastError();                                                                             \
  }
    CIQ_TC_CASE(16)
    CIQ_TC_CASE(32)
    CIQ_TC_CASE(64)
    CIQ_TC_CASE(128)
#undef CIQ_TC_CASE
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int tc_chunk_cols(int tp) {
  if (tp % 128 == 0) return 128;
  if (tp % 64 == 0) return 64;
  if (tp % 32 == 0) return 32;
  return 16;
}

cudaError_t launch_pack_v(const float* v, int64_t n, int64_t npad, int tp, const double* nrm, __half* planes,
                          float* inv_scale, cudaStream_t s) {
  const int tn = tc_chunk_cols(tp);
  const int64_t total = npad * (tp / 8);
  pack_v_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(v, n, npad, tp, tn, nrm, planes, inv_scale);
  return cudaGetLastError();
}

cudaError_t launch_mvm_tc(const TcArgs& a, cudaStream_t s) {
  const int tn = tc_chunk_cols(a.tp);
  switch (a.kind) {
    case 1: return launch_kind<1>(a, tn, s);
    case 2: return launch_kind<2>(a, tn, s);
    case 3: return launch_kind<3>(a, tn, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ciq
