// mvm_dense.cu -- the dense-K streaming MVM on the 5th-generation tensor cores (SURVEY K2, §8(a)
// row a4 for a precomputed K) and the split-fp16 operand preparation shared by the
// tensor-core MVMs (V planes, dense K planes).
//
// Operand layouts (SWIZZLE_NONE canonical core matrices, 8 rows x 16 B = 128 B contiguous):
//   V planes   [chunk][hi|lo][N/8][TN/8][8][8] fp16, MN-major: SBO = 128 B, LBO = TN/8 * 128 B
//   K planes   [rows/128][npad/64][16][8][8][8] fp16, K-major (one 128 x 64 tile = one bulk copy)
// V is pre-split by pack_v_kernel with a per-column power-of-two scale (exact) so that both
// halves stay normal; K by split_dense_kernel with one global power-of-two scale.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "tc_util.cuh"

namespace ciq {
namespace {

using namespace tc;

constexpr int BM = 128;           // rows per dense tile (TMEM lanes)
constexpr int BN = 128;           // V-plane rows per pair of K tiles
constexpr int DK = 64;            // K-dim (columns j of K) per stage
constexpr int D_THREADS = 256;    // warp 0 producer, warp 1 MMA issuer, warps 4..7 epilogue

// a 64-bit value made warp-uniform (lane 0's), so the compiler keeps MMA descriptors in uniform
// registers (no per-MMA R2UR in the issue sequence)
__device__ __forceinline__ uint64_t shfl64_d(uint64_t v) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, 0), hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), 0);
  return ((uint64_t)hi << 32) | lo;
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

// ============================================================================================
// Dense-K streaming MVM, persistent version: one CTA per SM streams the K planes of a
// sequence of units (row tile x column split x T chunk, round-robin) through one smem ring, the
// MMA warp accumulating unit k into TMEM O[k % 2]; the epilogue warps drain O[k % 2] while unit
// k + 1 streams, so no CTA ramp or epilogue is exposed between units (HBM-bound: every byte of
// the split K planes is read once per MVM).
// ============================================================================================
template <int TN>
struct D2Cfg {
  static constexpr int KT_BYTES = BM * DK * 2;
  static constexpr int VT_BYTES = DK * TN * 2;
  static constexpr int STAGE_BYTES = 2 * KT_BYTES + 2 * VT_BYTES;
  static constexpr int STAGES = (210 * 1024) / STAGE_BYTES > 8 ? 8 : (210 * 1024) / STAGE_BYTES;
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 1024;
  static constexpr int TMEM_COLS = 2 * TN < 32 ? 32 : 2 * TN;
};
static_assert(D2Cfg<64>::STAGES >= 4, "dense ring depth");

struct D2Bars {
  uint64_t full[8], empty[8];
  uint64_t o_full[2], o_empty[2];
  uint32_t tmem_base;
};

// 12 SS MMAs of one 64-wide K tile: 4 K-steps x (K_hi.V_hi, K_hi.V_lo, K_lo.V_hi).  ah / al:
// descriptors of the K_hi / K_lo tile (K-step +16), vh / vl: V slab descriptors (K-step +2 TN).
template <int TN>
__device__ __forceinline__ void mma_dense12(uint32_t d, uint64_t ah, uint64_t al, uint64_t vh, uint64_t vl, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, t;\n\t.reg .b64 a<4>, b<4>, c<4>, e<4>;\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "setp.eq.b32 t, %5, %5;\n\t"
      "mov.b64 a0, %1;\n\t add.s64 a1, %1, 16;\n\t add.s64 a2, %1, 32;\n\t add.s64 a3, %1, 48;\n\t"
      "mov.b64 b0, %2;\n\t add.s64 b1, %2, 16;\n\t add.s64 b2, %2, 32;\n\t add.s64 b3, %2, 48;\n\t"
      "mov.b64 c0, %3;\n\t add.s64 c1, %3, %6;\n\t add.s64 c2, %3, %7;\n\t add.s64 c3, %3, %8;\n\t"
      "mov.b64 e0, %4;\n\t add.s64 e1, %4, %6;\n\t add.s64 e2, %4, %7;\n\t add.s64 e3, %4, %8;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a0, c0, %9, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a0, e0, %9, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], b0, c0, %9, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, c1, %9, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, e1, %9, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], b1, c1, %9, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, c2, %9, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, e2, %9, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], b2, c2, %9, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, c3, %9, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, e3, %9, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], b3, c3, %9, t;\n\t}" ::"r"(d),
      "l"(ah), "l"(al), "l"(vh), "l"(vl), "r"(acc), "n"(2 * TN), "n"(4 * TN), "n"(6 * TN), "r"(idesc)
      : "memory");
}

// 8 SS MMAs with K_hi only (relaxation level 2, params.mvm_relax): K_hi.V_hi, K_hi.V_lo
template <int TN>
__device__ __forceinline__ void mma_dense8(uint32_t d, uint64_t ah, uint64_t vh, uint64_t vl, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, t;\n\t.reg .b64 a<4>, c<4>, e<4>;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 t, %4, %4;\n\t"
      "mov.b64 a0, %1;\n\t add.s64 a1, %1, 16;\n\t add.s64 a2, %1, 32;\n\t add.s64 a3, %1, 48;\n\t"
      "mov.b64 c0, %2;\n\t add.s64 c1, %2, %5;\n\t add.s64 c2, %2, %6;\n\t add.s64 c3, %2, %7;\n\t"
      "mov.b64 e0, %3;\n\t add.s64 e1, %3, %5;\n\t add.s64 e2, %3, %6;\n\t add.s64 e3, %3, %7;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a0, c0, %8, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a0, e0, %8, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, c1, %8, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, e1, %8, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, c2, %8, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, e2, %8, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, c3, %8, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, e3, %8, t;\n\t}" ::"r"(d),
      "l"(ah), "l"(vh), "l"(vl), "r"(acc), "n"(2 * TN), "n"(4 * TN), "n"(6 * TN), "r"(idesc)
      : "memory");
}

__device__ __forceinline__ bool elect_one_d() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t@p mov.u32 %0, 1;\n\t}" : "+r"(pred));
  return pred != 0;
}

template <int TN>
__global__ void __launch_bounds__(D_THREADS, 1) mvm_dense2_kernel(TcArgs args) {
  using C = D2Cfg<TN>;
  if (args.done != nullptr && args.done->done) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  D2Bars* bars = reinterpret_cast<D2Bars*>(ring + C::STAGES * C::STAGE_BYTES);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nkt = (int)(args.npad / DK);
  const size_t kplane = (size_t)args.kplane_elems;
  const size_t vplane = (size_t)args.vrows * TN;
  auto unit_geom = [&](int u, int& rt, int& split, int& chunk, int& kt0, int& nk) {
    chunk = u % args.chunks;
    const int t = u / args.chunks;
    split = t % args.nsplit;
    rt = t / args.nsplit;
    kt0 = nkt * split / args.nsplit;
    nk = nkt * (split + 1) / args.nsplit - kt0;
  };
  if (threadIdx.x == 0) {
    for (int s2 = 0; s2 < C::STAGES; ++s2) { mbar_init(&bars->full[s2], 1); mbar_init(&bars->empty[s2], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&bars->o_full[b], 1); mbar_init(&bars->o_empty[b], 4); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(&bars->tmem_base);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = __shfl_sync(0xffffffffu, bars->tmem_base, 0);
  // relaxation level 2 (params.mvm_relax): K_hi only -- half the K bytes
  const bool lowp = args.gate != nullptr && *args.gate >= 2;
  if (warp == 0) {
    if (lane == 0) {
      int g = 0;
      for (int u = blockIdx.x; u < args.nunits; u += gridDim.x) {
        int rt, split, chunk, kt0, nk;
        unit_geom(u, rt, split, chunk, kt0, nk);
        const __half* kh = args.kplanes + (size_t)rt * nkt * BM * DK;   // row tile within this rank's planes
        const __half* kl = kh + kplane;
        const __half* vh = args.vplanes + (size_t)chunk * 2 * vplane;
        const __half* vl = vh + vplane;
        for (int kk = 0; kk < nk; ++kk, ++g) {
          const int st = g % C::STAGES;
          mbar_wait_backoff(&bars->empty[st], ((g / C::STAGES) & 1) ^ 1);
          uint8_t* sb = ring + st * C::STAGE_BYTES;
          const int kt = kt0 + kk;
          mbar_arrive_expect_tx(&bars->full[st], lowp ? C::STAGE_BYTES - C::KT_BYTES : C::STAGE_BYTES);
          bulk_g2s(sb, kh + (size_t)kt * BM * DK, C::KT_BYTES, &bars->full[st]);
          if (!lowp) bulk_g2s(sb + C::KT_BYTES, kl + (size_t)kt * BM * DK, C::KT_BYTES, &bars->full[st]);
          const size_t voff = (size_t)(kt / 2) * BN * TN + (size_t)(kt & 1) * DK * TN;
          bulk_g2s(sb + 2 * C::KT_BYTES, vh + voff, C::VT_BYTES, &bars->full[st]);
          bulk_g2s(sb + 2 * C::KT_BYTES + C::VT_BYTES, vl + voff, C::VT_BYTES, &bars->full[st]);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_o = idesc_f16(128, TN, 0, 1);   // A (smem) K-major, B MN-major
    // A: K-major core matrices [16 row groups][8 k chunks]: LBO = 128 B, SBO = 8 * 128 B
    // B: MN-major [k chunk][n group]: LBO = TN/8 * 128 B, SBO = 128 B
    const uint64_t dah0 = smem_desc(smem_u32(ring), 128, (DK / 8) * 128);
    const uint64_t dvh0 = smem_desc(smem_u32(ring) + 2 * C::KT_BYTES, (TN / 8) * 128, 128);
    int g = 0, st = 0, k = 0;
    uint32_t ph = 0;
    for (int u = blockIdx.x; u < args.nunits; u += gridDim.x, ++k) {
      int rt, split, chunk, kt0, nk;
      unit_geom(u, rt, split, chunk, kt0, nk);
      const int ob = k & 1;
      if (k >= 2) mbar_wait(&bars->o_empty[ob], ((k - 2) >> 1) & 1);
      const uint32_t d = __shfl_sync(0xffffffffu, tbase + ob * TN, 0);
      for (int kk = 0; kk < nk; ++kk, ++g) {
        mbar_wait(&bars->full[st], ph);
        fence_after_sync();
        const uint64_t so = (uint64_t)((st * C::STAGE_BYTES) >> 4);
        const uint64_t ah = shfl64_d(dah0 + so), vh = shfl64_d(dvh0 + so);
        const uint32_t acc = __shfl_sync(0xffffffffu, kk > 0 ? 1u : 0u, 0);
        if (elect_one_d()) {
          if (lowp) mma_dense8<TN>(d, ah, vh, vh + (C::VT_BYTES >> 4), idesc_o, acc);
          else mma_dense12<TN>(d, ah, ah + (C::KT_BYTES >> 4), vh, vh + (C::VT_BYTES >> 4), idesc_o, acc);
          mma_commit(&bars->empty[st]);
          if (kk == nk - 1) mma_commit(&bars->o_full[ob]);
        }
        __syncwarp();
        if (++st == C::STAGES) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp >= 4) {
    const int q = warp % 4;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    int k = 0;
    for (int u = blockIdx.x; u < args.nunits; u += gridDim.x, ++k) {
      int rt, split, chunk, kt0, nk;
      unit_geom(u, rt, split, chunk, kt0, nk);
      const int ob = k & 1;
      mbar_wait(&bars->o_full[ob], (k >> 1) & 1);
      fence_after_sync();
      uint32_t o[TN];
#pragma unroll
      for (int cb = 0; cb < TN; cb += 8) tmem_ld8(tbase + ob * TN + lane_base + cb, &o[cb]);
      tmem_ld_wait();
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->o_empty[ob]);
      const int64_t i = args.row0 + (int64_t)rt * BM + q * 32 + lane;
      const bool row_ok = i < args.row1;
      const int col0 = chunk * TN;
      float* pout = args.p + (size_t)split * args.p_split_stride + (size_t)(i - args.row0) * args.tp + col0;
      const float* vrow = args.v + (size_t)i * args.tp + col0;
      double* ap = args.apart ? args.apart + ((size_t)(rt * args.nsplit + split) * 4 + q) * args.tp + col0 : nullptr;
#pragma unroll
      for (int m = 0; m < TN; m += 4) {
        float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f), r4 = v4;
        if (row_ok) {
          v4 = *reinterpret_cast<const float4*>(vrow + m);
          r4.x = __uint_as_float(o[m + 0]) * args.kscale_inv * args.inv_scale[col0 + m + 0];
          r4.y = __uint_as_float(o[m + 1]) * args.kscale_inv * args.inv_scale[col0 + m + 1];
          r4.z = __uint_as_float(o[m + 2]) * args.kscale_inv * args.inv_scale[col0 + m + 2];
          r4.w = __uint_as_float(o[m + 3]) * args.kscale_inv * args.inv_scale[col0 + m + 3];
          if (split == 0) {
            r4.x = fmaf(args.diag, v4.x, r4.x); r4.y = fmaf(args.diag, v4.y, r4.y);
            r4.z = fmaf(args.diag, v4.z, r4.z); r4.w = fmaf(args.diag, v4.w, r4.w);
          }
          *reinterpret_cast<float4*>(pout + m) = r4;
        }
        if (ap != nullptr) {
          const float pv[4] = {v4.x * r4.x, v4.y * r4.y, v4.z * r4.z, v4.w * r4.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float sum = warp_sum(pv[e]);
            if (lane == 0) ap[m + e] = (double)sum;
          }
        }
      }
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    fence_after_sync();
    tmem_dealloc<C::TMEM_COLS>(tbase);
  }
}

// max |K| over the row block (non-negative floats order like their bit patterns -> atomicMax)
__global__ void absmax_kernel(const float* __restrict__ k, int64_t ldk, int64_t rows, int64_t n,
                              unsigned int* __restrict__ out) {
  float m = 0.f;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * n; e += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(k[(e / n) * ldk + e % n]));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// K (rows x n fp32, ld) * scale -> K-major split planes [rows/128][npad/64][16][8][8][8] (hi, lo)
__global__ void split_dense_kernel(const float* __restrict__ k, int64_t ldk, int64_t rows, int64_t n, int64_t npad,
                                   float scale, __half* __restrict__ hi, __half* __restrict__ lo) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // one thread per (row, 8 columns)
  const int64_t rows_pad = (rows + BM - 1) / BM * BM;
  const int64_t groups = npad / 8;
  if (e >= rows_pad * groups) return;
  const int64_t i = e / groups, g = e % groups;
  const int64_t j0 = g * 8;
  uint32_t hw[4], lw[4];
#pragma unroll
  for (int m = 0; m < 8; m += 2) {
    float x0 = 0.f, x1 = 0.f;
    if (i < rows && j0 + m < n) x0 = k[i * ldk + j0 + m] * scale;
    if (i < rows && j0 + m + 1 < n) x1 = k[i * ldk + j0 + m + 1] * scale;
    const uint32_t h = tc::pack_half2(x0, x1);
    const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h));
    hw[m / 2] = h;
    lw[m / 2] = tc::pack_half2(x0 - hf.x, x1 - hf.y);
  }
  const int64_t rt = i / BM, r = i % BM, kt = j0 / DK, kc = (j0 % DK) / 8;
  const int64_t nkt = npad / DK;
  const size_t off = ((size_t)(rt * nkt + kt) * BM * DK) + (size_t)((r / 8) * (DK / 8) + kc) * 64 + (r % 8) * 8;
  *reinterpret_cast<uint4*>(hi + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
  *reinterpret_cast<uint4*>(lo + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
}

}  // namespace

int tc_chunk_cols(int tp) {
  if (tp % 64 == 0) return 64;
  if (tp % 32 == 0) return 32;
  return 16;
}

cudaError_t launch_pack_v(const float* v, int64_t n, int64_t npad, int tp, int tn, const double* nrm, __half* planes,
                          float* inv_scale, cudaStream_t s) {
  const int64_t total = npad * (tp / 8);
  pack_v_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(v, n, npad, tp, tn, nrm, planes, inv_scale);
  return cudaGetLastError();
}

cudaError_t launch_split_dense(const float* k, int64_t ldk, int64_t rows, int64_t n, int64_t npad, float scale,
                               __half* hi, __half* lo, cudaStream_t s) {
  const int64_t rows_pad = (rows + BM - 1) / BM * BM;
  const int64_t total = rows_pad * (npad / 8);
  split_dense_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(k, ldk, rows, n, npad, scale, hi, lo);
  return cudaGetLastError();
}

cudaError_t launch_absmax(const float* k, int64_t ldk, int64_t rows, int64_t n, unsigned int* out, cudaStream_t s) {
  absmax_kernel<<<1184, 256, 0, s>>>(k, ldk, rows, n, out);
  return cudaGetLastError();
}

cudaError_t launch_mvm_dense2(const TcArgs& a, int nsm, cudaStream_t s) {
  const int tn = tc_chunk_cols(a.tp);
  const int grid = a.nunits < nsm ? a.nunits : nsm;
  switch (tn) {
#define CIQ_D2_CASE(TNV)                                                                                    \
  case TNV: {                                                                                               \
    auto k = mvm_dense2_kernel<TNV>;                                                                        \
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, D2Cfg<TNV>::SMEM);  \
    if (e != cudaSuccess) return e;                                                                         \
    k<<<grid, D_THREADS, D2Cfg<TNV>::SMEM, s>>>(a);                                                         \
    return cudaGetLastError();                                                                              \
  }
    CIQ_D2_CASE(16)
    CIQ_D2_CASE(32)
    CIQ_D2_CASE(64)
#undef CIQ_D2_CASE
  }
  return cudaErrorInvalidValue;
}

}  // namespace ciq
