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
// Warp roles (384 threads): warps 0 / 2 = bulk-copy producers (features ring / V ring),
// warp 1 = TMEM allocator + single-thread MMA issuer, warps 4..11 = epilogue (TMEM lane quarter
// = warp % 4, column half = (warp - 4) / 4; two warps per SM sub-partition).  Three TMEM tile
// buffers: S(J) is overwritten IN PLACE by its k_hi|k_lo halves (32-column chunk c -> hi at
// [32c, 32c+16), lo at [32c+16, 32c+32)), the A operand of K(J).V(J); S runs three tiles ahead, so
// the tensor pipe computes KV(J-1) and S(J+2) while the epilogue exponentiates tile J.
// TMEM: buf0 | buf1 | buf2 | O (TN)  (<= 512 columns).
//
// Operand layouts (SWIZZLE_NONE canonical core matrices, 8 rows x 16 B = 128 B contiguous):
//   features  [N/8][KF/8][8][8] fp16, K-major: LBO = 128 B (K-adjacent), SBO = KF/8 * 128 B
//   V planes  [N/8][TN/8][8][8] fp16, MN-major: SBO = 128 B (N-adjacent), LBO = TN/8 * 128 B
// so every 128-row tile is one contiguous block, fetched with one bulk copy.  V is pre-split by
// pack_v_kernel with a per-column power-of-two scale (exact) so that both halves stay normal.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <stdlib.h>

#include "internal.h"
#include "tc_util.cuh"

namespace ciq {
namespace {

using namespace tc;

__device__ __forceinline__ uint64_t shfl64_d(uint64_t v) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, 0), hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), 0);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int KF = 32;           // feature contraction (3 * (d + 2) <= 32, padded)
constexpr int NUM_THREADS = 640;  // 4 role warps + 16 epilogue warps
constexpr int EPI_WARP0 = 4;
constexpr int NBUF = 3;          // TMEM S/K tile buffers (S is overwritten in place by K_hi|K_lo)
constexpr int TM_O = NBUF * 128; // O accumulator columns [384, 384 + TN)

// One smem ring, skewed by the S lookahead: stage J holds the V planes of tile J (read by KV(J))
// AND the column-point features of tile J+3 (read by S(J+3), which the MMA warp issues right after
// KV(J)), so each tile costs the MMA warp one stage wait and one stage release, and the producer
// runs STAGES tiles ahead of KV.  Features of tiles 0..2 come with the A rows in a prologue buffer.
// (The MMA warp's synchronisation count per tile is what limits the tensor pipe here: every
// mbarrier wait / tcgen05.commit on its path costs ~100 clk of issue while the tensor queue is
// shallow.)
template <int TN>
struct Cfg {
  static constexpr int FEAT_BYTES = BN * KF * 2;     // 8 KB
  static constexpr int V_BYTES = BN * TN * 2;        // one plane of one tile
  static constexpr int STAGES = 4;
  static constexpr int STAGE_BYTES = 2 * V_BYTES + FEAT_BYTES;
  static constexpr int PRO_BYTES = (1 + NBUF) * FEAT_BYTES;   // A rows + features of tiles 0..2
  static constexpr int SMEM = 1024 + PRO_BYTES + STAGES * STAGE_BYTES + 4096;
};

static_assert(Cfg<64>::SMEM <= 227 * 1024, "shared memory budget");

struct Bars {
  uint64_t full[4], empty[4];
  uint64_t s_full[NBUF], k_full[NBUF];
  uint64_t o_full, a_full;
  uint64_t probe_kv[2], probe_s[2];   // experiments only (dbg & 128): tensor-pipe completion probes
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

// 32 S values (one chunk of a row) -> 16 packed k_hi words + 16 packed k_lo words:
// k_hi = fp16(k) (round to nearest), k_lo = fp16(k - k_hi) -- k_hi + k_lo carries ~22 bits.
// (Measured alternatives, both slower: a truncation split -- k_hi = k with the low 13 mantissa
// bits cleared -- and FA4-style offload of every 4th pair to a degree-5 polynomial 2^x on the FMA
// pipe: 1.26 vs 1.14 ms, the epilogue is issue-bound as much as SFU-bound.)
template <int KIND, bool MASK>
__device__ __forceinline__ void exp_split_chunk(const uint32_t (&sv)[32], uint32_t (&hi)[16], uint32_t (&lo)[16],
                                                     int jvalid) {
#pragma unroll
  for (int c = 0; c < 32; c += 2) {
    float k0 = kernel_from_s<KIND>(__uint_as_float(sv[c]));
    float k1 = kernel_from_s<KIND>(__uint_as_float(sv[c + 1]));
    if (MASK) {
      k0 = (c < jvalid) ? k0 : 0.f;
      k1 = (c + 1 < jvalid) ? k1 : 0.f;
    }
#ifdef CIQ_EPI_TRUNC
    split_trunc2(k0, k1, hi[c / 2], lo[c / 2]);
#else
    const uint32_t h = pack_half2(k0, k1);
    const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h));
    hi[c / 2] = h;
    lo[c / 2] = pack_half2(k0 - hf.x, k1 - hf.y);
#endif
  }
}

// experiments only: per-tile clock64 stamps of CTA (0, 0) (build with CIQ_TC_TRACE=1 and run
// with CIQ_TC_DEBUG=128; compiled out otherwise -- the MMA warp's issue latency is critical)
#ifdef CIQ_TC_TRACE
#define CIQ_STAMP(slot, idx)                                                                      \
  do {                                                                                            \
    if (args.dbg_clk != nullptr && blockIdx.x == 0 && blockIdx.y == 0 && lane == 0 && (idx) < 256) \
      args.dbg_clk[(slot) * 256 + (idx)] = clock64();                                             \
  } while (0)
constexpr bool kTrace = true;
#else
#define CIQ_STAMP(slot, idx) \
  do {                       \
  } while (0)
constexpr bool kTrace = false;
#endif

template <int KIND, int TN, int CL>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    mvm_tc_kernel(TcArgs args) {
  using C = Cfg<TN>;
  if (args.done != nullptr && args.done->done) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* a_feat = smem;                              // A rows, then features of tiles 0..2
  uint8_t* ring = smem + C::PRO_BYTES;
  Bars* bars = reinterpret_cast<Bars*>(ring + C::STAGES * C::STAGE_BYTES);
  float* red = reinterpret_cast<float*>(bars + 1);  // [4][TN] alpha partial staging

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nsplit = args.nsplit;
  // Cluster of CL CTAs = CL consecutive row tiles of the same (split, chunk): they stream the same
  // column tiles J, so each producer fetches 1/CL of a stage and multicasts it to the whole cluster
  // (L2 -> SM traffic / CL).  blockIdx.x = ((rt / CL) * nsplit + split) * CL + rt % CL.
  const int crank = CL > 1 ? (int)cluster_ctarank() : 0;
  const int cgrp = blockIdx.x / CL;
  const int split = cgrp % nsplit;
  const int rt = (cgrp / nsplit) * CL + crank;
  const int chunk = blockIdx.y;
  const int64_t n = args.n;
  const int64_t i0 = args.row0 + (int64_t)rt * BM;  // global row of the tile (>= row1: padding CTA)
  const int ntiles = (int)((n + BN - 1) / BN);
  const int jt0 = (int)((int64_t)ntiles * split / nsplit), jt1 = (int)((int64_t)ntiles * (split + 1) / nsplit);
  const int njt = jt1 - jt0;
  const int npro = njt < NBUF ? njt : NBUF;         // tiles whose features come with the prologue

  if (threadIdx.x == 0) {
    // empty[s]: one arrival per CTA of the cluster (each consumer's MMA commit is multicast)
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&bars->full[s], 1); mbar_init(&bars->empty[s], CL); }
    for (int b = 0; b < NBUF; ++b) {
      mbar_init(&bars->s_full[b], 1);
      mbar_init(&bars->k_full[b], 16);  // the 16 epilogue warps
    }
    mbar_init(&bars->o_full, 1);
    mbar_init(&bars->a_full, 1);
    for (int i = 0; i < 2; ++i) { mbar_init(&bars->probe_kv[i], 1); mbar_init(&bars->probe_s[i], 1); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  fence_before_sync();
  if (CL > 1) cluster_sync();  // peers' barriers are initialised before any multicast lands
  else __syncthreads();
  fence_after_sync();
  const uint32_t tbase = bars->tmem_base;

  const size_t plane_elems = (size_t)args.npad * TN;  // one plane of one chunk
  const __half* vh = args.vplanes + (size_t)chunk * 2 * plane_elems;
  const __half* vl = vh + plane_elems;
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1);

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      // prologue (not multicast: A rows differ per CTA): A rows + features of tiles 0 .. npro-1
      mbar_arrive_expect_tx(&bars->a_full, (1 + npro) * C::FEAT_BYTES);
      const int64_t at = min(i0 / BM, args.npad / BM - 1);  // padding CTAs read a valid tile
      bulk_g2s(a_feat, args.feat_a + (size_t)at * BM * KF, C::FEAT_BYTES, &bars->a_full);
      for (int jj = 0; jj < npro; ++jj)
        bulk_g2s(a_feat + (1 + jj) * C::FEAT_BYTES, args.feat_b + (size_t)(jt0 + jj) * BN * KF, C::FEAT_BYTES,
                 &bars->a_full);
      for (int jj = 0; jj < njt; ++jj) {
        const int st = jj % C::STAGES;
        mbar_wait(&bars->empty[st], ((jj / C::STAGES) & 1) ^ 1);
        CIQ_STAMP(0, jj);
        uint8_t* sb = ring + st * C::STAGE_BYTES;
        const bool feat = jj + NBUF < njt;
        const uint8_t* gh = reinterpret_cast<const uint8_t*>(vh + (size_t)(jt0 + jj) * BN * TN);
        const uint8_t* gl = reinterpret_cast<const uint8_t*>(vl + (size_t)(jt0 + jj) * BN * TN);
        const uint8_t* gf = reinterpret_cast<const uint8_t*>(args.feat_b + (size_t)(jt0 + jj + NBUF) * BN * KF);
        // the whole stage arrives here: our slice plus (CL > 1) the peers' multicast slices
        mbar_arrive_expect_tx(&bars->full[st], 2 * C::V_BYTES + (feat ? C::FEAT_BYTES : 0));
        if (CL == 1) {
          bulk_g2s(sb, gh, C::V_BYTES, &bars->full[st]);
          bulk_g2s(sb + C::V_BYTES, gl, C::V_BYTES, &bars->full[st]);
          if (feat) bulk_g2s(sb + 2 * C::V_BYTES, gf, C::FEAT_BYTES, &bars->full[st]);
        } else {
          constexpr uint32_t vs = C::V_BYTES / CL, fs = C::FEAT_BYTES / CL;
          bulk_g2s_mc(sb + crank * vs, gh + crank * vs, vs, &bars->full[st], kMask);
          bulk_g2s_mc(sb + C::V_BYTES + crank * vs, gl + crank * vs, vs, &bars->full[st], kMask);
          if (feat) bulk_g2s_mc(sb + 2 * C::V_BYTES + crank * fs, gf + crank * fs, fs, &bars->full[st], kMask);
        }
      }
    }
  } else if (warp == 3) {
    // experiments only: completion times of KV(jj) and S(jj+3) in the tensor pipe
    if (kTrace && args.dbg_clk != nullptr && blockIdx.x == 0 && blockIdx.y == 0) {
      for (int jj = 0; jj < njt && jj < 256; ++jj) {
        mbar_wait(&bars->probe_kv[jj & 1], (jj >> 1) & 1);
        CIQ_STAMP(6, jj);
        mbar_wait(&bars->probe_s[jj & 1], (jj >> 1) & 1);
        CIQ_STAMP(7, jj);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp converged; one lane elected inside each MMA) ----
    // tensor-pipe order: S(0) S(1) S(2) | KV(0) S(3) | KV(1) S(4) | ...: S runs three tiles ahead
    // of the epilogue, KV(J) follows K(J).  Per tile: one stage wait, one k_full wait, two commits.
    {
      constexpr uint32_t idesc_s = idesc_f16(128, BN, 0, 0);   // A K-major, B K-major, N = 128
      constexpr uint32_t idesc_o = idesc_f16(128, TN, 0, 1);   // A (TMEM) K-major, B MN-major
      const uint32_t a_base = smem_u32(a_feat);
      // K-major features: LBO = 128 B (K-adjacent core), SBO = KF/8*128 B (8-row groups)
      auto issue_s = [&](int jj, uint32_t bf) {
        const uint32_t sb = tbase + (jj % NBUF) * 128;
#pragma unroll
        for (int kk = 0; kk < KF / 16; ++kk) {
          const uint64_t da = smem_desc(a_base + kk * 256, 128, (KF / 8) * 128);
          const uint64_t db = smem_desc(bf + kk * 256, 128, (KF / 8) * 128);
          mma_ss_warp(sb, da, db, idesc_s, kk > 0 ? 1u : 0u);
        }
        if (jj >= NBUF) CIQ_STAMP(8, jj - NBUF);
        mma_commit_warp(&bars->s_full[jj % NBUF]);
      };
      mbar_wait(&bars->a_full, 0);
      for (int jj = 0; jj < npro; ++jj) issue_s(jj, a_base + (1 + jj) * C::FEAT_BYTES);
      const bool probe = kTrace && args.dbg_clk != nullptr && blockIdx.x == 0 && blockIdx.y == 0;
      // Per tile jj: wait stage jj + K(jj); KV(jj) first half; then the previous stage's S(jj+2)
      // (it overwrites buffer (jj-1)%3, whose KV(jj-1) is already issued) and its release; then
      // KV(jj) second half.  The waits of tile jj+1 thus run while the tensor queue still holds
      // the second half of KV(jj), instead of while it drains.
      for (int jj = 0; jj < njt; ++jj) {
        const int b = jj % NBUF;
        const int st = jj % C::STAGES;
        const uint32_t sbase = smem_u32(ring + st * C::STAGE_BYTES);
        CIQ_STAMP(1, jj);
        mbar_wait(&bars->full[st], (jj / C::STAGES) & 1);
        CIQ_STAMP(3, jj);
        mbar_wait(&bars->k_full[b], (jj / NBUF) & 1);
        CIQ_STAMP(2, jj);
        fence_after_sync();
        const uint32_t kb = tbase + b * 128;
        const uint32_t o = tbase + TM_O;
        const uint64_t dvh0 = smem_desc(sbase, (TN / 8) * 128, 128);
        const uint64_t dvl0 = smem_desc(sbase + C::V_BYTES, (TN / 8) * 128, 128);
        auto kv_half = [&](int h) {
          if (args.dbg & 1) return;
          uint32_t kh[4], kl[4];
          uint64_t vhd[4], vld[4];
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4) {
            const int kk = 4 * h + s4;
            // K tile in place of S: chunk c = kk/2 holds k_hi pairs at [32c, 32c+16), k_lo at +16
            kh[s4] = kb + 32 * (kk >> 1) + 8 * (kk & 1);
            kl[s4] = kh[s4] + 16;
            // V: K-step of 16 rows j = 2 core-matrix rows along K (start address advances by
            // 2 * TN/8 * 128 B; descriptor start field is in 16-byte units)
            const uint64_t koff = (uint64_t)((kk * 2 * (TN / 8) * 128) >> 4);
            vhd[s4] = dvh0 + koff;
            vld[s4] = dvl0 + koff;
          }
          mma_ts_split4_warp(o, kh, kl, vhd, vld, idesc_o, (jj > 0 || h > 0) ? 1u : 0u);
        };
        kv_half(0);
        if (jj > 0) {
          const int pst = (jj - 1) % C::STAGES;
          // S(jj+2) overwrites buffer (jj-1)%3, read by KV(jj-1): tcgen05.mma instructions of one
          // thread execute in issue order, so no wait is needed.
          if (jj + 2 < njt) issue_s(jj + 2, smem_u32(ring + pst * C::STAGE_BYTES) + 2 * C::V_BYTES);
          if (probe) mma_commit_warp(&bars->probe_s[(jj - 1) & 1]);
          // the stage may be refilled once every CTA of the cluster is done with it
          if (CL == 1) mma_commit_warp(&bars->empty[pst]);
          else mma_commit_mc_warp(&bars->empty[pst], kMask);
        }
        kv_half(1);
        CIQ_STAMP(9, jj);
        if (probe) mma_commit_warp(&bars->probe_kv[jj & 1]);
      }
      if (njt > 0) {
        const int pst = (njt - 1) % C::STAGES;
        if (probe) mma_commit_warp(&bars->probe_s[(njt - 1) & 1]);
        if (CL == 1) mma_commit_warp(&bars->empty[pst]);
        else mma_commit_mc_warp(&bars->empty[pst], kMask);
      }
      mma_commit_warp(&bars->o_full);
    }
  } else if (warp >= EPI_WARP0) {
    // ---------------- epilogue: all 16 warps on every tile; warp w owns TMEM lane quarter w % 4
    // (rows 32q .. 32q+31) and the 32-column chunk cw = (w - 4) / 4 of the tile, so each SM
    // sub-partition runs four warps on the same tile (the SFU stays saturated) and a tile's K is
    // complete as early as possible -- with S three tiles ahead, the tensor pipe's KV(J) + S(J+3)
    // turnaround hides behind the exponentiation of tiles J+1, J+2.  (Two ping-pong groups of 8
    // warps on alternating tiles measured strictly serialised: each group waited for its S.) ----
    const int q = warp % 4;                         // TMEM lane quarter -> rows 32q .. 32q+31
    const int cw = (warp - EPI_WARP0) / 4;          // 32-column chunk of the tile
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    for (int jj = 0; jj < njt; ++jj) {
      const int b = jj % NBUF;
      const uint32_t tb = tbase + b * 128 + lane_base + 32 * cw;
      const int64_t jcol0 = (int64_t)(jt0 + jj) * BN + 32 * cw;
      const bool tail = jcol0 + 32 > n;
      mbar_wait(&bars->s_full[b], (jj / NBUF) & 1);
      if (warp == 4) CIQ_STAMP(4, jj);
      fence_after_sync();
      uint32_t sv[32];
      tmem_ld32(tb, sv);
      tmem_ld_wait();
      uint32_t hi[16], lo[16];
      if (args.dbg & 2) {
#pragma unroll
        for (int m = 0; m < 16; ++m) { hi[m] = sv[m]; lo[m] = sv[m + 16]; }
      } else if (tail) exp_split_chunk<KIND, true>(sv, hi, lo, (int)(n - jcol0));
      else exp_split_chunk<KIND, false>(sv, hi, lo, 32);
      // chunk c of S -> k_hi at [32c, 32c + 16), k_lo at [32c + 16, 32c + 32)
      tmem_st16(tb, hi);
      tmem_st16(tb + 16, lo);
      tmem_st_wait();
      fence_before_sync();
      __syncwarp();
      if (warp == 4) CIQ_STAMP(5, jj);
      if (lane == 0) mbar_arrive(&bars->k_full[b]);
    }
    const int c = (warp - EPI_WARP0) / 4;    // output column group for the final readout
    // ---- output: P_split = o2 * O / scale (+ diag V on split 0), alpha partials ----
    mbar_wait(&bars->o_full, 0);
    fence_after_sync();
    const int64_t i = i0 + q * 32 + lane;
    const bool row_ok = i < args.row1;
    constexpr int CPW = TN / 4;              // output columns per warp (4 warps per lane quarter)
    const int c_begin = c * CPW;
    float* pout = args.p + (size_t)split * args.p_split_stride;
    const int cglob0 = chunk * TN;
#pragma unroll
    for (int cb = 0; cb < CPW; cb += 16) {
      uint32_t o16[16];
      const int blk = (c_begin + cb) / 16 * 16;   // 16-column TMEM block containing our columns
      const int coff = (c_begin + cb) - blk;
      tmem_ld16(tbase + TM_O + lane_base + blk, o16);
      tmem_ld_wait();
      constexpr int NC = CPW < 16 ? CPW : 16;
#pragma unroll
      for (int cc = 0; cc < NC; ++cc) {
        const int col = cglob0 + c_begin + cb + cc;
        const float ov = __uint_as_float(o16[coff + cc]);
        float v = 0.f, out = 0.f;
        if (row_ok) {
          v = args.v[(size_t)i * args.tp + col];
          out = args.o2 * ov * args.inv_scale[col];
          if (split == 0) out = fmaf(args.diag, v, out);
          pout[(size_t)(i - args.row0) * args.tp + col] = out;
        }
        float part = v * out;
        part = warp_sum(part);
        if (lane == 0) red[q * TN + c_begin + cb + cc] = part;
      }
    }
  }
  fence_before_sync();
  // no CTA may exit while a peer can still multicast into its smem / arrive on its barriers
  if (CL > 1) cluster_sync();
  else __syncthreads();
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

template <int KIND, int TN, int CL>
cudaError_t launch_one(const TcArgs& a, cudaStream_t s) {
  auto k = mvm_tc_kernel<KIND, TN, CL>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<TN>::SMEM);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.nblk_x, a.tp / TN);
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = Cfg<TN>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, a);
}

template <int KIND, int TN>
cudaError_t launch_cl(const TcArgs& a, cudaStream_t s) {
  switch (a.cl) {
    case 1: return launch_one<KIND, TN, 1>(a, s);
    case 2: return launch_one<KIND, TN, 2>(a, s);
    case 4: return launch_one<KIND, TN, 4>(a, s);
  }
  return cudaErrorInvalidValue;
}

template <int KIND>
cudaError_t launch_kind(const TcArgs& a, int tn, cudaStream_t s) {
  switch (tn) {
    case 16: return launch_cl<KIND, 16>(a, s);
    case 32: return launch_cl<KIND, 32>(a, s);
    case 64: return launch_cl<KIND, 64>(a, s);
  }
  return cudaErrorInvalidValue;
}


// ============================================================================================
// Dense-K streaming MVM (SURVEY K2, §8(a) row a4 for a precomputed K): P = K V + sigma^2 V
// with K pre-split once (ciq_init) into fp16 planes K_hi + K_lo (x global power-of-two scale),
// i.e. the same 4 bytes per entry as fp32, laid out as K-major core matrices per 128 x 64 tile so
// each tile is one bulk copy.  HBM-bound: every byte of K is read once per MVM; the tensor core
// does the three split products (hi.hi + hi.lo + lo.hi) with fp32 accumulation in TMEM.
// Warps: 0 = producer (4-stage ring of K_hi | K_lo | V_hi | V_lo), 1 = MMA issuer, 4..7 = epilogue.
// ============================================================================================
constexpr int DK = 64;            // K-dim (columns j of K) per stage
constexpr int D_THREADS = 256;

template <int TN>
struct DCfg {
  static constexpr int KT_BYTES = BM * DK * 2;        // one fp16 plane of a 128 x 64 K tile (16 KB)
  static constexpr int VT_BYTES = DK * TN * 2;        // one plane of a 64-row V slab
  static constexpr int STAGE_BYTES = 2 * KT_BYTES + 2 * VT_BYTES;
#ifndef CIQ_DENSE_STAGES
#define CIQ_DENSE_STAGES 2
#endif
  static constexpr int STAGES = CIQ_DENSE_STAGES;
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 2048;
};
static_assert(DCfg<64>::SMEM <= 227 * 1024, "shared memory budget");
#ifndef CIQ_DENSE_CTAS
#define CIQ_DENSE_CTAS 2   // resident CTAs per SM (measured: 2 x 2 stages beats 1 x 4, C2 MVM -11%)
#endif


struct DBars {
  uint64_t full[CIQ_DENSE_STAGES], empty[CIQ_DENSE_STAGES];
  uint64_t o_full;
  uint32_t tmem_base;
};

template <int TN>
__global__ void __launch_bounds__(D_THREADS, CIQ_DENSE_CTAS) mvm_dense_tc_kernel(TcArgs args) {
  using C = DCfg<TN>;
  if (args.done != nullptr && args.done->done) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  DBars* bars = reinterpret_cast<DBars*>(ring + C::STAGES * C::STAGE_BYTES);
  float* red = reinterpret_cast<float*>(bars + 1);  // [4][TN]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nsplit = args.nsplit;
  const int rt = blockIdx.x / nsplit, split = blockIdx.x % nsplit;
  const int chunk = blockIdx.y;
  const int64_t n = args.n;
  const int64_t i0 = args.row0 + (int64_t)rt * BM;
  const int nkt = (int)(args.npad / DK);                      // K tiles along j (npad multiple of 128)
  const int kt0 = (int)((int64_t)nkt * split / nsplit), kt1 = (int)((int64_t)nkt * (split + 1) / nsplit);
  const int nk = kt1 - kt0;
  const int rt_local = (int)((i0 - args.row0) / BM);          // row tile within this rank's K planes
  if (threadIdx.x == 0) {
    for (int s2 = 0; s2 < C::STAGES; ++s2) { mbar_init(&bars->full[s2], 1); mbar_init(&bars->empty[s2], 1); }
    mbar_init(&bars->o_full, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<64>(&bars->tmem_base);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = bars->tmem_base;
  const size_t kplane = (size_t)args.kplane_elems;             // elements of one K plane
  const __half* kh = args.kplanes + (size_t)rt_local * nkt * BM * DK;
  const __half* kl = kh + kplane;
  const size_t vplane = (size_t)args.npad * TN;
  const __half* vh = args.vplanes + (size_t)chunk * 2 * vplane;
  const __half* vl = vh + vplane;
  if (warp == 0) {
    if (lane == 0) {
      for (int kk = 0; kk < nk; ++kk) {
        const int st = kk % C::STAGES;
        mbar_wait(&bars->empty[st], ((kk / C::STAGES) & 1) ^ 1);
        uint8_t* sb = ring + st * C::STAGE_BYTES;
        const int kt = kt0 + kk;
        mbar_arrive_expect_tx(&bars->full[st], C::STAGE_BYTES);
        bulk_g2s(sb, kh + (size_t)kt * BM * DK, C::KT_BYTES, &bars->full[st]);
        bulk_g2s(sb + C::KT_BYTES, kl + (size_t)kt * BM * DK, C::KT_BYTES, &bars->full[st]);
        // V slab of rows [64 kt, 64 kt + 64): half of the 128-row V tile (kc-major => contiguous)
        const size_t voff = (size_t)(kt / 2) * BN * TN + (size_t)(kt & 1) * DK * TN;
        bulk_g2s(sb + 2 * C::KT_BYTES, vh + voff, C::VT_BYTES, &bars->full[st]);
        bulk_g2s(sb + 2 * C::KT_BYTES + C::VT_BYTES, vl + voff, C::VT_BYTES, &bars->full[st]);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_o = idesc_f16(128, TN, 0, 1);   // A (smem) K-major, B MN-major
    for (int kk = 0; kk < nk; ++kk) {
      const int st = kk % C::STAGES;
      mbar_wait(&bars->full[st], (kk / C::STAGES) & 1);
      fence_after_sync();
      const uint32_t a_h = smem_u32(ring + st * C::STAGE_BYTES);
      const uint32_t a_l = a_h + C::KT_BYTES;
      const uint32_t v_h = a_h + 2 * C::KT_BYTES;
      const uint32_t v_l = v_h + C::VT_BYTES;
#pragma unroll
      for (int ks = 0; ks < DK / 16; ++ks) {
        // A: K-major core matrices [16 row groups][8 k chunks]: LBO = 128 B, SBO = 8*128 B; K step 256 B
        const uint64_t dah = smem_desc(a_h + ks * 256, 128, (DK / 8) * 128);
        const uint64_t dal = smem_desc(a_l + ks * 256, 128, (DK / 8) * 128);
        // B: MN-major [k chunk][n group]: LBO = TN/8*128 B, SBO = 128 B; K step 2 k-chunks
        const uint32_t koff = ks * 2 * (TN / 8) * 128;
        const uint64_t dvh = smem_desc(v_h + koff, (TN / 8) * 128, 128);
        const uint64_t dvl = smem_desc(v_l + koff, (TN / 8) * 128, 128);
        mma_ss_warp(tbase, dah, dvh, idesc_o, (kk > 0 || ks > 0) ? 1u : 0u);
        mma_ss_warp(tbase, dah, dvl, idesc_o, 1u);
        mma_ss_warp(tbase, dal, dvh, idesc_o, 1u);
      }
      mma_commit_warp(&bars->empty[st]);
    }
    mma_commit_warp(&bars->o_full);
  } else if (warp >= 4) {
    const int q = warp % 4;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    mbar_wait(&bars->o_full, 0);
    fence_after_sync();
    const int64_t i = i0 + q * 32 + lane;
    const bool row_ok = i < args.row1 && nk > 0;
    float* pout = args.p + (size_t)split * args.p_split_stride;
    const int cglob0 = chunk * TN;
#pragma unroll
    for (int cb = 0; cb < TN; cb += 16) {
      uint32_t o16[16];
      tmem_ld16(tbase + lane_base + cb, o16);
      tmem_ld_wait();
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        const int col = cglob0 + cb + cc;
        float v = 0.f, out = 0.f;
        if (i < args.row1) {
          v = args.v[(size_t)i * args.tp + col];
          out = row_ok ? __uint_as_float(o16[cc]) * args.kscale_inv * args.inv_scale[col] : 0.f;
          if (split == 0) out = fmaf(args.diag, v, out);
          pout[(size_t)(i - args.row0) * args.tp + col] = out;
        }
        float part = v * out;
        part = warp_sum(part);
        if (lane == 0) red[q * TN + cb + cc] = part;
      }
    }
  }
  fence_before_sync();
  __syncthreads();
  if (args.apart != nullptr) {
    for (int c = threadIdx.x; c < TN; c += D_THREADS) {
      double sum = 0.0;
      for (int qq = 0; qq < 4; ++qq) sum += (double)red[qq * TN + c];
      args.apart[(size_t)blockIdx.x * args.tp + chunk * TN + c] = sum;
    }
  }
  if (warp == 1) {
    fence_after_sync();
    tmem_dealloc<64>(tbase);
  }
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
  const size_t vplane = (size_t)args.npad * TN;
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
          mbar_arrive_expect_tx(&bars->full[st], C::STAGE_BYTES);
          bulk_g2s(sb, kh + (size_t)kt * BM * DK, C::KT_BYTES, &bars->full[st]);
          bulk_g2s(sb + C::KT_BYTES, kl + (size_t)kt * BM * DK, C::KT_BYTES, &bars->full[st]);
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
          mma_dense12<TN>(d, ah, ah + (C::KT_BYTES >> 4), vh, vh + (C::VT_BYTES >> 4), idesc_o, acc);
          tc_commit(&bars->empty[st]);
          if (kk == nk - 1) tc_commit(&bars->o_full[ob]);
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

// Column chunk TN per CTA.  Capped at 64: the single smem ring needs >= NBUF + 1 = 4 stages
// (S runs three tiles ahead of KV), which at TN = 128 would exceed shared memory; wider T is
// handled by more chunks (the K tile is recomputed per chunk -- cheap next to the 3 GEMMs).
int tc_cluster_size() {
  static const int cl = [] {
    const char* e = getenv("CIQ_TC_CLUSTER");
    const int v = e ? atoi(e) : 1;
    return (v == 1 || v == 2 || v == 4) ? v : 1;
  }();
  return cl;
}

int dense_ctas_per_sm() { return CIQ_DENSE_CTAS; }

int tc_chunk_cols(int tp) {
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

cudaError_t launch_mvm_dense_tc(const TcArgs& a, cudaStream_t s) {
  const int tn = tc_chunk_cols(a.tp);
  dim3 grid(a.nblk_x, a.tp / tn);
  switch (tn) {
#define CIQ_DTC_CASE(TNV)                                                                                   \
  case TNV: {                                                                                               \
    auto k = mvm_dense_tc_kernel<TNV>;                                                                      \
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, DCfg<TNV>::SMEM);   \
    if (e != cudaSuccess) return e;                                                                         \
    k<<<grid, D_THREADS, DCfg<TNV>::SMEM, s>>>(a);                                                          \
    return cudaGetLastError();                                                                              \
  }
    CIQ_DTC_CASE(16)
    CIQ_DTC_CASE(32)
    CIQ_DTC_CASE(64)
#undef CIQ_DTC_CASE
  }
  return cudaErrorInvalidValue;
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
