// mvm_tc3.cu -- the fused matrix-free kernel MVM on CTA PAIRS (tcgen05 cta_group::2; SURVEY K1,
// §8(a) row a4):  P = K(X, X) V + sigma^2 V with K never materialised in HBM.
//
// Status (measured on B200): this kernel is the tensor-core MVM for d > 8 (feature
// contraction KF = 64, 3 (d + 2) <= 64), which the one-CTA kernel mvm_tc2.cu does not take.  For
// d <= 8 mvm_tc2.cu stays the default: at C3 this pair kernel takes 1.19 ms per MVM vs 0.95 ms.
// It was built to deepen the S look-ahead -- on a pair one M = 256 MMA covers the 128 TMEM lanes
// of both SMs, so a S/K buffer is 64 columns and six fit next to a double-buffered O -- but the
// pair runs its two epilogues in lockstep (every KV waits for the slower SM's K plus a remote
// mbarrier arrival), a single issuer blocks on the MMA queue for 12 of the 14 MMAs of a tile, and
// the tensor pipe idles ~55% (ncu, profiles/ncu_k1v3_r02.txt).  Tried and measured: four / two
// epilogue groups (1.19 / 1.28 ms), S issued before the K wait (no change), relaxed instead of
// release.cluster remote arrivals (1.31 -> 1.19 ms: a release compiles to MEMBAR.ALL.GPU).
//
// Per tile J of a unit (pair rows I = 256: rows 128 r .. 128 r + 127 on CTA r; columns J = 64):
//   (1) S = A_I . B_J^T   (kind::f16 SS, M = 256, N = 64, K = KF: augmented split-fp16 features,
//       S_ij = -(log2 e / 2) ||x_i - x_j||^2 / l^2; CTA r holds B columns 32 r .. 32 r + 31);
//   (2) epilogue warps of each CTA: tcgen05.ld S -> k = kernel(S) (ex2 on the SFU), masked past N
//       -> split k = k_hi + k_lo (fp16) -> tcgen05.st in place;
//   (3) O += K . V_J (TS: A from each CTA's TMEM; B = V_J, CTA r holding RHS columns
//       r TN/2 .. (r+1) TN/2 - 1, MN-major): k_hi.v_hi + k_hi.v_lo + k_lo.v_hi.
// TMEM (512 columns per CTA): S/K buffers b = 0..5 at [64 b, 64 b + 64), O double buffer at
// [384 + TN o, 384 + TN (o + 1)).
//
// Synchronisation across the pair: the leader (cluster rank 0) issues every MMA and commits with
// .multicast::cluster to the same barrier in both CTAs (S ready, smem stage free, O ready, A rows
// free).  Barriers the leader waits on receive arrivals from both CTAs: K ready (epilogue warps of
// both CTAs, relaxed remote arrive after tcgen05.wait::st + fence) and O drained.  The
// peer's bulk copies complete on its own barriers; a relay warp in the peer forwards each completed
// phase to the leader's barrier (stages, A rows, prologue).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "tc_util.cuh"

namespace ciq {
namespace {

using namespace tc;

constexpr int BM3 = 128;            // rows per CTA per tile (TMEM lanes); a pair covers 256
constexpr int BN3 = 64;             // columns per tile
constexpr int NT3 = 640;            // warps: 0 producer, 1 MMA (leader) / TMEM alloc, 2-3 relays (peer), 4..19 epilogue
constexpr int EPI0 = 4;
#ifndef CIQ_TC3_GROUPS
#define CIQ_TC3_GROUPS 4
#endif
// Epilogue groups: tile g goes to group g % NGRP; a group of WPG = 16 / NGRP warps covers the 4 TMEM
// lane quarters x 2 32-column chunks of a tile (NCH chunks per warp).  Fewer groups = fewer tiles
// held by the epilogue = more S look-ahead out of the NB3 buffers (NB3 - NGRP tiles).
constexpr int NGRP = CIQ_TC3_GROUPS;
static_assert(NGRP == 2 || NGRP == 4, "epilogue groups");
constexpr int WPG = 16 / NGRP;
constexpr int NCH = 8 / WPG;
constexpr int NB3 = 6;              // S/K TMEM buffers (64 columns each)
// S look-ahead: S(g + SK) is issued at step g BEFORE the issuer waits for K(g), into the buffer
// KV(g - 1) (issued at step g - 1) reads -- so S is neither queued behind KV(g) nor gated by the
// epilogue finishing tile g.
constexpr int SK = NB3 - 1;
constexpr int TMO3 = NB3 * BN3;     // O double buffer at [384, 384 + 2 TN)
constexpr int KARR = WPG * 2;       // K-ready arrivals per tile: the group's warps in both CTAs
constexpr int OARR = 16 * 2;        // O-drained arrivals per unit: 16 epilogue warps in both CTAs

template <int TN, int KF>
struct Cfg3 {
  static constexpr int TH = TN / 2;                   // RHS columns whose V planes this CTA holds
  static constexpr int A_BYTES = BM3 * KF * 2;        // this CTA's 128 rows of features
  static constexpr int F_BYTES = (BN3 / 2) * KF * 2;  // this CTA's 32 column features of a tile
  static constexpr int V_BYTES = BN3 * TH * 2;        // one plane of this CTA's V half of a tile
  static constexpr int STAGE = 2 * V_BYTES + F_BYTES;
  static constexpr int FIXED = 2 * A_BYTES + NB3 * F_BYTES;
  static constexpr int ST_RAW = (200 * 1024 - FIXED) / STAGE;
  static constexpr int STAGES = ST_RAW > 16 ? 16 : ST_RAW;
  static constexpr int RING_OFF = FIXED;
  static constexpr int SMEM = 1024 + RING_OFF + STAGES * STAGE + 1024;
};
static_assert(Cfg3<64, 32>::STAGES >= 8 && Cfg3<64, 64>::STAGES >= 8, "ring depth");
static_assert(Cfg3<64, 64>::SMEM <= 227 * 1024, "shared memory budget");

struct Bars3 {
  uint64_t full[16], empty[16];
  uint64_t s_full[NB3], k_full[NB3];
  uint64_t a_full[2], a_empty[2];
  uint64_t pro_full, o_full[2], o_empty[2];
  uint32_t tmem_base;
  uint32_t flags[16];   // per ring stage: the issuer's schedule for that tile (leader's producer)
};

enum : uint32_t {
  F_ACC = 1u << 0,      // KV accumulates into O (not the first tile of its unit)
  F_OLAST = 1u << 1,    // last tile of its unit: commit o_full[F_OB] after KV
  F_OWAIT = 1u << 2,    // first tile of a unit k >= 2: wait o_empty[F_OB] (phase F_OPH)
  F_OPH = 1u << 3,
  F_SVALID = 1u << 4,   // S(g + SK) exists
  F_SFIRST = 1u << 5,   // S(g + SK) is the first tile of its unit: wait a_full[F_KB] (phase F_APH)
  F_APH = 1u << 6,
  F_SLAST = 1u << 7,    // S(g + SK) is the last tile of its unit: commit a_empty[F_KB]
  F_KB = 1u << 8,       // A-rows buffer of S(g + SK)'s unit
  F_OB = 1u << 9,       // O buffer of KV(g)'s unit
};

// Position in the flattened tile sequence of one CTA pair: unit u (local index k), tile jj of njt.
struct Cur3 {
  int k, u, jj, njt, jt0, split, chunk, rt;
  CIQ_DEVICE void decode(const TcArgs& a, int ntiles) {
    chunk = u % a.chunks;
    const int t = u / a.chunks;
    split = t % a.nsplit;
    rt = t / a.nsplit;
    jt0 = ntiles * split / a.nsplit;
    njt = ntiles * (split + 1) / a.nsplit - jt0;
  }
  CIQ_DEVICE void start(const TcArgs& a, int ntiles) {
    k = 0;
    u = blockIdx.x / 2;
    jj = 0;
    if (u < a.nunits) decode(a, ntiles);
  }
  CIQ_DEVICE bool valid(const TcArgs& a) const { return u < a.nunits; }
  CIQ_DEVICE void advance(const TcArgs& a, int ntiles) {
    if (++jj == njt) {
      jj = 0;
      ++k;
      u += gridDim.x / 2;
      if (u < a.nunits) decode(a, ntiles);
    }
  }
  CIQ_DEVICE int J() const { return jt0 + jj; }
};

CIQ_DEVICE bool elect_one3() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t@p mov.u32 %0, 1;\n\t}" : "+r"(pred));
  return pred != 0;
}

// experiments only (-DCIQ_TC_TRACE, env CIQ_TC_DEBUG=128): clock64 stamps of pair 0 per tile
// (each SM's own clock: leader and peer columns are not comparable), printed by run_mvm
#ifdef CIQ_TC_TRACE
#define T3_STAMP(slot, idx)                                                                        \
  do {                                                                                             \
    if (args.dbg_clk != nullptr && blockIdx.x < 2 && (idx) < 256)                                  \
      args.dbg_clk[(slot) * 256 + (idx)] = clock64();                                              \
  } while (0)
#else
#define T3_STAMP(slot, idx) \
  do {                      \
  } while (0)
#endif

// arrive on the barrier at the same offset in both CTAs of the pair once the issued MMAs complete
CIQ_DEVICE void commit_pair(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "h"((uint16_t)3)
               : "memory");
}

CIQ_DEVICE uint64_t shfl64_3(uint64_t v) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, 0), hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), 0);
  return ((uint64_t)hi << 32) | lo;
}

template <int KIND>
CIQ_DEVICE float kern3(float s) {
  // s = -(log2 e / 2) r^2; KIND 4-6: lengthscale derivatives (as kern in mvm_tc2.cu)
  if (KIND == 1) return ex2_approx(s);
  if (KIND == 4) return (-1.3862943611198906f * s) * ex2_approx(s);
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(fmaxf(0.f, -1.3862943611198906f * s)));
  if (KIND == 2) {
    const float a = 2.2360679774997896f * r;
    return (1.f + a + a * a * (1.f / 3.f)) * ex2_approx(-1.4426950408889634f * a);
  }
  if (KIND == 5) {
    const float a = 2.2360679774997896f * r;
    return a * a * (1.f + a) * (1.f / 3.f) * ex2_approx(-1.4426950408889634f * a);
  }
  const float a = 1.7320508075688772f * r;
  if (KIND == 6) return a * a * ex2_approx(-1.4426950408889634f * a);
  return (1.f + a) * ex2_approx(-1.4426950408889634f * a);
}

// 32 S values -> 16 packed k_hi words + 16 packed k_lo words (truncation split, as mvm_tc2.cu)
template <int KIND, bool MASK>
CIQ_DEVICE void exp_split3(const uint32_t (&sv)[32], uint32_t (&hi)[16], uint32_t (&lo)[16], int jvalid) {
#pragma unroll
  for (int c = 0; c < 32; c += 2) {
    float k0 = kern3<KIND>(__uint_as_float(sv[c]));
    float k1 = kern3<KIND>(__uint_as_float(sv[c + 1]));
    if (MASK) {
      k0 = (c < jvalid) ? k0 : 0.f;
      k1 = (c + 1 < jvalid) ? k1 : 0.f;
    }
    split_trunc2(k0, k1, hi[c / 2], lo[c / 2]);
  }
}

// S of a pair tile: KF/16 SS MMAs (M = 256, N = 64), K-step = +256 B = +16 descriptor units.
template <int KF>
CIQ_DEVICE void mma_s3(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc) {
  if (KF == 32) {
    asm volatile(
        "{\n\t.reg .pred t, f;\n\t.reg .b64 a1, b1;\n\t"
        "setp.ne.b32 t, %3, 0;\n\tsetp.eq.b32 f, %3, 0;\n\t"
        "add.s64 a1, %1, 16;\n\tadd.s64 b1, %2, 16;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, f;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, t;\n\t}" ::"r"(d),
        "l"(da), "l"(db), "r"(idesc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred t, f;\n\t.reg .b64 a1, b1, a2, b2, a3, b3;\n\t"
        "setp.ne.b32 t, %3, 0;\n\tsetp.eq.b32 f, %3, 0;\n\t"
        "add.s64 a1, %1, 16;\n\tadd.s64 b1, %2, 16;\n\t"
        "add.s64 a2, %1, 32;\n\tadd.s64 b2, %2, 32;\n\t"
        "add.s64 a3, %1, 48;\n\tadd.s64 b3, %2, 48;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, f;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, t;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, t;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, t;\n\t}" ::"r"(d),
        "l"(da), "l"(db), "r"(idesc)
        : "memory");
  }
}

// KV of a pair tile: O (+)= K . V_J, 4 K-steps x (k_hi.v_hi, k_hi.v_lo, k_lo.v_hi) = 12 TS MMAs.
// kb: TMEM K buffer (K-step s -> k_hi at 32 (s/2) + 8 (s%2), k_lo at +16); dv: V_hi descriptor of
// the stage (this CTA's TH columns; V_lo at +8 TH, K-step s at +2 TH s descriptor units).
template <int TH>
CIQ_DEVICE void mma_kv3(uint32_t o, uint32_t kb, uint64_t dv, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, t;\n\t.reg .b32 h<4>, l<4>;\n\t.reg .b64 vh<4>, vl<4>;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 t, %4, %4;\n\t"
      "add.u32 h0, %1, 0;\n\t add.u32 h1, %1, 8;\n\t add.u32 h2, %1, 32;\n\t add.u32 h3, %1, 40;\n\t"
      "add.u32 l0, %1, 16;\n\t add.u32 l1, %1, 24;\n\t add.u32 l2, %1, 48;\n\t add.u32 l3, %1, 56;\n\t"
      "add.s64 vh0, %2, 0;\n\t add.s64 vh1, %2, %5;\n\t add.s64 vh2, %2, %6;\n\t add.s64 vh3, %2, %7;\n\t"
      "add.s64 vl0, %2, %8;\n\t add.s64 vl1, %2, %9;\n\t add.s64 vl2, %2, %10;\n\t add.s64 vl3, %2, %11;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [h0], vh0, %3, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [h0], vl0, %3, t;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [l0], vh0, %3, t;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [h1], vh1, %3, t;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [h1], vl1, %3, t;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [l1], vh1, %3, t;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [h2], vh2, %3, t;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [h2], vl2, %3, t;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [l2], vh2, %3, t;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [h3], vh3, %3, t;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [h3], vl3, %3, t;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [l3], vh3, %3, t;\n\t}" ::"r"(o),
      "r"(kb), "l"(dv), "r"(idesc), "r"(acc), "n"(2 * TH), "n"(4 * TH), "n"(6 * TH), "n"(8 * TH),
      "n"(10 * TH), "n"(12 * TH), "n"(14 * TH)
      : "memory");
}

template <int KIND, int TN, int KF>
__global__ void __launch_bounds__(NT3, 1) mvm_tc3_kernel(TcArgs args) {
  using C = Cfg3<TN, KF>;
  constexpr int TH = C::TH;
  if (args.done != nullptr && args.done->done) return;   // same flag in both CTAs of the pair
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* abuf = smem;                                  // [2][A_BYTES]
  uint8_t* pro = smem + 2 * C::A_BYTES;                  // [NB3][F_BYTES]
  uint8_t* ring = smem + C::RING_OFF;
  Bars3* bars = reinterpret_cast<Bars3*>(ring + C::STAGES * C::STAGE);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int64_t n = args.n;
  const int ntiles = (int)((n + BN3 - 1) / BN3);

  if (threadIdx.x == 0) {
    const uint32_t nl = leader ? 2 : 1;   // leader: own bulk copies + the peer relay's arrival
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&bars->full[s], nl); mbar_init(&bars->empty[s], 1); }
    for (int b = 0; b < NB3; ++b) { mbar_init(&bars->s_full[b], 1); mbar_init(&bars->k_full[b], KARR); }
    for (int b = 0; b < 2; ++b) { mbar_init(&bars->a_full[b], nl); mbar_init(&bars->a_empty[b], 1); }
    mbar_init(&bars->pro_full, nl);
    for (int o = 0; o < 2; ++o) { mbar_init(&bars->o_full[o], 1); mbar_init(&bars->o_empty[o], OARR); }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&bars->tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  fence_before_sync();
  cluster_sync();   // barriers of both CTAs initialised, TMEM allocated in both
  fence_after_sync();
  const uint32_t tbase = bars->tmem_base;
  const size_t plane = (size_t)args.vrows * TH;   // one plane of one TH-wide layout chunk

  // tiles of this pair
  int ntot = 0, nunit = 0;
  for (int u = blockIdx.x / 2; u < args.nunits; u += gridDim.x / 2) {
    const int split = (u / args.chunks) % args.nsplit;
    ntot += ntiles * (split + 1) / args.nsplit - ntiles * split / args.nsplit;
    ++nunit;
  }

  if (warp == 0) {
    // ---------------- producer (one thread per CTA): this CTA's halves of every operand ----------------
    if (lane == 0) {
      Cur3 c, f;
      c.start(args, ntiles);
      if (c.valid(args)) {
        const int64_t i0 = args.row0 + (int64_t)c.rt * (2 * BM3) + BM3 * rank;
        mbar_arrive_expect_tx(&bars->a_full[0], C::A_BYTES);
        bulk_g2s(abuf, args.feat_a + (size_t)i0 * KF, C::A_BYTES, &bars->a_full[0]);
        mbar_arrive_expect_tx(&bars->pro_full, SK * C::F_BYTES);
        for (int i = 0; i < SK; ++i)
          bulk_g2s(pro + i * C::F_BYTES, args.feat_b + ((size_t)(c.jt0 + i) * BN3 + 32 * rank) * KF, C::F_BYTES,
                   &bars->pro_full);
        f = c;
        for (int i = 0; i < SK; ++i) f.advance(args, ntiles);
      }
      for (int g = 0; c.valid(args); ++g) {
        const bool fv = f.valid(args);
        if (fv && f.jj == 0 && f.k > 0) {   // S of unit f.k starts with tile g + SK: its A rows
          const int kb = f.k & 1;
          mbar_wait_backoff(&bars->a_empty[kb], ((f.k >> 1) & 1) ^ 1);
          const int64_t i0 = args.row0 + (int64_t)f.rt * (2 * BM3) + BM3 * rank;
          mbar_arrive_expect_tx(&bars->a_full[kb], C::A_BYTES);
          bulk_g2s(abuf + kb * C::A_BYTES, args.feat_a + (size_t)i0 * KF, C::A_BYTES, &bars->a_full[kb]);
        }
        const int st = g % C::STAGES;
        mbar_wait_backoff(&bars->empty[st], ((g / C::STAGES) & 1) ^ 1);
        if (leader) T3_STAMP(0, g);
        {
          uint32_t fl = 0;
          if (c.jj > 0) fl |= F_ACC;
          if (c.jj == c.njt - 1) fl |= F_OLAST;
          if (c.k & 1) fl |= F_OB;
          if (c.jj == 0 && c.k >= 2) fl |= F_OWAIT | ((((c.k >> 1) - 1) & 1) ? F_OPH : 0u);
          if (fv) {
            fl |= F_SVALID | ((f.k & 1) ? F_KB : 0u);
            if (f.jj == 0) fl |= F_SFIRST | (((f.k >> 1) & 1) ? F_APH : 0u);
            if (f.jj == f.njt - 1) fl |= F_SLAST;
          }
          bars->flags[st] = fl;   // published to the issuer by the full[st] arrive below
        }
        uint8_t* sb = ring + st * C::STAGE;
        mbar_arrive_expect_tx(&bars->full[st], 2 * C::V_BYTES + (fv ? C::F_BYTES : 0));
        const __half* vh = args.vplanes + (size_t)(c.chunk * 2 + rank) * 2 * plane + (size_t)c.J() * BN3 * TH;
        bulk_g2s(sb, vh, C::V_BYTES, &bars->full[st]);
        bulk_g2s(sb + C::V_BYTES, vh + plane, C::V_BYTES, &bars->full[st]);
        if (fv)
          bulk_g2s(sb + 2 * C::V_BYTES, args.feat_b + ((size_t)f.J() * BN3 + 32 * rank) * KF, C::F_BYTES,
                   &bars->full[st]);
        c.advance(args, ntiles);
        if (fv) f.advance(args, ntiles);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the leader's warp 1 issues for the pair ----------------
    if (leader && ntot > 0) {
      constexpr uint32_t idesc_s = idesc_f16(256, BN3, 0, 0);   // A, B K-major, M = 256, N = 64
      constexpr uint32_t idesc_o = idesc_f16(256, TN, 0, 1);    // A (TMEM) K-major, B MN-major
      // K-major features: LBO = 128 B, SBO = KF/8 * 128 B; V halves MN-major: LBO = TH/8 * 128 B, SBO = 128 B
      const uint64_t da0 = smem_desc(smem_u32(abuf), 128, (KF / 8) * 128);
      const uint64_t dpro = smem_desc(smem_u32(pro), 128, (KF / 8) * 128);
      const uint64_t dring_f = smem_desc(smem_u32(ring) + 2 * C::V_BYTES, 128, (KF / 8) * 128);
      const uint64_t dring_v = smem_desc(smem_u32(ring), (TH / 8) * 128, 128);
      Cur3 s;
      s.start(args, ntiles);
      mbar_wait_cl(&bars->a_full[0], 0);
      mbar_wait_cl(&bars->pro_full, 0);
      fence_after_sync();
      for (int i = 0; i < SK && s.valid(args) && s.k == 0; ++i) {
        const uint32_t d = __shfl_sync(0xffffffffu, tbase + i * BN3, 0);
        const uint64_t db = shfl64_3(dpro + (uint64_t)((i * C::F_BYTES) >> 4));
        const bool last = s.jj == s.njt - 1;
        if (elect_one3()) {
          mma_s3<KF>(d, da0, db, idesc_s);
          commit_pair(&bars->s_full[i]);
          if (last) commit_pair(&bars->a_empty[0]);
        }
        __syncwarp();
        s.advance(args, ntiles);
      }
      int st = 0, b = 0;
      uint32_t ph_st = 0, ph_b = 0;
      for (int g = 0; g < ntot; ++g) {
        mbar_wait(&bars->full[st], ph_st);
        if (lane == 0) T3_STAMP(1, g);
        const uint32_t fl = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile uint32_t*>(&bars->flags[st]), 0);
        const uint32_t soff16 = (uint32_t)((st * C::STAGE) >> 4);
        if (fl & F_SVALID) {   // S(g + SK) into the buffer of tile g - 1 (its KV was issued at step g - 1)
          const int bs = b == 0 ? NB3 - 1 : b - 1;
          const int kb = (fl & F_KB) ? 1 : 0;
          if (fl & F_SFIRST) mbar_wait(&bars->a_full[kb], (fl & F_APH) ? 1u : 0u);
          fence_after_sync();
          const uint32_t sbu = __shfl_sync(0xffffffffu, tbase + bs * BN3, 0);
          const uint64_t dau = shfl64_3(da0 + (uint64_t)(kb * (C::A_BYTES >> 4)));
          const uint64_t dfu = shfl64_3(dring_f + soff16);
          if (elect_one3()) {
            mma_s3<KF>(sbu, dau, dfu, idesc_s);
            commit_pair(&bars->s_full[bs]);
            if (fl & F_SLAST) commit_pair(&bars->a_empty[kb]);
          }
          __syncwarp();
        }
        if (lane == 0) T3_STAMP(4, g);
        mbar_wait(&bars->k_full[b], ph_b);
        if (lane == 0) T3_STAMP(2, g);
        const uint32_t ob = (fl & F_OB) ? 1u : 0u;
        if (fl & F_OWAIT) mbar_wait(&bars->o_empty[ob], (fl & F_OPH) ? 1u : 0u);
        fence_after_sync();
        const uint32_t kbu = __shfl_sync(0xffffffffu, tbase + b * BN3, 0);
        const uint32_t tou = __shfl_sync(0xffffffffu, tbase + TMO3 + TN * ob, 0);
        const uint64_t dvu = shfl64_3(dring_v + soff16);
        if (elect_one3()) {
          mma_kv3<TH>(tou, kbu, dvu, idesc_o, fl & F_ACC);
          if (fl & F_OLAST) commit_pair(&bars->o_full[ob]);
        }
        __syncwarp();
        if (lane == 0) T3_STAMP(3, g);
        if (elect_one3()) commit_pair(&bars->empty[st]);
        __syncwarp();
        if (++st == C::STAGES) { st = 0; ph_st ^= 1; }
        if (++b == NB3) { b = 0; ph_b ^= 1; }
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ---------------- relays (peer CTA only): forward completed phases of the peer's own bulk
    // copies to the leader's barriers (warp 2: ring stages; warp 3: prologue + A rows).  The arrive
    // is relaxed: the bytes are already in the peer's shared memory when its barrier phase
    // completes, and a release at cluster scope (MEMBAR.ALL.GPU, ~0.6 us) serialised one stage per
    // membar -- measured as the pair kernel's limit (1.31 ms per C3 MVM). ----------------
    if (!leader && lane == 0 && ntot > 0) {
      if (warp == 2) {
        const uint32_t rfull = mapa_u32(smem_u32(&bars->full[0]), 0);
        for (int g = 0; g < ntot; ++g) {
          const int st = g % C::STAGES;
          mbar_wait_backoff(&bars->full[st], (g / C::STAGES) & 1);
          mbar_arrive_cluster_relaxed(rfull + st * 8);
          T3_STAMP(9, g);
        }
      } else {
        mbar_wait_backoff(&bars->pro_full, 0);
        mbar_arrive_cluster_relaxed(mapa_u32(smem_u32(&bars->pro_full), 0));
        const uint32_t rafull = mapa_u32(smem_u32(&bars->a_full[0]), 0);
        for (int k = 0; k < nunit; ++k) {
          mbar_wait_backoff(&bars->a_full[k & 1], (k >> 1) & 1);
          mbar_arrive_cluster_relaxed(rafull + (k & 1) * 8);
        }
      }
    }
  } else {
    // ---------------- epilogue: 16 warps per CTA in NGRP groups (tile g -> group g % NGRP); warp w
    // works on TMEM lane quarter q = w % 4 and NCH 32-column chunks of the tile starting at cc0;
    // it reads out O columns [slice * TN/4, +TN/4) ----------------
    const int q = warp % 4;
    const int grp = (warp - EPI0) / WPG;
    const int cc0 = NCH == 2 ? 0 : ((warp - EPI0) >> 2) & 1;
    const int slice = (warp - EPI0) >> 2;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t rk_full = mapa_u32(smem_u32(&bars->k_full[0]), 0);
    const uint32_t ro_empty = mapa_u32(smem_u32(&bars->o_empty[0]), 0);
    Cur3 c, prev;
    c.start(args, ntiles);
    prev = c;
    auto readout = [&](const Cur3& u) {
      // O columns [slice * CPW, +CPW) of rows 32 q + lane of this CTA
      constexpr int CPW = TN / 4;
      const int ob = u.k & 1;
      uint32_t o[CPW];
      mbar_wait(&bars->o_full[ob], (u.k >> 1) & 1);
      fence_after_sync();
      const uint32_t ta = tbase + TMO3 + TN * ob + slice * CPW + lane_base;
#pragma unroll
      for (int m = 0; m < CPW; m += 8) tmem_ld8(ta + m, &o[m]);
      tmem_ld_wait();
      fence_before_sync();
      __syncwarp();
      if (lane == 0) {   // O drained into registers (wait::ld + fence above)
        if (leader) mbar_arrive(&bars->o_empty[ob]);
        else mbar_arrive_cluster_relaxed(ro_empty + ob * 8);
      }
      const int64_t i = args.row0 + (int64_t)u.rt * (2 * BM3) + BM3 * rank + 32 * q + lane;
      const bool row_ok = i < args.row1;
      const int col0 = u.chunk * TN + slice * CPW;
      float* pout = args.p + (size_t)u.split * args.p_split_stride + (size_t)(i - args.row0) * args.tp + col0;
      const float* vrow = args.v + (size_t)i * args.tp + col0;
      double* ap = args.apart
                       ? args.apart + ((size_t)(u.rt * args.nsplit + u.split) * 8 + q * 2 + rank) * args.tp + col0
                       : nullptr;
#pragma unroll
      for (int m = 0; m < CPW; m += 4) {
        float4 v4 = make_float4(0.f, 0.f, 0.f, 0.f), r4 = v4;
        if (row_ok) {
          v4 = *reinterpret_cast<const float4*>(vrow + m);
          r4.x = args.o2 * __uint_as_float(o[m + 0]) * args.inv_scale[col0 + m + 0];
          r4.y = args.o2 * __uint_as_float(o[m + 1]) * args.inv_scale[col0 + m + 1];
          r4.z = args.o2 * __uint_as_float(o[m + 2]) * args.inv_scale[col0 + m + 2];
          r4.w = args.o2 * __uint_as_float(o[m + 3]) * args.inv_scale[col0 + m + 3];
          if (u.split == 0) {
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
    };
    int b = 0;
    uint32_t ph_b = 0;
    for (int g = 0; c.valid(args); ++g) {
      if (lane == 0 && warp == EPI0 && leader) T3_STAMP(12, g);
      if ((g & (NGRP - 1)) == grp) {
        const bool stamp = lane == 0 && (warp - EPI0) % WPG == 0;
        if (stamp) T3_STAMP(leader ? 10 : 13, g);
        mbar_wait(&bars->s_full[b], ph_b);
        if (stamp) T3_STAMP(leader ? 5 : 7, g);
        fence_after_sync();
#pragma unroll 1
        for (int ch = cc0; ch < cc0 + NCH; ++ch) {
          const uint32_t tb = tbase + b * BN3 + 32 * ch + lane_base;
          const int64_t jcol0 = (int64_t)c.J() * BN3 + 32 * ch;
          uint32_t sv[32];
          tmem_ld32(tb, sv);
          tmem_ld_wait();
          uint32_t hi[16], lo[16];
          if (jcol0 + 32 > n) exp_split3<KIND, true>(sv, hi, lo, (int)(n - jcol0));
          else exp_split3<KIND, false>(sv, hi, lo, 32);
          tmem_st16(tb, hi);
          tmem_st16(tb + 16, lo);
        }
        tmem_st_wait();
        fence_before_sync();
        __syncwarp();
        if (stamp) T3_STAMP(leader ? 6 : 8, g);
        if (lane == 0) {   // K(g) in this CTA's TMEM is complete (wait::st + fence above)
          if (leader) mbar_arrive(&bars->k_full[b]);
          else mbar_arrive_cluster_relaxed(rk_full + b * 8);
        }
        if (stamp) T3_STAMP(leader ? 11 : 13, g);
        // first tile this warp takes in unit k: unit k-1's last KV is issued
        if (c.k > 0 && c.k != prev.k) readout(prev);
        prev = c;
      }
      c.advance(args, ntiles);
      if (++b == NB3) { b = 0; ph_b ^= 1; }
    }
    if (prev.valid(args)) readout(prev);
  }
  fence_before_sync();
  __syncthreads();
  cluster_sync();   // no CTA leaves while its peer may still signal its barriers or read its TMEM / smem
  if (warp == 1) {
    fence_after_sync();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  }
}

template <int KIND, int TN, int KF>
cudaError_t launch3(const TcArgs& a, int pairs, cudaStream_t s) {
  auto k = mvm_tc3_kernel<KIND, TN, KF>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg3<TN, KF>::SMEM);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(NT3);
  cfg.dynamicSmemBytes = Cfg3<TN, KF>::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, a);
}

template <int KIND, int KF>
cudaError_t launch3_tn(const TcArgs& a, int tn, int pairs, cudaStream_t s) {
  switch (tn) {
    case 32: return launch3<KIND, 32, KF>(a, pairs, s);
    case 64: return launch3<KIND, 64, KF>(a, pairs, s);
  }
  return cudaErrorInvalidValue;
}

template <int KIND>
cudaError_t launch3_kf(const TcArgs& a, int tn, int pairs, cudaStream_t s) {
  return a.kf == 64 ? launch3_tn<KIND, 64>(a, tn, pairs, s) : launch3_tn<KIND, 32>(a, tn, pairs, s);
}

}  // namespace

// The pair kernel needs an RHS chunk of >= 32 columns (each CTA holds TN/2 >= 16 of the MMA's N,
// and a TS MMA on a pair needs N % 32 == 0) and >= NB3 + 2 column tiles per unit (prologue of
// SK S tiles inside the first unit).
bool tc3_supported(int tn, int64_t n, int nsplit) {
  const int64_t ntiles = (n + BN3 - 1) / BN3;
  return (tn == 32 || tn == 64) && ntiles / nsplit >= NB3 + 2;
}

int tc3_min_tiles() { return NB3 + 2; }

int tc3_units(int64_t rows, int nsplit, int chunks) { return (int)((rows + 2 * BM3 - 1) / (2 * BM3)) * nsplit * chunks; }

cudaError_t launch_mvm_tc3(const TcArgs& a, int nsm, cudaStream_t s) {
  const int tn = tc_chunk_cols(a.tp);
  const int pairs = a.nunits < nsm / 2 ? a.nunits : nsm / 2;
  switch (a.kind) {
    case 1: return launch3_kf<1>(a, tn, pairs, s);
    case 2: return launch3_kf<2>(a, tn, pairs, s);
    case 3: return launch3_kf<3>(a, tn, pairs, s);
    case 11: return launch3_kf<4>(a, tn, pairs, s);
    case 12: return launch3_kf<5>(a, tn, pairs, s);
    case 13: return launch3_kf<6>(a, tn, pairs, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ciq
