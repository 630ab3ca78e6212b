// mvm_tc2.cu -- the fused matrix-free kernel MVM, persistent 256-row version (SURVEY K1, §8(a)
// row a4):  P = K(X, X) V + sigma^2 V with K never materialised in HBM.
//
// Why a second design (measured on B200, profiles/ncu_k1_r01b.txt and DESIGN.md §8): the 128-row
// kernel in mvm_tc.cu streams 40 KB of V planes + column features from L2 per 128x128 tile of
// kernel evaluations, i.e. 6.3 GB per C3 MVM; with the B200 L2 -> SM limit (~6.3 KB/clk chip-wide)
// that alone costs ~0.5 ms, as much as the SFU (ex2) floor, and its skeleton without any exp /
// KV work already took 0.57 ms.  Here:
//   * a CTA unit is 256 rows (two 128-lane halves) x a column range, streamed in 64-column tiles:
//     per 16384 kernel evaluations the CTA loads 16 KB of V planes + 4 KB of features (half);
//   * the grid is persistent (one CTA per SM, units round-robin), so the per-CTA ramp (TMEM
//     alloc, barrier init, first loads) and the output read-out are paid once per SM, and the
//     stream of tiles continues across unit boundaries (the smem ring, the S look-ahead and the
//     TMEM buffers all run over the flattened tile sequence of the CTA).
//
// Per tile J of a unit (rows I = 256, columns J = 64):
//   (1) S_h = A_{I,h} . B_J^T, h = 0, 1  (tcgen05 kind::f16 SS, M=128 N=64 K=32: augmented split-fp16
//       features, S_ij = -(log2 e / 2) ||x_i - x_j||^2 / l^2 exactly as in mvm_tc.cu);
//   (2) 16 epilogue warps: tcgen05.ld S -> k = kernel(S) (ex2 on the SFU), masked past N ->
//       split k = k_hi + k_lo (fp16) -> tcgen05.st in place (chunk c -> hi at [32c, 32c+16),
//       lo at [32c+16, 32c+32));
//   (3) O_h += K_h . V_J (TS: A from TMEM, B = V_J MN-major): k_hi.v_hi + k_hi.v_lo + k_lo.v_hi.
// TMEM (512 columns): NB2 S/K buffers b at [128 b, 128 b + 128) (half h at +64 h), then NO2 O
// slots (slot s, half h at 128 NB2 + 2 TN s + TN h; units alternate slots).  S runs NB2 tiles ahead
// of KV.  Default NB2 = NO2 = 2 (see CIQ_TC2_NB below).
// Smem: A features of the unit (256 rows, double-buffered across units), features of the first
// NB2 tiles, and a ring whose stage g holds V(g) and the column features of tile g+NB2 (skewed:
// one stage wait / release per tile on the MMA warp), and per reading warp a 2 KB transpose buffer.
// The output read-out of unit k is done by the epilogue group that takes the first tile of unit
// k+1, right after that tile (O is drained to registers through the smem transpose, released,
// then written with coalesced stores; the alpha partials by lane-group shuffles); the CTA's alpha
// partials are reduced in the kernel tail when the recurrence asks for it (TcArgs::alpha_out).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "tc_util.cuh"

#include "kern_epi.cuh"

namespace ciq {
namespace {

using namespace tc;

constexpr int BM2 = 256;            // rows per unit (two 128-lane halves)
constexpr int BN2 = 64;             // columns per tile
constexpr int KF2 = 32;             // feature contraction
constexpr int NT2 = 640;            // 4 role warps + 16 epilogue warps
constexpr int EPI0 = 4;
// TMEM: S/K buffers x 128 columns + O slots x 2 TN.  Round 2, with the 66-tile accumulation chains
// (16 units per CTA at C3): 2 S/K buffers + 2 O slots beat 3 + 1 (MVM 0.99-1.00 vs 1.01-1.02 ms,
// profiles/ab_k1_oslots_r02.txt) -- the unit read-out no longer stalls the next unit's first KV,
// which outweighs the shallower S look-ahead.
#ifndef CIQ_TC2_NB
#define CIQ_TC2_NB 2
#endif
#ifndef CIQ_TC2_OSLOTS
#define CIQ_TC2_OSLOTS 2
#endif
constexpr int NB2 = CIQ_TC2_NB;     // S/K TMEM buffers
constexpr int NO2 = CIQ_TC2_OSLOTS; // O accumulator slots (2: the next unit's KV never waits for a read-out)
constexpr int TMO = NB2 * 128;      // O slot s, half h at TMO + s 2 TN + h TN
static_assert(NB2 * 128 + NO2 * 128 <= 512 && NO2 >= 1 && NO2 <= 2, "TMEM budget (TN <= 64)");
// Ping-pong epilogue (measured: 0.937 vs 1.088 ms per C3 MVM for all 16 warps on every tile,
// profiles/): two groups of 8 warps take alternate tiles.
constexpr int EPI_ARRIVALS = 4;    // epilogue warps per tile and half
constexpr int RO_ARRIVALS = 4;     // warps reading out O_h of a unit, per half (one group)
constexpr int RO_BYTES = 32 * 16 * 4;   // read-out transpose scratch per warp: 32 rows x 16 fp32

template <int TN>
struct Cfg2 {
  static constexpr int A_BYTES = BM2 * KF2 * 2;      // 16 KB
  static constexpr int F_BYTES = BN2 * KF2 * 2;      // 4 KB
  static constexpr int V_BYTES = BN2 * TN * 2;       // one plane of one tile
  static constexpr int STAGE = 2 * V_BYTES + F_BYTES;
  static constexpr int STAGES = 8;
  static constexpr int RING_OFF = 2 * A_BYTES + NB2 * F_BYTES;
  static constexpr int RO_OFF = RING_OFF + STAGES * STAGE + 1024;   // after the barriers
  static constexpr int SMEM = 1024 + RO_OFF + 8 * RO_BYTES;
};
static_assert(Cfg2<64>::SMEM <= 227 * 1024, "shared memory budget");

struct Bars2 {
  uint64_t full[8], empty[8];              // smem ring (empty: one commit per MMA warp)
  uint64_t s_full[NB2][2], k_full[NB2][2];   // per TMEM buffer and 128-row half
  uint64_t a_full[2], a_empty[2];
  uint64_t pro_full, o_full[NO2][2], o_empty[NO2][2];
  uint32_t tmem_base;
  int eff_nsplit, eff_nunits;   // this launch's unit grid (Sched)
  int lowp;                     // second relaxation level: k_hi only (exp_hi, mma_kv8)
  uint32_t flags[8];   // per ring stage: the MMA issuers' schedule for that tile (written by the producer)
};

// Schedule of tile g (KV) and tile g+3 (S), computed by the producer (which has slack) so the MMA
// issuers -- whose every instruction costs epilogue issue slots -- only test bits.
enum : uint32_t {
  F_ACC = 1u << 0,      // KV accumulates into O (not the first tile of its unit)
  F_OLAST = 1u << 1,    // last tile of its unit: commit o_full after KV
  F_OWAIT = 1u << 2,    // first tile of a unit after the first: wait o_empty (phase F_OPH)
  F_OPH = 1u << 3,
  F_SVALID = 1u << 4,   // S(g+3) exists
  F_SFIRST = 1u << 5,   // S(g+3) is the first tile of its unit: wait a_full[F_KB] (phase F_APH)
  F_APH = 1u << 6,
  F_SLAST = 1u << 7,    // S(g+3) is the last tile of its unit: commit a_empty[F_KB]
  F_KB = 1u << 8,       // A-rows buffer of S(g+3)'s unit
  F_OSLOT = 1u << 9,    // O slot of tile g's unit (NO2 = 2)
};

// 64-column tile of K of the launch's t-th tile (its column window, TcArgs::win_* / skip_*)
CIQ_DEVICE int window_tile(const TcArgs& a, int t) {
  int j = (a.win_hi > 0 ? a.win_lo : 0) + t;
  if (a.skip_hi > a.skip_lo && j >= a.skip_lo) j += a.skip_hi - a.skip_lo;
  return j;
}

// Position in the flattened tile sequence of one CTA: unit u (local index k), tile jj of njt.
// The launch's unit grid: column splits x units (TcArgs::nsplit / nunits, or the relaxed
// schedule's nsplit_alt / nunits_alt when *gate != 0 -- chosen once per launch, kept in smem).
struct Sched {
  const volatile int* g;   // -> Bars2::eff_nsplit, eff_nunits (read at each use: no pinned registers)
  int chunks;
  CIQ_DEVICE int nsplit() const { return g[0]; }
  CIQ_DEVICE int nunits() const { return g[1]; }
};

struct Cur {
  int k, u, jj, njt, jt0, split, chunk, rt;
  CIQ_DEVICE void decode(const Sched& a, int ntiles) {
    chunk = u % a.chunks;
    const int t = u / a.chunks;
    split = t % a.nsplit();
    rt = t / a.nsplit();
    jt0 = ntiles * split / a.nsplit();          // ntiles * nsplit < 2^31 (checked on the host)
    njt = ntiles * (split + 1) / a.nsplit() - jt0;
  }
  CIQ_DEVICE void start(const Sched& a, int ntiles) {
    k = 0;
    u = blockIdx.x;
    jj = 0;
    if (u < a.nunits()) decode(a, ntiles);
  }
  CIQ_DEVICE bool valid(const Sched& a) const { return u < a.nunits(); }
  CIQ_DEVICE void advance(const Sched& a, int ntiles) {
    if (++jj == njt) {
      jj = 0;
      ++k;
      u += gridDim.x;
      if (u < a.nunits()) decode(a, ntiles);
    }
  }
  CIQ_DEVICE int J(const TcArgs& a) const { return window_tile(a, jt0 + jj); }
};

// KV(J) of one half: O_h (+)= K_h . V_J, 4 K-steps x (k_hi.v_hi, k_hi.v_lo, k_lo.v_hi) = 12 TS MMAs,
// issued by one elected thread; all operands are immediates off three uniform bases, so the
// compiler emits ~2 uniform-datapath instructions per MMA.  o: TMEM O of the half; kb: TMEM K
// buffer of the half (K-step s -> k_hi at 32 (s/2) + 8 (s%2), k_lo at +16); dv: V_hi descriptor of
// the stage (V_lo at +8 TN, K-step s at +2 TN s in descriptor units); acc: accumulate into O.
template <int TN>
CIQ_DEVICE void mma_kv12(uint32_t o, uint32_t kb, uint64_t dv, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, t;\n\t.reg .b32 h<4>, l<4>;\n\t.reg .b64 vh<4>, vl<4>;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 t, %4, %4;\n\t"
      "add.u32 h0, %1, 0;\n\t add.u32 h1, %1, 8;\n\t add.u32 h2, %1, 32;\n\t add.u32 h3, %1, 40;\n\t"
      "add.u32 l0, %1, 16;\n\t add.u32 l1, %1, 24;\n\t add.u32 l2, %1, 48;\n\t add.u32 l3, %1, 56;\n\t"
      "add.s64 vh0, %2, 0;\n\t add.s64 vh1, %2, %5;\n\t add.s64 vh2, %2, %6;\n\t add.s64 vh3, %2, %7;\n\t"
      "add.s64 vl0, %2, %8;\n\t add.s64 vl1, %2, %9;\n\t add.s64 vl2, %2, %10;\n\t add.s64 vl3, %2, %11;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h0], vh0, %3, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h0], vl0, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [l0], vh0, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h1], vh1, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h1], vl1, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [l1], vh1, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h2], vh2, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h2], vl2, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [l2], vh2, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h3], vh3, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h3], vl3, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [l3], vh3, %3, t;\n\t}" ::"r"(o),
      "r"(kb), "l"(dv), "r"(idesc), "r"(acc), "n"(2 * TN), "n"(4 * TN), "n"(6 * TN), "n"(8 * TN),
      "n"(10 * TN), "n"(12 * TN), "n"(14 * TN)
      : "memory");
}

// KV(J) of one half with k_hi only (second relaxation level): k_hi.v_hi + k_hi.v_lo, 8 TS MMAs
template <int TN>
CIQ_DEVICE void mma_kv8(uint32_t o, uint32_t kb, uint64_t dv, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, t;\n\t.reg .b32 h<4>;\n\t.reg .b64 vh<4>, vl<4>;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 t, %4, %4;\n\t"
      "add.u32 h0, %1, 0;\n\t add.u32 h1, %1, 8;\n\t add.u32 h2, %1, 32;\n\t add.u32 h3, %1, 40;\n\t"
      "add.s64 vh0, %2, 0;\n\t add.s64 vh1, %2, %5;\n\t add.s64 vh2, %2, %6;\n\t add.s64 vh3, %2, %7;\n\t"
      "add.s64 vl0, %2, %8;\n\t add.s64 vl1, %2, %9;\n\t add.s64 vl2, %2, %10;\n\t add.s64 vl3, %2, %11;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h0], vh0, %3, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h0], vl0, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h1], vh1, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h1], vl1, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h2], vh2, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h2], vl2, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h3], vh3, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [h3], vl3, %3, t;\n\t}" ::"r"(o),
      "r"(kb), "l"(dv), "r"(idesc), "r"(acc), "n"(2 * TN), "n"(4 * TN), "n"(6 * TN), "n"(8 * TN),
      "n"(10 * TN), "n"(12 * TN), "n"(14 * TN)
      : "memory");
}

// experiments only: per-tile clock64 stamps of CTA 0 (build with CIQ_TC_TRACE, run with
// CIQ_TC_DEBUG=128; same slots as mvm_tc.cu)
#ifdef CIQ_TC_TRACE
#define T2_STAMP(slot, idx)                                                                  \
  do {                                                                                       \
    if (args.dbg_clk != nullptr && blockIdx.x == 0 && lane == 0 && (idx) < 256)              \
      args.dbg_clk[(slot) * 256 + (idx)] = clock64();                                        \
  } while (0)
#else
#define T2_STAMP(slot, idx) \
  do {                      \
  } while (0)
#endif

template <int KIND, int TN>
__global__ void __launch_bounds__(NT2, 1) mvm_tc2_kernel(TcArgs args) {
  using C = Cfg2<TN>;
  if (args.done != nullptr && args.done->done) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* abuf = smem;                                  // [2][A_BYTES]
  uint8_t* pro = smem + 2 * C::A_BYTES;                  // [3][F_BYTES]
  uint8_t* ring = smem + C::RING_OFF;
  Bars2* bars = reinterpret_cast<Bars2*>(ring + C::STAGES * C::STAGE);
  static_assert(sizeof(Bars2) <= 1024, "barrier block");

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t n = args.n;
  const int ntiles = tc2_window_tiles(args);   // this launch's column tiles

  if (threadIdx.x == 0) {
    const bool alt = args.gate != nullptr && *args.gate != 0;   // relaxed schedule (params.mvm_relax)
    bars->eff_nsplit = alt ? args.nsplit_alt : args.nsplit;
    bars->eff_nunits = alt ? args.nunits_alt : args.nunits;
    bars->lowp = (args.gate != nullptr && *args.gate >= 2) ? 1 : 0;
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&bars->full[s], 1); mbar_init(&bars->empty[s], 2); }
    for (int b = 0; b < NB2; ++b)
      for (int h = 0; h < 2; ++h) { mbar_init(&bars->s_full[b][h], 1); mbar_init(&bars->k_full[b][h], EPI_ARRIVALS); }
    for (int b = 0; b < 2; ++b) { mbar_init(&bars->a_full[b], 1); mbar_init(&bars->a_empty[b], 2); }
    mbar_init(&bars->pro_full, 1);
    for (int o = 0; o < NO2; ++o)
      for (int h = 0; h < 2; ++h) { mbar_init(&bars->o_full[o][h], 1); mbar_init(&bars->o_empty[o][h], RO_ARRIVALS); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = bars->tmem_base;
  const Sched sch{&bars->eff_nsplit, args.chunks};
  const bool lowp = bars->lowp != 0;
  const size_t plane = (size_t)args.vrows * TN;   // one plane of one chunk

  if (warp == 0) {
    // ---------------- producer (one thread) ----------------
    if (lane == 0) {
      Cur c, f;
      c.start(sch, ntiles);
      if (c.valid(sch)) {
        // prologue: A rows of unit 0 and the column features of its first three tiles (njt >= 4)
        const int64_t i0 = args.row0 + (int64_t)c.rt * BM2;
        mbar_arrive_expect_tx(&bars->a_full[0], C::A_BYTES);
        bulk_g2s(abuf, args.feat_a + (size_t)i0 * KF2, C::A_BYTES, &bars->a_full[0]);
        const int npro = c.njt < NB2 ? c.njt : NB2;
        mbar_arrive_expect_tx(&bars->pro_full, npro * C::F_BYTES);
        for (int i = 0; i < npro; ++i)
          bulk_g2s(pro + i * C::F_BYTES, args.feat_b + (size_t)window_tile(args, c.jt0 + i) * BN2 * KF2, C::F_BYTES, &bars->pro_full);
        f = c;
        for (int i = 0; i < NB2; ++i) f.advance(sch, ntiles);
      }
      for (int g = 0; c.valid(sch); ++g) {
        const bool fv = f.valid(sch);
        if (fv && f.jj == 0 && f.k > 0) {   // S of unit f.k starts with tile g+3: its A rows
          const int kb = f.k & 1;
          mbar_wait_backoff(&bars->a_empty[kb], ((f.k >> 1) & 1) ^ 1);
          const int64_t i0 = args.row0 + (int64_t)f.rt * BM2;
          mbar_arrive_expect_tx(&bars->a_full[kb], C::A_BYTES);
          bulk_g2s(abuf + kb * C::A_BYTES, args.feat_a + (size_t)i0 * KF2, C::A_BYTES, &bars->a_full[kb]);
        }
        const int st = g % C::STAGES;
        mbar_wait_backoff(&bars->empty[st], ((g / C::STAGES) & 1) ^ 1);
        T2_STAMP(0, g);
        {
          uint32_t fl = 0;
          if (c.jj > 0) fl |= F_ACC;
          if (c.jj == c.njt - 1) fl |= F_OLAST;
          // the first KV of unit k overwrites O slot k % NO2: unit k - NO2 must be read out
          if (c.jj == 0 && c.k >= NO2) fl |= F_OWAIT | ((((c.k - NO2) / NO2) & 1) ? F_OPH : 0u);
          if (NO2 > 1 && (c.k & 1)) fl |= F_OSLOT;
          if (fv) {
            fl |= F_SVALID | ((f.k & 1) ? F_KB : 0u);
            if (f.jj == 0) fl |= F_SFIRST | (((f.k >> 1) & 1) ? F_APH : 0u);
            if (f.jj == f.njt - 1) fl |= F_SLAST;
          }
          bars->flags[st] = fl;   // published to the MMA issuers by the full[st] arrive below
        }
        uint8_t* sb = ring + st * C::STAGE;
        mbar_arrive_expect_tx(&bars->full[st], 2 * C::V_BYTES + (fv ? C::F_BYTES : 0));
        const __half* vh = args.vplanes + (size_t)c.chunk * 2 * plane + (size_t)c.J(args) * BN2 * TN;
        bulk_g2s(sb, vh, C::V_BYTES, &bars->full[st]);
        bulk_g2s(sb + C::V_BYTES, vh + plane, C::V_BYTES, &bars->full[st]);
        if (fv) bulk_g2s(sb + 2 * C::V_BYTES, args.feat_b + (size_t)f.J(args) * BN2 * KF2, C::F_BYTES, &bars->full[st]);
        c.advance(sch, ntiles);
        if (fv) f.advance(sch, ntiles);
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ---------------- MMA issuers: warp 1 (SM sub-partition 1) owns the rows of half 0, warp 2
    // (sub-partition 2) those of half 1 -- S_h, KV_h and O_h are independent, and each issuer shares
    // its sub-partition with ex2-bound epilogue warps, so the issue work is split between two.
    // Kept lean: ring / buffer indices and phase bits are counters; each MMA batch is one asm with
    // immediates off warp-uniform bases, issued by an elected thread. ----------------
    const int h = warp - 1;
    constexpr uint32_t idesc_s = idesc_f16(128, BN2, 0, 0);   // A, B K-major, N = 64
    constexpr uint32_t idesc_o = idesc_f16(128, TN, 0, 1);    // A (TMEM) K-major, B MN-major
    Cur kv, s;
    kv.start(sch, ntiles);
    s = kv;
    // K-major features: LBO = 128 B (K-adjacent core), SBO = KF/8 * 128 B (8-row groups);
    // V planes MN-major: LBO = TN/8 * 128 B, SBO = 128 B.
    const uint64_t da0 = smem_desc(smem_u32(abuf) + h * (C::A_BYTES / 2), 128, (KF2 / 8) * 128);
    const uint64_t dpro = smem_desc(smem_u32(pro), 128, (KF2 / 8) * 128);
    const uint64_t dring_f = smem_desc(smem_u32(ring) + 2 * C::V_BYTES, 128, (KF2 / 8) * 128);
    const uint64_t dring_v = smem_desc(smem_u32(ring), (TN / 8) * 128, 128);
    const uint32_t tb_h = tbase + 64 * h;         // half h of every S / K buffer
    const uint32_t to_h0 = tbase + TMO + TN * h;   // O_h of slot 0 (slot 1 at + 2 TN)
    if (kv.valid(sch)) {
      mbar_wait(&bars->a_full[0], 0);
      mbar_wait(&bars->pro_full, 0);
      fence_after_sync();
      for (int i = 0; i < NB2 && s.valid(sch) && s.k == 0; ++i) {
        const uint32_t d = __shfl_sync(0xffffffffu, tb_h + i * 128, 0);
        const uint64_t db = shfl64(dpro + (uint64_t)((i * C::F_BYTES) >> 4));
        const bool last = s.jj == s.njt - 1;
        if (elect_one()) {
          mma_s2(d, da0, db, idesc_s);
          commit_one(&bars->s_full[i][h]);
          if (last) commit_one(&bars->a_empty[0]);
        }
        __syncwarp();
        s.advance(sch, ntiles);
      }
    }
    // tiles of this CTA: the loop below runs on the producer's per-stage flags only
    int ntot = 0;
    for (int u = blockIdx.x; u < sch.nunits(); u += gridDim.x) {
      const int split = (u / sch.chunks) % sch.nsplit();
      ntot += ntiles * (split + 1) / sch.nsplit() - ntiles * split / sch.nsplit();
    }
    int st = 0, b = 0;
    uint32_t ph_st = 0, ph_b = 0;
    for (int g = 0; g < ntot; ++g) {
      if (h == 0) T2_STAMP(1, g);
      mbar_wait(&bars->full[st], ph_st);
      const uint32_t fl = __shfl_sync(0xffffffffu, *reinterpret_cast<volatile uint32_t*>(&bars->flags[st]), 0);
      if (h == 0) T2_STAMP(3, g);
      mbar_wait(&bars->k_full[b][h], ph_b);
      if (h == 0) T2_STAMP(2, g);
      const int oslot = (fl & F_OSLOT) ? 1 : 0;
      if (fl & F_OWAIT) mbar_wait(&bars->o_empty[oslot][h], (fl & F_OPH) ? 1u : 0u);
      const uint32_t to_h = to_h0 + oslot * 2 * TN;
      fence_after_sync();
      const uint32_t soff16 = (uint32_t)((st * C::STAGE) >> 4);
      // __shfl_sync(.., 0): values the compiler treats as warp-uniform (uniform registers, no
      // per-MMA R2UR / VOTEU in the issue sequence)
      const uint32_t kbu = __shfl_sync(0xffffffffu, tb_h + b * 128, 0);
      const uint64_t dvu = shfl64(dring_v + soff16);
      if (elect_one()) {
        if (!(args.dbg & 1)) {
          if (lowp) mma_kv8<TN>(to_h, kbu, dvu, idesc_o, fl & F_ACC);
          else mma_kv12<TN>(to_h, kbu, dvu, idesc_o, fl & F_ACC);
        }
        if (fl & F_OLAST) commit_one(&bars->o_full[oslot][h]);
      }
      __syncwarp();
      if (h == 0) T2_STAMP(9, g);
      if (fl & F_SVALID) {   // S(g+3): its features are in stage g (skewed ring); buffer b is free
        const int kb = (fl & F_KB) ? 1 : 0;
        if (fl & F_SFIRST) mbar_wait(&bars->a_full[kb], (fl & F_APH) ? 1u : 0u);
        const uint64_t dau = shfl64(da0 + (uint64_t)(kb * (C::A_BYTES >> 4)));
        const uint64_t dfu = shfl64(dring_f + soff16);
        if (elect_one()) {
          mma_s2(kbu, dau, dfu, idesc_s);
          commit_one(&bars->s_full[b][h]);
          if (fl & F_SLAST) commit_one(&bars->a_empty[kb]);
        }
        __syncwarp();
        if (h == 0) T2_STAMP(8, g);
      }
      if (elect_one()) commit_one(&bars->empty[st]);
      __syncwarp();
      if (++st == C::STAGES) { st = 0; ph_st ^= 1; }
      if (++b == NB2) { b = 0; ph_b ^= 1; }
    }
  } else if (warp >= EPI0) {
    // ---------------- epilogue: 16 warps; warp w works on TMEM lane quarter q = w % 4.  Two groups
    // of 8 warps take alternate tiles (group = (w - 4) / 8), a warp covers half h = ((w - 4) / 4) % 2,
    // both 32-column chunks -- while one group sits in its TMEM load / store / barrier latencies the
    // other keeps the SFU busy. ----------------
    const int q = warp % 4;
    const int grp = (warp - EPI0) >> 3;
    const int h = ((warp - EPI0) >> 2) & 1;
    constexpr int NCH = 2;      // 32-column chunks per warp per tile
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    // read-out scratch of this warp (h, q) of the reading group
    float* rbuf = reinterpret_cast<float*>(smem + C::RO_OFF + (h * 4 + q) * RO_BYTES);
    Cur c;
    c.start(sch, ntiles);
    // the unit before c's unit (valid once c has left the CTA's first unit): (u, k) only, decoded
    // when it is read out (registers: the epilogue runs at the 96-per-thread cap)
    int pu_u = c.u, pu_k = c.k;
    // Read-out of a finished unit: the group that takes tile 0 of unit k reads out all TN columns of
    // O_h of unit k-1 (the first KV of unit k waits for that group only), in passes of 16 columns.
    // O arrives row-per-lane (TMEM lane = row); it goes through a swizzled shared-memory transpose
    // so that V is loaded and P stored coalesced (lane -> rows lane/4 + 8k, 4 columns at 4 (lane%4)):
    // row-per-lane global accesses cost 32 L1 wavefronts per instruction, and a read-out was ~10k
    // cycles of L1 traffic (measured with the per-tile trace).
    constexpr int NP = TN / 16;
    auto readout = [&](int uu, int kk) {
      Cur u;
      u.u = uu;
      u.k = kk;
      u.decode(sch, ntiles);
      const int64_t ib = args.row0 + (int64_t)u.rt * BM2 + 128 * h + 32 * q;   // first row of the warp
      const int colu = u.chunk * TN;
      const int ch = lane & 3, rl = lane >> 2;
      // coalesced layout: rows ib + rl + 8 k (k = 0..3), columns c0 + 4 ch .. + 3
      auto vload = [&](int c0, float4 (&v)[4]) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t i = ib + rl + 8 * k;
          v[k] = i < args.row1 ? __ldg(reinterpret_cast<const float4*>(args.v + (size_t)i * args.tp + colu + c0 + 4 * ch))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
      float* pbase = args.p + (size_t)u.split * args.p_split_stride + colu + 4 * ch;
      double* ap = args.apart ? args.apart + ((size_t)(u.rt * sch.nsplit() + u.split) * 8 + q * 2 + h) * args.tp + colu
                              : nullptr;
      if (warp == 4 || warp == 12) T2_STAMP(10, u.k);
      // V one pass ahead (its L2 latency overlaps the O wait and the previous pass)
      float4 vn[4];
      vload(0, vn);
      const int oslot = u.k % NO2;
      mbar_wait(&bars->o_full[oslot][h], (u.k / NO2) & 1);
      if (warp == 4 || warp == 12) T2_STAMP(11, u.k);
      fence_after_sync();
      const int sw = (lane >> 1) & 3;   // swizzle of this lane's row in the row-per-lane phase
#pragma unroll 1
      for (int pass = 0; pass < NP; ++pass) {
        const int c0 = pass * 16;
        float4 vc[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) vc[k] = vn[k];
        uint32_t o[16];
        const uint32_t ta = tbase + TMO + oslot * 2 * TN + TN * h + c0 + lane_base;
        tmem_ld8(ta, &o[0]);
        tmem_ld8(ta + 8, &o[8]);
        if (pass + 1 < NP) vload(c0 + 16, vn);
        const float4 s4 = __ldg(reinterpret_cast<const float4*>(args.inv_scale + colu + c0 + 4 * ch));
        tmem_ld_wait();
        if (pass == NP - 1) {   // O_h is in registers: the next unit's first KV may overwrite it
          fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars->o_empty[oslot][h]);
          if (warp == 4 || warp == 12) T2_STAMP(12, u.k);
        }
        // row-per-lane -> smem: row = lane, 16-byte chunk j at position j ^ ((row >> 1) & 3)
        // (conflict-free for both phases: 8 lanes of a wavefront hit 8 distinct 4-bank groups)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint4*>(rbuf + lane * 16 + ((j ^ sw) << 2)) = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
        __syncwarp();
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int r = rl + 8 * k;
          const float4 ov = *reinterpret_cast<const float4*>(rbuf + r * 16 + ((ch ^ ((r >> 1) & 3)) << 2));
          const float4 vv = vc[k];
          float4 r4;
          r4.x = args.o2 * ov.x * s4.x;
          r4.y = args.o2 * ov.y * s4.y;
          r4.z = args.o2 * ov.z * s4.z;
          r4.w = args.o2 * ov.w * s4.w;
          if (u.split == 0 && !args.no_diag) {
            r4.x = fmaf(args.diag, vv.x, r4.x); r4.y = fmaf(args.diag, vv.y, r4.y);
            r4.z = fmaf(args.diag, vv.z, r4.z); r4.w = fmaf(args.diag, vv.w, r4.w);
          }
          const int64_t i = ib + r;
          if (i < args.row1) *reinterpret_cast<float4*>(pbase + (size_t)(i - args.row0) * args.tp + c0) = r4;
          a0 = fmaf(vv.x, r4.x, a0); a1 = fmaf(vv.y, r4.y, a1); a2 = fmaf(vv.z, r4.z, a2); a3 = fmaf(vv.w, r4.w, a3);
        }
        __syncwarp();   // rbuf is rewritten by the next pass
        if (ap != nullptr) {   // alpha partials of the warp's 32 rows: sum over the 8 lanes of column chunk ch
#pragma unroll
          for (int xo = 4; xo < 32; xo <<= 1) {
            a0 += __shfl_xor_sync(0xffffffffu, a0, xo);
            a1 += __shfl_xor_sync(0xffffffffu, a1, xo);
            a2 += __shfl_xor_sync(0xffffffffu, a2, xo);
            a3 += __shfl_xor_sync(0xffffffffu, a3, xo);
          }
          if (rl == 0) {
            double* d = ap + c0 + 4 * ch;
            d[0] = a0; d[1] = a1; d[2] = a2; d[3] = a3;
          }
        }
      }
      if (warp == 4 || warp == 12) T2_STAMP(13, u.k);
    };
    // L2 prefetch of this warp's V rows of unit u (read ~njt tiles later by the read-out): the
    // warp's 32 rows x TN columns, one 128-byte line per lane and step
    auto prefetch_v = [&](const Cur& u) {
      const int64_t ib = args.row0 + (int64_t)u.rt * BM2 + 128 * h + 32 * q;
      constexpr int LPR = TN * 4 / 128 > 0 ? TN * 4 / 128 : 1;   // 128-byte lines per row
#pragma unroll
      for (int e = lane; e < 32 * LPR; e += 32) {
        const int64_t i = ib + e / LPR;
        if (i < args.row1)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(args.v + (size_t)i * args.tp + u.chunk * TN + (e % LPR) * 32));
      }
    };
    int b = 0;
    uint32_t ph_b = 0;
    int g = 0;
    for (; c.valid(sch); ++g) {
      if ((g & 1) == grp) {
        mbar_wait(&bars->s_full[b][h], ph_b);
        if (warp == 4) T2_STAMP(4, g);
        fence_after_sync();
#pragma unroll 1
        for (int ch = 0; ch < NCH; ++ch) {
          const int cc = ch;
          const uint32_t tb = tbase + b * 128 + 64 * h + 32 * cc + lane_base;
          const int64_t jcol0 = (int64_t)c.J(args) * BN2 + 32 * cc;
          uint32_t sv[32];
          tmem_ld32(tb, sv);
          tmem_ld_wait();
          if (lowp) {   // second relaxation level: k_hi only
            uint32_t hi[16];
            if (jcol0 + 32 > n) exp_hi<KIND, true>(sv, hi, (int)(n - jcol0));
            else exp_hi<KIND, false>(sv, hi, 32);
            tmem_st16(tb, hi);
          } else {
            uint32_t hi[16], lo[16];
            if (args.dbg & 2) {
#pragma unroll
              for (int m = 0; m < 16; ++m) { hi[m] = sv[m]; lo[m] = sv[m + 16]; }
            } else if (jcol0 + 32 > n) {
              exp_split<KIND, true>(sv, hi, lo, (int)(n - jcol0));
            } else {
              exp_split<KIND, false>(sv, hi, lo, 32);
            }
            tmem_st16(tb, hi);
            tmem_st16(tb + 16, lo);
          }
        }
        tmem_st_wait();
        fence_before_sync();
        __syncwarp();
        if (warp == 4) T2_STAMP(5, g);
        if (warp == 19) T2_STAMP(6, g);
        if (lane == 0) mbar_arrive(&bars->k_full[b][h]);
        if (c.jj == 0) {
          prefetch_v(c);
          if (c.k > 0) readout(pu_u, pu_k);   // unit k-1 is complete (its last KV is issued)
        }
      }
      const int old_u = c.u, old_k = c.k;
      c.advance(sch, ntiles);
      if (!c.valid(sch) || c.k != old_k) { pu_u = old_u; pu_k = old_k; }
      if (++b == NB2) { b = 0; ph_b ^= 1; }
    }
    // the CTA's last unit: one group (all of its TN columns) / every warp (its column half)
    if (pu_u < sch.nunits() && grp == 0) readout(pu_u, pu_k);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    fence_after_sync();
    tmem_dealloc<512>(tbase);
  }
  if (args.alpha_out != nullptr) {   // fused alpha (TcArgs): this CTA's read-outs are complete
    const int tp = args.tp;
    for (int col = threadIdx.x; col < tp; col += NT2) {
      double sum = 0.0;
      for (int u = blockIdx.x; u < sch.nunits(); u += gridDim.x) {
        const int chunk = u % args.chunks;
        if (col / TN != chunk) continue;
        const size_t r0 = (size_t)(u / args.chunks) * 8;   // rows (rt * nsplit + split) * 8 + (q, h) slot
#pragma unroll
        for (int sl = 0; sl < 8; ++sl) sum += args.apart[(r0 + sl) * tp + col];
      }
      args.cta_part[(size_t)blockIdx.x * tp + col] = sum;
    }
    __threadfence();
    __syncthreads();
    __shared__ bool s_last;
    if (threadIdx.x == 0) s_last = atomicAdd(args.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (s_last) {
      __threadfence();
      // the CTAs' rows in G = NT2 / tp contiguous groups (fixed), each summed in CTA order by one
      // thread per column (L2 loads, __ldcg: published by the other CTAs' fence + ticket), then the
      // groups in order
      double* s_grp = reinterpret_cast<double*>(smem);   // [NT2]: the ring is free now
      const int nb = (int)gridDim.x;
      const int G = tp <= NT2 ? NT2 / tp : 1;
      const int grp = threadIdx.x / tp, col = threadIdx.x % tp;
      if (grp < G) {
        const int b0 = nb * grp / G, b1 = nb * (grp + 1) / G;
        double sum = 0.0;
        int b = b0;
        for (; b + 4 <= b1; b += 4) {
          double x[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) x[e] = __ldcg(args.cta_part + (size_t)(b + e) * tp + col);
#pragma unroll
          for (int e = 0; e < 4; ++e) sum += x[e];
        }
        for (; b < b1; ++b) sum += __ldcg(args.cta_part + (size_t)b * tp + col);
        if (tp <= NT2) s_grp[threadIdx.x] = sum;
      }
      __syncthreads();
      for (int cc = threadIdx.x; cc < tp; cc += NT2) {
        double sum = 0.0;
        if (tp <= NT2) {
          for (int gg = 0; gg < G; ++gg) sum += s_grp[gg * tp + cc];
        } else {
          for (int bb = 0; bb < nb; ++bb) sum += __ldcg(args.cta_part + (size_t)bb * tp + cc);
        }
        const double nr = args.alpha_nrm[cc];
        args.alpha_out[cc] = args.alpha_frozen[cc] ? 0.0 : sum / (nr * nr);
      }
      if (threadIdx.x == 0) *args.ticket = 0u;   // for the next launch (stream-ordered)
    }
  }
}

template <int KIND, int TN>
cudaError_t launch2(const TcArgs& a, int grid, cudaStream_t s) {
  auto k = mvm_tc2_kernel<KIND, TN>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg2<TN>::SMEM);
  if (e != cudaSuccess) return e;
  k<<<grid, NT2, Cfg2<TN>::SMEM, s>>>(a);
  return cudaGetLastError();
}

template <int KIND>
cudaError_t launch2_kind(const TcArgs& a, int tn, int grid, cudaStream_t s) {
  switch (tn) {
    case 16: return launch2<KIND, 16>(a, grid, s);
    case 32: return launch2<KIND, 32>(a, grid, s);
    case 64: return launch2<KIND, 64>(a, grid, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int tc2_units(int64_t rows, int nsplit, int chunks) { return (int)((rows + BM2 - 1) / BM2) * nsplit * chunks; }

// Column splits of the unit grid: enough units for the persistent CTAs to finish together
// (max units per CTA x tiles per unit minimal), each split keeping >= min_tiles column tiles, and at most
// kMaxChain tiles per unit.  The chain bound is an accuracy bound: the tensor core adds each MMA
// into the fp32 TMEM accumulator with a round-toward-zero bias, measured on B200 as a relative
// shrink of ~1.1e-8 per accumulated MMA (12 per tile).  It is the error that dominates the
// full-size solve: at C3 the solve's error against the float64 oracle is proportional to the chain
// length (profiles/chain_nsplit_r02.txt: 264 / 130 / 65 / 33 tiles -> 2.6e-4 / 1.35e-4 / 7.0e-5 /
// 3.6e-5, same rule and J; a numpy emulation of the round-toward-zero accumulation,
// scripts/diag_rz_chain.py, shows the same proportionality), while fp32 vectors and fp32 kernel
// entries alone give ~1e-5 (scripts/diag_fp32_floor.py).  66 tiles keep C3 inside north_star's
// 1e-4.  The per-split partial products are summed in fp32 (round to
// nearest) by the consumer.
int tc2_choose_nsplit(int64_t rows, int64_t n, int chunks, int nsm, int min_tiles, int64_t max_chain) {
  const int64_t kMaxChain = max_chain > 0 ? max_chain : kTc2MaxChain;
  const int64_t nrt = (rows + BM2 - 1) / BM2;
  const int64_t ntiles = (n + BN2 - 1) / BN2;
  const int smin = (int)((ntiles + kMaxChain - 1) / kMaxChain);
  int best = smin;
  double best_cost = 1e300;
  for (int s = smin; s <= smin + 15; ++s) {
    if (ntiles / s < min_tiles && s > smin) break;
    const int64_t units = nrt * chunks * s;
    const int64_t per_cta = (units + nsm - 1) / nsm;
    const double cost = (double)per_cta * (double)((ntiles + s - 1) / s) * (1.0 + 0.002 * s);
    if (cost < best_cost * 0.995) { best_cost = cost; best = s; }
  }
  return best;
}

cudaError_t launch_mvm_tc2(const TcArgs& a, int nsm, cudaStream_t s) {
  const int tn = tc_chunk_cols(a.tp);
  const int cap = a.grid_cap > 0 && a.grid_cap < nsm ? a.grid_cap : nsm;
  const int grid = a.nunits < cap ? a.nunits : cap;
  switch (a.kind) {
    case 1: return launch2_kind<1>(a, tn, grid, s);
    case 2: return launch2_kind<2>(a, tn, grid, s);
    case 3: return launch2_kind<3>(a, tn, grid, s);
    case 11: return launch2_kind<4>(a, tn, grid, s);
    case 12: return launch2_kind<5>(a, tn, grid, s);
    case 13: return launch2_kind<6>(a, tn, grid, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ciq
