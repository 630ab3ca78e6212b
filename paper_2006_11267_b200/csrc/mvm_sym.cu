// mvm_sym.cu -- the symmetric-tile matrix-free kernel MVM (§8(a) row a4):
// P = K(X, X) V + sigma^2 V with every kernel value of the strict upper triangle evaluated ONCE and
// used twice, k(x_i, x_j) = k(x_j, x_i) (K is symmetric), so the SFU-bound epilogue
// (ex2, and sqrt for Matern) does half the work of mvm_tc2.cu.
//
// Geometry: 128 x 128 tiles (R, C) of the N x N kernel matrix, row block R <= column block C.
//   * forward product  O_R += K_RC V_C  (TS: A = K from TMEM, as in mvm_tc2.cu);
//   * transposed product  O'_C += K_RC^T V_R  (SS: A = K^T from shared memory -- the epilogue
//     writes k_hi / k_lo there too, in the MN-major operand layout, so the same bits serve as
//     A = K^T without a transpose), skipped on the diagonal tile R = C.
// A unit is (column group G: B consecutive column blocks, row range k: A_ROWS row blocks), tiles
// walked row by row, c >= r only.  Row r's forward product accumulates over its tiles of the
// unit in TMEM (double-buffered); the B transposed products of the group accumulate over the
// unit's rows in B TMEM accumulators.  Each accumulator is written once per unit as an fp32
// partial product to a slot of its 128-row block; sym_reduce_kernel sums the slots of each block
// in a fixed order (deterministic), applies o^2 * 2^-e_c and sigma^2 V, and forms the fixed-order
// alpha partials.  Accumulation chains are <= B or A_ROWS tiles (<= 384 MMAs), far below the
// round-toward-zero bias bound of mvm_tc2.cu.
//
// TMEM (512 columns): NB S/K buffers b at [128 b, 128 b + 128) (K in place, 32-column chunk c
// -> k_hi at [32c, 32c+16), k_lo at [32c+16, 32c+32)); forward O at [128 NB, 128 NB + 2 TN); the B
// transposed accumulators after it.
// Smem: two K^T buffers (hi | lo, 32 KB each; buffer = tile parity = epilogue group), two row
// buffers (features + V planes of row block R), and a ring of column-block stages (V_C planes +
// features of C).
// Roles: warp 0 producer (bulk copies), warp 1 S + forward issuer, warp 2 transposed issuer,
// warps 4-19 epilogue in two ping-pong groups of 8 (tile parity); each group also reads out the
// accumulators that the previous tile completed.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "internal.h"
#include "kern_epi.cuh"
#include "tc_util.cuh"

namespace ciq {
namespace {

using namespace tc;

constexpr int SB = 128;       // tile rows = tile columns
constexpr int KFS = 32;       // feature contraction (d <= 8)
constexpr int NTS = 640;      // 4 role warps + 16 epilogue warps
constexpr int EPI0S = 4;
constexpr int A_ROWS = 16;    // row blocks per unit
#ifndef CIQ_SYM_SLEEP
#define CIQ_SYM_SLEEP 64
#endif

template <int TN>
struct CfgS {
  // TMEM S/K buffers: three for 16-column chunks (S runs two tiles ahead of the epilogue; with
  // two, each group waited for S(g + 2) behind KV(g): 19% of the epilogue's stall samples at C5,
  // profiles/ncu_sym_c5_r02.txt); the rest of the 512 columns holds the accumulators
  static constexpr int NB = TN == 16 ? 3 : 2;
  static constexpr int B = TN == 16 ? 6 : 6;             // column blocks per group
  static constexpr int ST = TN == 16 ? 3 : 2;            // ring stages
  static constexpr int KT_PLANE = SB * SB * 2;           // one fp16 plane of a K^T tile (32 KB)
  static constexpr int F_BYTES = SB * KFS * 2;           // features of one block (8 KB)
  static constexpr int V_BYTES = SB * TN * 2;            // one V plane of one block
  static constexpr int ROW = F_BYTES + 2 * V_BYTES;      // row buffer: feat_R | V_R hi | V_R lo
  static constexpr int STAGE = 2 * V_BYTES + F_BYTES;    // ring stage: V_C hi | V_C lo | feat_C
  static constexpr int ROW_OFF = 4 * KT_PLANE;
  static constexpr int RING_OFF = ROW_OFF + 2 * ROW;
  static constexpr int BAR_OFF = RING_OFF + ST * STAGE;
  static constexpr int SMEM = 1024 + BAR_OFF + 1024;
  static constexpr int TM_O = NB * 128;
  static constexpr int TM_T = NB * 128 + 2 * TN;
};
static_assert(CfgS<16>::TM_T + CfgS<16>::B * 16 <= 512, "TMEM budget");
static_assert(CfgS<32>::TM_T + CfgS<32>::B * 32 <= 512, "TMEM budget");
static_assert(CfgS<16>::SMEM <= 227 * 1024 && CfgS<32>::SMEM <= 227 * 1024, "shared memory budget");

// Waits of the MMA issuers on the epilogue (k_full): most of their time; polled with a short
// sleep so they do not take issue slots from the epilogue warps of their sub-partitions
// (measured: C3-shaped, 16 RHS 0.786 -> 0.757 ms; C5 unchanged).
CIQ_DEVICE void wait_issuer(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) __nanosleep(CIQ_SYM_SLEEP);
}

struct BarsS {
  uint64_t full[3], empty[3];          // ring
  uint64_t rfull[2], rempty[2];        // row buffers (rempty: S issuer + transposed issuer)
  uint64_t s_full[3], k_full[3];       // S(g) in TMEM buffer g % NB; K(g) written (TMEM + smem)
  uint64_t kt_empty[2];                // transposed MMAs of tile g done with K^T buffer g & 1
  uint64_t o_full[2], o_empty[2];      // forward accumulators (row parity)
  uint64_t t_full[12], t_empty[12];    // transposed accumulators
  uint32_t tmem_base;
};
static_assert(sizeof(BarsS) <= 1024, "barrier block");

// Position in the tile sequence of one CTA.  Units u = blockIdx.x + i * gridDim.x over
// sym_units (x chunks); unit: column blocks [c0, c1), row blocks [r0, r1); tile (r, c), c >= r.
struct SCur {
  int u, chunk, G, k, r0, r1, c0, c1, r, c, rowseq;
  CIQ_DEVICE void load(const TcArgs& a) {
    const int2 e = a.sym_units[u / a.chunks];
    chunk = u % a.chunks;
    G = e.x;
    k = e.y;
    c0 = G * a.sym_b;
    c1 = min(c0 + a.sym_b, a.sym_nb);
    r0 = k * A_ROWS;
    r1 = min(min(r0 + A_ROWS, a.sym_nb), c1);
    r = r0;
    c = max(r, c0);
  }
  CIQ_DEVICE void start(const TcArgs& a) {
    u = blockIdx.x;
    rowseq = 0;
    if (u < a.nunits) load(a);
  }
  CIQ_DEVICE bool valid(const TcArgs& a) const { return u < a.nunits; }
  CIQ_DEVICE void advance(const TcArgs& a) {
    if (++c < c1) return;
    ++rowseq;
    if (++r < r1) {
      c = max(r, c0);
      return;
    }
    u += gridDim.x;
    if (u < a.nunits) load(a);
  }
  CIQ_DEVICE bool row_first() const { return c == max(r, c0); }
  CIQ_DEVICE bool row_last() const { return c == c1 - 1; }
  CIQ_DEVICE bool tv() const { return r < c; }
  CIQ_DEVICE bool t_first() const { return r < c && r == r0; }
  CIQ_DEVICE bool t_last() const { return r < c && r == min(r1, c) - 1; }
  CIQ_DEVICE int ci() const { return c - c0; }
};

// Forward KV of 4 K-steps (64 columns of the tile): O (+)= K . V_C, k_hi.v_hi + k_hi.v_lo +
// k_lo.v_hi per K-step; A from TMEM (kb: K-step s -> k_hi at 32 (s/2) + 8 (s%2), k_lo at +16),
// B = V_C MN-major (K-step s at +2 TN descriptor units, V_lo at +16 TN).
template <int TN>
CIQ_DEVICE void mma_fwd12(uint32_t o, uint32_t kb, uint64_t dv, uint32_t idesc, uint32_t acc) {
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
      "r"(kb), "l"(dv), "r"(idesc), "r"(acc), "n"(2 * TN), "n"(4 * TN), "n"(6 * TN), "n"(16 * TN),
      "n"(18 * TN), "n"(20 * TN), "n"(22 * TN)
      : "memory");
}

// Transposed product of 4 K-steps (64 rows of the tile): O' (+)= K^T . V_R, both operands from
// shared memory.  da: K^T hi plane (MN-major: K-step s = 16 rows of the tile at +256 descriptor
// units, the lo plane at +2048); db: V_R hi (K-step at +2 TN, V_lo at +16 TN).
template <int TN>
CIQ_DEVICE void mma_tr12(uint32_t o, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, t;\n\t.reg .b64 ah<4>, al<4>, bh<4>, bl<4>;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 t, %4, %4;\n\t"
      "add.s64 ah0, %1, 0;\n\t add.s64 ah1, %1, 256;\n\t add.s64 ah2, %1, 512;\n\t add.s64 ah3, %1, 768;\n\t"
      "add.s64 al0, %1, 2048;\n\t add.s64 al1, %1, 2304;\n\t add.s64 al2, %1, 2560;\n\t add.s64 al3, %1, 2816;\n\t"
      "add.s64 bh0, %2, 0;\n\t add.s64 bh1, %2, %5;\n\t add.s64 bh2, %2, %6;\n\t add.s64 bh3, %2, %7;\n\t"
      "add.s64 bl0, %2, %8;\n\t add.s64 bl1, %2, %9;\n\t add.s64 bl2, %2, %10;\n\t add.s64 bl3, %2, %11;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ah0, bh0, %3, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ah0, bl0, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], al0, bh0, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ah1, bh1, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ah1, bl1, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], al1, bh1, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ah2, bh2, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ah2, bl2, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], al2, bh2, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ah3, bh3, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], ah3, bl3, %3, t;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], al3, bh3, %3, t;\n\t}" ::"r"(o),
      "l"(da), "l"(db), "r"(idesc), "r"(acc), "n"(2 * TN), "n"(4 * TN), "n"(6 * TN), "n"(16 * TN),
      "n"(18 * TN), "n"(20 * TN), "n"(22 * TN)
      : "memory");
}

CIQ_DEVICE void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Partial-product slot of 128-row block X: the forward partial of column group G (G >= X / B),
// then the transposed partials of row ranges k (k * A_ROWS < X).
CIQ_DEVICE int slot_fwd(const TcArgs& a, int X, int G) { return a.sym_base[X] + (G - X / a.sym_b); }
CIQ_DEVICE int slot_tr(const TcArgs& a, int X, int k) { return a.sym_base[X] + (a.sym_ng - X / a.sym_b) + k; }

template <int KIND, int TN>
__global__ void __launch_bounds__(NTS, 1) mvm_sym_kernel(TcArgs args) {
  using C = CfgS<TN>;
  if (args.done != nullptr && args.done->done) return;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* rowb = smem + C::ROW_OFF;
  uint8_t* ring = smem + C::RING_OFF;
  BarsS* bars = reinterpret_cast<BarsS*>(smem + C::BAR_OFF);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t n = args.n;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::ST; ++s) { mbar_init(&bars->full[s], 1); mbar_init(&bars->empty[s], 1); }
    for (int b = 0; b < C::NB; ++b) { mbar_init(&bars->s_full[b], 1); mbar_init(&bars->k_full[b], 8); }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars->rfull[b], 1);
      mbar_init(&bars->rempty[b], 2);
      mbar_init(&bars->kt_empty[b], 1);
      mbar_init(&bars->o_full[b], 1);
      mbar_init(&bars->o_empty[b], 8);
    }
    for (int b = 0; b < C::B; ++b) { mbar_init(&bars->t_full[b], 1); mbar_init(&bars->t_empty[b], 8); }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem_base);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = bars->tmem_base;
  const size_t plane = (size_t)args.vrows * TN;   // one plane of one chunk

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      SCur t;
      t.start(args);
      for (int g = 0; t.valid(args); ++g) {
        const __half* vp = args.vplanes + (size_t)t.chunk * 2 * plane;
        if (t.row_first()) {   // row block r: its features (S's A operand) and V_R (the transposed B)
          const int rb = t.rowseq & 1;
          mbar_wait_backoff(&bars->rempty[rb], ((t.rowseq >> 1) & 1) ^ 1);
          uint8_t* dst = rowb + rb * C::ROW;
          mbar_arrive_expect_tx(&bars->rfull[rb], C::ROW);
          bulk_g2s(dst, args.feat_a + (size_t)t.r * SB * KFS, C::F_BYTES, &bars->rfull[rb]);
          bulk_g2s(dst + C::F_BYTES, vp + (size_t)t.r * SB * TN, C::V_BYTES, &bars->rfull[rb]);
          bulk_g2s(dst + C::F_BYTES + C::V_BYTES, vp + plane + (size_t)t.r * SB * TN, C::V_BYTES, &bars->rfull[rb]);
        }
        const int st = g % C::ST;
        mbar_wait_backoff(&bars->empty[st], ((g / C::ST) & 1) ^ 1);
        uint8_t* sb = ring + st * C::STAGE;
        mbar_arrive_expect_tx(&bars->full[st], C::STAGE);
        bulk_g2s(sb, vp + (size_t)t.c * SB * TN, C::V_BYTES, &bars->full[st]);
        bulk_g2s(sb + C::V_BYTES, vp + plane + (size_t)t.c * SB * TN, C::V_BYTES, &bars->full[st]);
        bulk_g2s(sb + 2 * C::V_BYTES, args.feat_b + (size_t)t.c * SB * KFS, C::F_BYTES, &bars->full[st]);
        t.advance(args);
      }
    }
  } else if (warp == 1) {
    // ---------------- S and forward-product issuer ----------------
    constexpr uint32_t idesc_s = idesc_f16(128, SB, 0, 0);   // features K-major, N = 128
    constexpr uint32_t idesc_o = idesc_f16(128, TN, 0, 1);   // A (TMEM), B = V MN-major
    // K-major features: LBO = 128 B, SBO = KF/8 * 128 B; V planes MN-major: LBO = TN/8 * 128 B, SBO = 128 B
    const uint64_t drow_f = smem_desc(smem_u32(rowb), 128, (KFS / 8) * 128);
    const uint64_t dring_f = smem_desc(smem_u32(ring) + 2 * C::V_BYTES, 128, (KFS / 8) * 128);
    const uint64_t dring_v = smem_desc(smem_u32(ring), (TN / 8) * 128, 128);
    SCur kv, s;
    kv.start(args);
    s = kv;
    int gs = 0;
    auto issue_s = [&]() {   // S(gs) into TMEM buffer gs % NB (its previous K consumed by KV(gs - NB))
      const int st = gs % C::ST;
      mbar_wait(&bars->full[st], (gs / C::ST) & 1);
      const int rb = s.rowseq & 1;
      if (s.row_first()) mbar_wait(&bars->rfull[rb], (s.rowseq >> 1) & 1);
      fence_after_sync();
      const int sbuf = gs % C::NB;
      const uint32_t d = __shfl_sync(0xffffffffu, tbase + sbuf * 128, 0);
      const uint64_t da = shfl64(drow_f + (uint64_t)((rb * C::ROW) >> 4));
      const uint64_t db = shfl64(dring_f + (uint64_t)((st * C::STAGE) >> 4));
      const bool last = s.row_last();
      if (elect_one()) {
        mma_s2(d, da, db, idesc_s);
        commit_one(&bars->s_full[sbuf]);
        if (last) commit_one(&bars->rempty[rb]);
      }
      __syncwarp();
      s.advance(args);
      ++gs;
    };
    for (int i = 0; i < C::NB && s.valid(args); ++i) issue_s();
    for (int g = 0; kv.valid(args); ++g) {
      const int kbuf = g % C::NB;
      wait_issuer(&bars->k_full[kbuf], (g / C::NB) & 1);
      const int fb = kv.rowseq & 1;
      const bool first = kv.row_first(), last = kv.row_last();
      if (first) mbar_wait(&bars->o_empty[fb], ((kv.rowseq >> 1) & 1) ^ 1);
      fence_after_sync();
      const int st = g % C::ST;
      const uint32_t o = __shfl_sync(0xffffffffu, tbase + C::TM_O + fb * TN, 0);
      const uint32_t kb = __shfl_sync(0xffffffffu, tbase + kbuf * 128, 0);
      const uint64_t dv = shfl64(dring_v + (uint64_t)((st * C::STAGE) >> 4));
      if (elect_one()) {
        mma_fwd12<TN>(o, kb, dv, idesc_o, first ? 0u : 1u);
        mma_fwd12<TN>(o, kb + 64, dv + (uint64_t)(8 * TN), idesc_o, 1u);
        commit_one(&bars->empty[st]);
        if (last) commit_one(&bars->o_full[fb]);
      }
      __syncwarp();
      kv.advance(args);
      if (s.valid(args)) issue_s();
    }
  } else if (warp == 2) {
    // ---------------- transposed-product issuer ----------------
    constexpr uint32_t idesc_t = idesc_f16(128, TN, 1, 1);   // A = K^T MN-major, B = V MN-major
    const uint64_t dkt = smem_desc(smem_u32(smem), 16 * 128, 128);   // K^T: LBO = 16 core rows, SBO = 128 B
    const uint64_t drow_v = smem_desc(smem_u32(rowb) + C::F_BYTES, (TN / 8) * 128, 128);
    SCur t;
    t.start(args);
    uint32_t tused = 0, tpar = 0;
    for (int g = 0; t.valid(args); ++g) {
      wait_issuer(&bars->k_full[g % C::NB], (g / C::NB) & 1);
      const int rb = t.rowseq & 1;
      if (t.row_first()) mbar_wait(&bars->rfull[rb], (t.rowseq >> 1) & 1);
      const bool tv = t.tv(), tl = t.t_last(), rl = t.row_last();
      const int ci = t.ci();
      if (tv && t.t_first() && ((tused >> ci) & 1)) mbar_wait(&bars->t_empty[ci], ((tpar >> ci) & 1) ^ 1);
      fence_after_sync();
      const uint32_t o = __shfl_sync(0xffffffffu, tbase + C::TM_T + ci * TN, 0);
      const uint64_t da = shfl64(dkt + (uint64_t)(((g & 1) * 2 * C::KT_PLANE) >> 4));
      const uint64_t db = shfl64(drow_v + (uint64_t)((rb * C::ROW) >> 4));
      const uint32_t acc = t.t_first() ? 0u : 1u;
      if (elect_one()) {
        if (tv) {
          mma_tr12<TN>(o, da, db, idesc_t, acc);
          mma_tr12<TN>(o, da + 1024, db + (uint64_t)(8 * TN), idesc_t, 1u);
        }
        commit_one(&bars->kt_empty[g & 1]);
        if (tl) commit_one(&bars->t_full[ci]);
        if (rl) commit_one(&bars->rempty[rb]);
      }
      __syncwarp();
      if (tl) {
        tused |= 1u << ci;
        tpar ^= 1u << ci;
      }
      t.advance(args);
    }
  } else if (warp >= EPI0S) {
    // ---------------- epilogue: group grp = tile parity; warp covers TMEM lane quarter q and the
    // column half hh (two 32-column chunks) ----------------
    const int q = warp % 4;
    const int grp = (warp - EPI0S) >> 3;
    const int hh = ((warp - EPI0S) >> 2) & 1;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const int il = 32 * q + lane;   // row of the tile
    const uint32_t kt0 = smem_u32(smem) + ((il >> 3) << 11) + ((il & 7) << 4);
    constexpr int CPW = TN / 2;     // read-out columns per warp
    // accumulator read-out of a completed tile: forward (row r of unit (G, k)) and transposed
    // (column block c); rows of the partial slot = tile rows, columns [hh CPW, +CPW)
    struct Done {
      int fwd, tr, chunk, X_f, slot_f, fb, ph_f, ci, X_t, slot_t, ph_t;
    };
    auto readout_acc = [&](uint32_t tcol, uint64_t* full, uint32_t ph, uint64_t* empty, int chunk, int slot) {
      uint32_t o[CPW];
      mbar_wait(full, ph);
      fence_after_sync();
#pragma unroll
      for (int m = 0; m < CPW; m += 8) tmem_ld8(tbase + tcol + hh * CPW + m + lane_base, &o[m]);
      tmem_ld_wait();
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(empty);
      float* dst = args.sym_part + (((size_t)chunk * args.sym_slots + slot) * SB + il) * TN + hh * CPW;
#pragma unroll
      for (int m = 0; m < CPW; m += 4)
        *reinterpret_cast<float4*>(dst + m) = make_float4(__uint_as_float(o[m]), __uint_as_float(o[m + 1]),
                                                          __uint_as_float(o[m + 2]), __uint_as_float(o[m + 3]));
    };
    auto readout = [&](const Done& d) {
      if (d.fwd) readout_acc(C::TM_O + d.fb * TN, &bars->o_full[d.fb], d.ph_f, &bars->o_empty[d.fb], d.chunk, d.slot_f);
      if (d.tr) readout_acc(C::TM_T + d.ci * TN, &bars->t_full[d.ci], d.ph_t, &bars->t_empty[d.ci], d.chunk, d.slot_t);
    };
    SCur c;
    c.start(args);
    Done prev{};
    uint32_t tpar = 0;
    int g = 0;
    for (; c.valid(args); ++g) {
      if ((g & 1) == grp) {
        const int bb = g & 1, sb = g % C::NB;
        mbar_wait(&bars->s_full[sb], (g / C::NB) & 1);
        fence_after_sync();
        const uint32_t ktb = kt0 + bb * 2 * C::KT_PLANE;
#pragma unroll 1
        for (int ch = 0; ch < 2; ++ch) {
          const int cc = 2 * hh + ch;
          const uint32_t tb = tbase + sb * 128 + 32 * cc + lane_base;
          const int64_t jcol0 = (int64_t)c.c * SB + 32 * cc;
          uint32_t sv[32];
          tmem_ld32(tb, sv);
          tmem_ld_wait();
          uint32_t hi[16], lo[16];
          if (jcol0 + 32 > n) exp_split<KIND, true>(sv, hi, lo, (int)(n - jcol0));
          else exp_split<KIND, false>(sv, hi, lo, 32);
          tmem_st16(tb, hi);
          tmem_st16(tb + 16, lo);
          // the transposed MMAs of tile g - 2 must be done with this K^T buffer: waited for only
          // here, after the first chunk's kernel values (they overlap the MMAs' tail)
          if (ch == 0) mbar_wait(&bars->kt_empty[bb], ((g >> 1) & 1) ^ 1);
          // K^T operand: element (j, i) of the MN-major A at core (i / 8, j / 8), row i % 8
          const uint32_t kc = ktb + ((uint32_t)(4 * cc) << 7);
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            st_shared_v4(kc + (m << 7), hi[4 * m], hi[4 * m + 1], hi[4 * m + 2], hi[4 * m + 3]);
            st_shared_v4(kc + C::KT_PLANE + (m << 7), lo[4 * m], lo[4 * m + 1], lo[4 * m + 2], lo[4 * m + 3]);
          }
        }
        tmem_st_wait();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        fence_before_sync();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->k_full[sb]);
        if (g > 0) readout(prev);
      }
      // what tile g completes (read out by the group of tile g + 1)
      Done d{};
      d.chunk = c.chunk;
      if (c.row_last()) {
        d.fwd = 1;
        d.fb = c.rowseq & 1;
        d.ph_f = (c.rowseq >> 1) & 1;
        d.X_f = c.r;
        d.slot_f = slot_fwd(args, c.r, c.G);
      }
      if (c.t_last()) {
        d.tr = 1;
        d.ci = c.ci();
        d.ph_t = (tpar >> d.ci) & 1;
        tpar ^= 1u << d.ci;
        d.X_t = c.c;
        d.slot_t = slot_tr(args, c.c, c.k);
      }
      prev = d;
      c.advance(args);
    }
    if (g > 0 && (g & 1) == grp) readout(prev);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    fence_after_sync();
    tmem_dealloc<512>(tbase);
  }
}

// P rows of block X (all chunks): the fixed-order sum of the block's partial slots, scaled by
// o^2 2^-e_c, + sigma^2 V; alpha partials apart[X][col] = sum over the block's rows of v p.
template <int TN>
__global__ void __launch_bounds__(SB * TN / 4) sym_reduce_kernel(TcArgs a) {
  if (a.done != nullptr && a.done->done) return;
  constexpr int C4 = TN / 4;
  __shared__ double red[SB * TN];
  const int X = blockIdx.x, chunk = blockIdx.y;
  const int row = threadIdx.x / C4, c4 = threadIdx.x % C4;
  const int s0 = a.sym_base[X], s1 = a.sym_base[X + 1];
  const float4* part = reinterpret_cast<const float4*>(a.sym_part) + ((size_t)chunk * a.sym_slots * SB + row) * C4 + c4;
  const size_t sstride = (size_t)SB * C4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  int s = s0;
  for (; s + 4 <= s1; s += 4) {   // four loads in flight, summed in slot order
    const float4 p0 = part[(size_t)s * sstride], p1 = part[(size_t)(s + 1) * sstride];
    const float4 p2 = part[(size_t)(s + 2) * sstride], p3 = part[(size_t)(s + 3) * sstride];
    acc.x = (((acc.x + p0.x) + p1.x) + p2.x) + p3.x;
    acc.y = (((acc.y + p0.y) + p1.y) + p2.y) + p3.y;
    acc.z = (((acc.z + p0.z) + p1.z) + p2.z) + p3.z;
    acc.w = (((acc.w + p0.w) + p1.w) + p2.w) + p3.w;
  }
  for (; s < s1; ++s) {
    const float4 p0 = part[(size_t)s * sstride];
    acc.x += p0.x; acc.y += p0.y; acc.z += p0.z; acc.w += p0.w;
  }
  const int64_t i = (int64_t)X * SB + row;
  const int col = chunk * TN + 4 * c4;
  float4 r = make_float4(0.f, 0.f, 0.f, 0.f), v = r;
  if (i < a.n) {
    v = *reinterpret_cast<const float4*>(a.v + (size_t)i * a.tp + col);
    r.x = fmaf(a.diag, v.x, a.o2 * acc.x * a.inv_scale[col]);
    r.y = fmaf(a.diag, v.y, a.o2 * acc.y * a.inv_scale[col + 1]);
    r.z = fmaf(a.diag, v.z, a.o2 * acc.z * a.inv_scale[col + 2]);
    r.w = fmaf(a.diag, v.w, a.o2 * acc.w * a.inv_scale[col + 3]);
    *reinterpret_cast<float4*>(a.p + (size_t)i * a.tp + col) = r;
  }
  if (a.apart == nullptr) return;
  red[row * TN + 4 * c4 + 0] = (double)(v.x * r.x);
  red[row * TN + 4 * c4 + 1] = (double)(v.y * r.y);
  red[row * TN + 4 * c4 + 2] = (double)(v.z * r.z);
  red[row * TN + 4 * c4 + 3] = (double)(v.w * r.w);
  __syncthreads();
  for (int h = SB / 2; h > 0; h >>= 1) {   // fixed-order tree over the rows of the block
    for (int e = threadIdx.x; e < h * TN; e += blockDim.x) red[e] += red[e + h * TN];
    __syncthreads();
  }
  if (threadIdx.x < TN) a.apart[(size_t)X * a.tp + chunk * TN + threadIdx.x] = red[threadIdx.x];
}

template <int KIND, int TN>
cudaError_t launch_sym(const TcArgs& a, int grid, cudaStream_t s) {
  auto k = mvm_sym_kernel<KIND, TN>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgS<TN>::SMEM);
  if (e != cudaSuccess) return e;
  k<<<grid, NTS, CfgS<TN>::SMEM, s>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  sym_reduce_kernel<TN><<<dim3(a.sym_nb, a.chunks), SB * TN / 4, 0, s>>>(a);
  return cudaGetLastError();
}

template <int KIND>
cudaError_t launch_sym_kind(const TcArgs& a, int tn, int grid, cudaStream_t s) {
  switch (tn) {
    case 16: return launch_sym<KIND, 16>(a, grid, s);
    case 32: return launch_sym<KIND, 32>(a, grid, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

bool sym_supported(int tn) { return tn == 16 || tn == 32; }

int sym_group_blocks(int tn) { return tn == 16 ? CfgS<16>::B : CfgS<32>::B; }

// Units (column group G, row range k) of the upper block triangle, largest first (so the
// round-robin over persistent CTAs is balanced to within one unit), and the partial-slot prefix
// sums: block X owns (ng - X / B) forward slots and ceil(X / A_ROWS) transposed slots.
void sym_geometry(int64_t n, int tn, std::vector<int2>* units, std::vector<int>* base, int* ng, int* slots) {
  const int nb = (int)((n + SB - 1) / SB);
  const int B = sym_group_blocks(tn);
  *ng = (nb + B - 1) / B;
  units->clear();
  std::vector<std::pair<int, int2>> tmp;
  for (int G = 0; G < *ng; ++G) {
    const int c0 = G * B, c1 = std::min(c0 + B, nb);
    for (int k = 0; k * A_ROWS < c1; ++k) {
      const int r0 = k * A_ROWS, r1 = std::min(std::min(r0 + A_ROWS, nb), c1);
      int tiles = 0;
      for (int r = r0; r < r1; ++r) tiles += c1 - std::max(r, c0);
      tmp.push_back({tiles, make_int2(G, k)});
    }
  }
  std::stable_sort(tmp.begin(), tmp.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
  for (const auto& e : tmp) units->push_back(e.second);
  base->assign(nb + 1, 0);
  for (int X = 0; X < nb; ++X) (*base)[X + 1] = (*base)[X] + (*ng - X / B) + (X + A_ROWS - 1) / A_ROWS;
  *slots = (*base)[nb];
}

cudaError_t launch_mvm_sym(const TcArgs& a, int nsm, cudaStream_t s) {
  const int tn = tc_chunk_cols(a.tp);
  const int grid = a.nunits < nsm ? a.nunits : nsm;
  switch (a.kind) {
    case 1: return launch_sym_kind<1>(a, tn, grid, s);
    case 2: return launch_sym_kind<2>(a, tn, grid, s);
    case 3: return launch_sym_kind<3>(a, tn, grid, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace ciq
