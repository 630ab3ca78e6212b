// kern_epi.cuh -- device pieces shared by the matrix-free tensor-core MVMs (mvm_tc2.cu, mvm_sym.cu):
// the kernel-function epilogue (S -> k -> split fp16 k_hi + k_lo), the distance-GEMM issue, and
// the elected-thread / commit helpers.  Internal linkage in each translation unit.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "tc_util.cuh"

// k = k_hi + k_lo by truncation (k_hi = k with the low 13 mantissa bits cleared, k_lo = k - k_hi in
// one packed FADD2): 2 LOP3 + FADD2 + 2 F2FP per pair instead of F2FP + 2 HADD2 + 2 FADD + F2FP
// (measured in this kernel: 0.908 vs 0.932 ms per C3 MVM, same accuracy).  CIQ_EPI_ROUND restores
// the rounding split.
#ifndef CIQ_EPI_ROUND
#define CIQ_EPI_TRUNC
#endif

namespace ciq {
namespace {

using namespace tc;

CIQ_DEVICE bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t@p mov.u32 %0, 1;\n\t}" : "+r"(pred));
  return pred != 0;
}

CIQ_DEVICE void commit_one(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

CIQ_DEVICE uint64_t shfl64(uint64_t v) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, 0), hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), 0);
  return ((uint64_t)hi << 32) | lo;
}

// KIND 1-3: RBF, Matern-5/2, Matern-3/2; KIND 4-6: their lengthscale derivatives l dk/dl / o^2
// (the hyper-parameter gradient, ciq_hyper_grad): r^2 e^{-r^2/2}, a^2 (1 + a) e^{-a} / 3, a^2 e^{-a}.
template <int KIND>
CIQ_DEVICE float kern(float s) {
  // s = -(log2 e / 2) r^2
  if (KIND == 1) return ex2_approx(s);
  if (KIND == 4) return (-1.3862943611198906f * s) * ex2_approx(s);
  // r^2 = -2 ln2 s; sqrt.approx (one MUFU.SQRT, ~2^-23 relative) instead of the IEEE sqrtf sequence
  // with its slow-path call
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

// Matern forms for a pair of entries with packed fp32x2 arithmetic (FMUL2 / FFMA2: half the
// FMA-pipe instructions of kern<>, whose epilogue is issue-bound); the
// constants are folded so that sqrt gives a = sqrt(c) r directly: a^2 = -(2 ln2 c) s.
CIQ_DEVICE uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
CIQ_DEVICE void upk2(uint64_t v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
CIQ_DEVICE uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
CIQ_DEVICE uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
template <int KIND>
CIQ_DEVICE void kern_pair(float s0, float s1, float& k0, float& k1) {
  // KIND 2: a = sqrt5 r, k = (1 + a + a^2/3) e^{-a};  KIND 3: a = sqrt3 r, k = (1 + a) e^{-a}
  constexpr float c2ln2 = KIND == 2 ? -6.931471805599453f : -4.1588830833596715f;   // -(2 ln2) * 5 or * 3
  const uint64_t x = mul2(pk2(s0, s1), pk2(c2ln2, c2ln2));
  float x0, x1;
  upk2(x, x0, x1);
  float a0, a1;
  // |x|: S can be a rounding-level negative at r ~ 0, where sqrt(|x|) ~ 0 is the right value and
  // the absolute value is a free operand modifier of MUFU.SQRT (no FMNMX)
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(a0) : "f"(fabsf(x0)));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(a1) : "f"(fabsf(x1)));
  const uint64_t a = pk2(a0, a1);
  const uint64_t e = mul2(a, pk2(-1.4426950408889634f, -1.4426950408889634f));
  float e0, e1;
  upk2(e, e0, e1);
  e0 = ex2_approx(e0);
  e1 = ex2_approx(e1);
  uint64_t poly;
  if (KIND == 2) poly = fma2(a, fma2(a, pk2(1.f / 3.f, 1.f / 3.f), pk2(1.f, 1.f)), pk2(1.f, 1.f));
  else poly = fma2(a, pk2(1.f, 1.f), pk2(1.f, 1.f));
  upk2(mul2(poly, pk2(e0, e1)), k0, k1);
}

template <int KIND, bool MASK>
CIQ_DEVICE void exp_split(const uint32_t (&sv)[32], uint32_t (&hi)[16], uint32_t (&lo)[16], int jvalid) {
#pragma unroll
  for (int c = 0; c < 32; c += 2) {
    float k0, k1;
#ifndef CIQ_NO_PAIR_MATERN
    if (KIND == 2 || KIND == 3) {
      kern_pair<KIND>(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1]), k0, k1);
    } else
#endif
    {
      k0 = kern<KIND>(__uint_as_float(sv[c]));
      k1 = kern<KIND>(__uint_as_float(sv[c + 1]));
    }
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

// Second relaxation level (params.mvm_relax): k rounded to fp16 only (one
// cvt.rn per pair, no low part) -- the late iterations' MVM uses K_hi . (V_hi + V_lo).
template <int KIND, bool MASK>
CIQ_DEVICE void exp_hi(const uint32_t (&sv)[32], uint32_t (&hi)[16], int jvalid) {
#pragma unroll
  for (int c = 0; c < 32; c += 2) {
    float k0, k1;
#ifndef CIQ_NO_PAIR_MATERN
    if (KIND == 2 || KIND == 3) {
      kern_pair<KIND>(__uint_as_float(sv[c]), __uint_as_float(sv[c + 1]), k0, k1);
    } else
#endif
    {
      k0 = kern<KIND>(__uint_as_float(sv[c]));
      k1 = kern<KIND>(__uint_as_float(sv[c + 1]));
    }
    if (MASK) {
      k0 = (c < jvalid) ? k0 : 0.f;
      k1 = (c + 1 < jvalid) ? k1 : 0.f;
    }
    hi[c / 2] = pack_half2(k0, k1);
  }
}

// S(J) of one 128-row half: two SS MMAs (K-steps of 16 over the K = 32 feature contraction),
// issued by one elected thread.  d: TMEM columns of the half; da: A descriptor of the half's rows;
// db: column features of the tile.  K-step: +256 B = +16 in descriptor units.
CIQ_DEVICE void mma_s2(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred t, f;\n\t.reg .b64 a1, b1;\n\t"
      "setp.ne.b32 t, %3, 0;\n\t"
      "setp.eq.b32 f, %3, 0;\n\t"
      "add.s64 a1, %1, 16;\n\t"
      "add.s64 b1, %2, 16;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, f;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, t;\n\t}" ::"r"(d),
      "l"(da), "l"(db), "r"(idesc)
      : "memory");
}

}  // namespace
}  // namespace ciq
