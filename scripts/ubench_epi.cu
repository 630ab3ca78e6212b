// ubench_epi.cu -- throughput of the instruction mix of the K1 epilogue (ex2 + fp16 split), to
// locate the per-SM bound of mvm_tc_kernel's exponentiation phase.  Standalone experiment:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench scripts/ubench_epi.cu && /tmp/ubench
#include <cuda_fp16.h>
#include <cstdio>

__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ unsigned pack(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<unsigned*>(&h);
}
// degree-3 minimax-ish exp2 on the FMA pipe (Cody-Waite: 2^x = 2^floor(x) * p(frac))
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float f = floorf(x);
  const float r = x - f;
  float p = fmaf(r, 0.0555041086648216f, 0.2402265069591007f);
  p = fmaf(p, r, 0.6931471805599453f);
  p = fmaf(p, r, 1.0f);
  return __int_as_float(__float_as_int(p) + ((int)f << 23));
}

template <int MODE>
__global__ void bench(float* out, int iters, float seed) {
  float s[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) s[k] = -0.001f * (threadIdx.x + k) * seed;
  unsigned acc = 0;
  float facc = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; k += 2) {
      const float a = s[k] - it * 1e-7f, b = s[k + 1] - it * 1e-7f;  // 2 FADD (or FFMA) per pair
      if (MODE == 0) {  // MUFU only
        facc += ex2a(a) + ex2a(b);
      } else if (MODE == 1) {  // F2FP only
        acc ^= pack(a, b);
      } else if (MODE == 2) {  // full rounding split
        const float k0 = ex2a(a), k1 = ex2a(b);
        const unsigned h = pack(k0, k1);
        const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h));
        acc ^= h ^ pack(k0 - hf.x, k1 - hf.y);
      } else if (MODE == 3) {  // split without exp
        const unsigned h = pack(a, b);
        const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h));
        acc ^= h ^ pack(a - hf.x, b - hf.y);
      } else if (MODE == 4) {  // polynomial exp + split
        const float k0 = ex2_poly(a), k1 = ex2_poly(b);
        const unsigned h = pack(k0, k1);
        const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h));
        acc ^= h ^ pack(k0 - hf.x, k1 - hf.y);
      } else if (MODE == 5) {  // half the pairs on MUFU, half polynomial
        const float k0 = ex2a(a), k1 = ex2_poly(b);
        const unsigned h = pack(k0, k1);
        const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h));
        acc ^= h ^ pack(k0 - hf.x, k1 - hf.y);
      } else if (MODE == 6) {  // truncation split (no round trip)
        const float k0 = ex2a(a), k1 = ex2a(b);
        const float h0 = __uint_as_float(__float_as_uint(k0) & 0xFFFFE000u);
        const float h1 = __uint_as_float(__float_as_uint(k1) & 0xFFFFE000u);
        acc ^= pack(h0, h1) ^ pack(k0 - h0, k1 - h1);
      } else if (MODE == 7) {  // cvt.rn.f16x2 of both halves via one F2FP each + HADD2.F32 pair
        facc += __half2float(__float2half_rn(a)) + __half2float(__float2half_rn(b));
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = facc + (float)acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int iters = 4096;
  const char* names[] = {"mufu ex2 only", "f2fp pack only", "ex2 + round split", "round split (no exp)",
                         "poly exp + split", "half mufu half poly + split", "ex2 + trunc split", "cvt f16 round trip"};
  for (int mode = 0; mode < 8; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      const int blocks = 148 * 4, threads = 512;
      cudaEventRecord(e0);
      switch (mode) {
        case 0: bench<0><<<blocks, threads>>>(out, iters, 1.f); break;
        case 1: bench<1><<<blocks, threads>>>(out, iters, 1.f); break;
        case 2: bench<2><<<blocks, threads>>>(out, iters, 1.f); break;
        case 3: bench<3><<<blocks, threads>>>(out, iters, 1.f); break;
        case 4: bench<4><<<blocks, threads>>>(out, iters, 1.f); break;
        case 5: bench<5><<<blocks, threads>>>(out, iters, 1.f); break;
        case 6: bench<6><<<blocks, threads>>>(out, iters, 1.f); break;
        case 7: bench<7><<<blocks, threads>>>(out, iters, 1.f); break;
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 1) {
        const double elems = (double)blocks * threads * iters * 16;
        printf("%-30s %8.3f ms  %7.2f Gelem/s  %6.2f elem/clk/SM (at %d MHz nominal)\n", names[mode], ms,
               elems / ms * 1e-6, elems / (ms * 1e-3) / 148 / (clk_khz * 1e3), clk_khz / 1000);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
