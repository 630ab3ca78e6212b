// ubench_tmem.cu -- K1 epilogue building blocks in isolation (16 epilogue warps per CTA, 1 CTA/SM):
//   mode 0: tcgen05.ld 32x32b.x32 + wait::ld                       (TMEM read rate)
//   mode 1: tcgen05.st 32x32b.x16 x2 + wait::st                    (TMEM write rate)
//   mode 2: ld + wait + st x2 + wait                               (K1's TMEM traffic per chunk)
//   mode 3: mode 2 + ex2 + round split (the full epilogue chunk, no barriers)
//   mode 4: mode 3 with truncation split (FADD2)
//   mode 5: mode 3, ld of the NEXT chunk issued before the math of this one (software pipelined)
//   mode 6: ex2 + round split on registers only (no TMEM)
// Reports clk per 32x32 chunk per warp and elements/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2006_11267_b200/csrc -o /tmp/ubt scripts/ubench_tmem.cu
#include <cstdio>

#include "tc_util.cuh"

using namespace ciq::tc;

template <int MODE>
__device__ __forceinline__ void chunk_math(const uint32_t (&sv)[32], uint32_t (&hi)[16], uint32_t (&lo)[16]) {
#pragma unroll
  for (int c = 0; c < 32; c += 2) {
    const float k0 = ex2_approx(__uint_as_float(sv[c])), k1 = ex2_approx(__uint_as_float(sv[c + 1]));
    if (MODE == 4) {
      split_trunc2(k0, k1, hi[c / 2], lo[c / 2]);
    } else {
      const uint32_t h = pack_half2(k0, k1);
      const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h));
      hi[c / 2] = h;
      lo[c / 2] = pack_half2(k0 - hf.x, k1 - hf.y);
    }
  }
}

template <int MODE, int NW>
__global__ void __launch_bounds__(640, 1) tm(long long* out, int iters, volatile int* sink) {
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tb = tbase_s;
  if (warp >= 4 && warp < 4 + NW) {
    const int q = warp % 4, cw = (warp - 4) / 4;
    const uint32_t taddr = tb + ((uint32_t)(q * 32) << 16) + 32 * cw;
    uint32_t acc = 0;
    uint32_t sv[32], hi[16], lo[16];
#pragma unroll
    for (int m = 0; m < 32; ++m) sv[m] = __float_as_uint(-0.01f * (lane + m));
#pragma unroll
    for (int m = 0; m < 16; ++m) { hi[m] = sv[m]; lo[m] = sv[m + 16]; }
    __syncwarp();
    const long long t0 = clock64();
    if (MODE == 5) { tmem_ld32(taddr, sv); }
    for (int it = 0; it < iters; ++it) {
      const uint32_t ta = taddr + 128 * (it & 1);
      if (MODE == 0 || MODE == 2 || MODE == 3 || MODE == 4) {
        tmem_ld32(ta, sv);
        tmem_ld_wait();
      }
      if (MODE == 5) {
        tmem_ld_wait();
        uint32_t cur[32];
#pragma unroll
        for (int m = 0; m < 32; ++m) cur[m] = sv[m];
        tmem_ld32(taddr + 128 * ((it + 1) & 1), sv);
        chunk_math<3>(cur, hi, lo);
      }
      if (MODE == 3 || MODE == 4) chunk_math<MODE>(sv, hi, lo);
      if (MODE == 6) {
#pragma unroll
        for (int m = 0; m < 32; ++m) sv[m] += 1;
        chunk_math<3>(sv, hi, lo);
#pragma unroll
        for (int m = 0; m < 16; ++m) acc ^= hi[m] ^ lo[m];
      }
      if (MODE == 0) {
#pragma unroll
        for (int m = 0; m < 32; ++m) acc ^= sv[m];
      }
      if (MODE == 1 || MODE == 2 || MODE == 3 || MODE == 4 || MODE == 5) {
        tmem_st16(ta, hi);
        tmem_st16(ta + 16, lo);
        tmem_st_wait();
      }
    }
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 16 + (warp - 4)] = t1 - t0;
    if (acc == 0x12345678u) *sink = 1;
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    fence_after_sync();
    tmem_dealloc<512>(tb);
  }
}

template <int MODE, int NW>
void run(const char* name, long long* out, long long* h, int* sink) {
  const int iters = 4000;
  tm<MODE, NW><<<148, 640>>>(out, iters, sink);
  tm<MODE, NW><<<148, 640>>>(out, iters, sink);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, out, 148 * 16 * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  int cnt = 0;
  for (int b = 0; b < 148; ++b)
    for (int w = 0; w < NW; ++w) { avg += h[b * 16 + w]; ++cnt; }
  avg /= cnt;
  const double per = avg / iters;
  printf("%-46s warps %2d: %7.1f clk/chunk/warp  %6.2f elem/clk/SM  (%s)\n", name, NW, per, NW * 1024.0 / per,
         cudaGetErrorString(e));
}

int main() {
  long long *out, h[148 * 16];
  int* sink;
  cudaMalloc(&out, sizeof(h));
  cudaMalloc(&sink, 4);
  run<0, 16>("ld32 + wait", out, h, sink);
  run<1, 16>("st16 x2 + wait", out, h, sink);
  run<2, 16>("ld + st (K1 traffic)", out, h, sink);
  run<2, 8>("ld + st (K1 traffic)", out, h, sink);
  run<2, 4>("ld + st (K1 traffic)", out, h, sink);
  run<3, 16>("ld + ex2 + round split + st", out, h, sink);
  run<3, 8>("ld + ex2 + round split + st", out, h, sink);
  run<4, 16>("ld + ex2 + trunc split + st", out, h, sink);
  run<5, 16>("pipelined ld + ex2 + round split + st", out, h, sink);
  run<6, 16>("ex2 + round split (registers)", out, h, sink);
  run<6, 8>("ex2 + round split (registers)", out, h, sink);
  return 0;
}
