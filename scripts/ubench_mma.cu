// ubench_mma.cu -- issue rate of tcgen05.mma kind::f16 shapes/operand placements used by K1
// (standalone experiment; numerics irrelevant, operands are zero):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2006_11267_b200/csrc \
//        -o scripts/_ubench_mma scripts/ubench_mma.cu && scripts/_ubench_mma
#include <cstdio>

#include "tc_util.cuh"

using namespace ciq::tc;

__device__ __forceinline__ uint64_t desc_sw(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = smem_desc(saddr, lbo, sbo);
  d |= (uint64_t)layout << 61;
  return d;
}

// MODE: 0 TS N=64 B MN-major (K1's KV)   1 SS N=64 B MN-major   2 TS N=64 B K-major
//       3 TS N=128 B MN-major            4 TS N=256 B MN-major  5 SS N=64 A,B K-major
//       6 SS N=128 K-major (K1's S)       7 SS N=64 K-major SWIZZLE_128B A and B
//       8 TS N=64 B K-major SWIZZLE_128B
template <int MODE>
__global__ void __launch_bounds__(128, 1) mma_rate(long long* out, int rounds) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tb = tbase_s;
  if (warp == 0) {
    constexpr uint32_t N = (MODE == 3 || MODE == 6) ? 128 : (MODE == 4 ? 256 : 64);
    constexpr bool b_mn = (MODE == 0 || MODE == 1 || MODE == 3 || MODE == 4);
    constexpr uint32_t idesc = idesc_f16(128, N, 0, b_mn ? 1 : 0);
    const uint32_t a_s = smem_u32(smem);              // A 128 x 16 (4 KB) per K step
    const uint32_t b_s = smem_u32(smem + 32 * 1024);  // B up to 256 x 16
    const long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
#pragma unroll
      for (int k = 0; k < 24; ++k) {
        const uint32_t d = (N == 256) ? tb : tb + 128 * (k & 1);  // two accumulators (one at N = 256)
        if (MODE == 0 || MODE == 3 || MODE == 4) {
          mma_ts_warp(d, tb + 384 + 8 * (k & 7), smem_desc(b_s, (N / 8) * 128, 128), idesc, 1u);
        } else if (MODE == 2) {
          mma_ts_warp(d, tb + 384 + 8 * (k & 7), smem_desc(b_s, 128, 256), idesc, 1u);
        } else if (MODE == 8) {
          mma_ts_warp(d, tb + 384 + 8 * (k & 7), desc_sw(b_s + 32 * (k & 3), 16, 1024, 2), idesc, 1u);
        } else if (MODE == 1) {
          mma_ss_warp(d, smem_desc(a_s, 128, 256), smem_desc(b_s, (N / 8) * 128, 128), idesc, 1u);
        } else if (MODE == 5 || MODE == 6) {
          mma_ss_warp(d, smem_desc(a_s, 128, 256), smem_desc(b_s, 128, 256), idesc, 1u);
        } else if (MODE == 7) {
          mma_ss_warp(d, desc_sw(a_s + 32 * (k & 3), 16, 1024, 2), desc_sw(b_s + 32 * (k & 3), 16, 1024, 2), idesc, 1u);
        }
      }
    }
    mma_commit_warp(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    fence_after_sync();
    tmem_dealloc<512>(tb);
  }
}

template <int MODE>
void run(const char* name, long long* out, long long* h) {
  const int rounds = 2000, smem = 96 * 1024 + 1024;
  cudaFuncSetAttribute(mma_rate<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_rate<MODE><<<148, 128, smem>>>(out, rounds);
  mma_rate<MODE><<<148, 128, smem>>>(out, rounds);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, out, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  printf("%-40s %7.1f clk/MMA  (%s)\n", name, avg / (rounds * 24.0), cudaGetErrorString(e));
}

int main() {
  long long *out, h[148];
  cudaMalloc(&out, 148 * sizeof(long long));
  run<0>("TS N=64 B MN-major (K1 KV)", out, h);
  run<1>("SS N=64 B MN-major", out, h);
  run<2>("TS N=64 B K-major", out, h);
  run<3>("TS N=128 B MN-major", out, h);
  run<4>("TS N=256 B MN-major", out, h);
  run<5>("SS N=64 K-major", out, h);
  run<6>("SS N=128 K-major (K1 S)", out, h);
  run<7>("SS N=64 K-major SW128", out, h);
  run<8>("TS N=64 B K-major SW128", out, h);
  return 0;
}
