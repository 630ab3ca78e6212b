// ubench_mma_pair.cu -- issue / execution rate of back-to-back TS MMAs (A from TMEM, B MN-major
// from smem, kind::f16) on one CTA (cta_group::1, M = 128) vs a CTA pair (cta_group::2, M = 256),
// for N = 64 / 128: is K1's pair kernel (mvm_tc3.cu) bound by MMA issue?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2006_11267_b200/csrc \
//        -o scripts/_ubench_mma_pair scripts/ubench_mma_pair.cu && scripts/_ubench_mma_pair
#include <cstdio>

#include "tc_util.cuh"

using namespace ciq::tc;

__device__ __forceinline__ bool cute_elect() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t@p mov.u32 %0, 1;\n\t}" : "+r"(pred));
  return pred != 0;
}

template <int CG, int N>
__device__ __forceinline__ void mma_ts_g(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc) {
  if (CG == 1)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, 1, 1;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc)
                 : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, 1, 1;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc)
                 : "memory");
}

template <int CG, int N>
__global__ void __launch_bounds__(128, 1) rate(long long* out, int rounds) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    if (CG == 1) {
      tmem_alloc<512>(&tbase_s);
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase_s)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  fence_before_sync();
  if (CG == 2) cluster_sync(); else __syncthreads();
  fence_after_sync();
  const uint32_t tb = tbase_s;
  constexpr int NL = N / CG;   // B columns held by this CTA
  if (warp == 1 && rank == 0) {
    constexpr uint32_t idesc = idesc_f16(128 * CG, N, 0, 1);
    const uint32_t kb = tb, o = tb + 256;
    const uint64_t dv = smem_desc(smem_u32(smem), (NL / 8) * 128, 128);
    const long long t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
#pragma unroll
      for (int kk = 0; kk < 24; ++kk) {
        const uint32_t a = kb + 8 * (kk % 8);
        if (cute_elect()) mma_ts_g<CG, N>(o, a, dv + (uint64_t)(((kk % 4) * 2 * NL * 16) >> 4), idesc);
        __syncwarp();
      }
    }
    const long long t1 = clock64();
    if (cute_elect()) {
      if (CG == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      else
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                         smem_u32(&bar)),
                     "h"((uint16_t)3)
                     : "memory");
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    const long long t2 = clock64();
    if (threadIdx.x == 32 && blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  if (CG == 2 && warp == 1 && rank == 1) mbar_wait(&bar, 0);   // the multicast commit arrives here too
  fence_before_sync();
  if (CG == 2) cluster_sync(); else __syncthreads();
  if (warp == 0) {
    fence_after_sync();
    if (CG == 1) tmem_dealloc<512>(tb);
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
  }
}

template <int CG, int N>
void run(const char* name, int rounds) {
  long long* d;
  cudaMalloc(&d, 16);
  auto k = rate<CG, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(CG);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 80 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  for (int w = 0; w < 2; ++w) cudaLaunchKernelEx(&cfg, k, d, rounds);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-36s issue %6.1f clk/MMA   complete %6.1f clk/MMA   (%s)\n", name, h[0] / (rounds * 24.0),
         h[1] / (rounds * 24.0), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<1, 64>("cta_group::1 M=128 N=64 K=16", 2000);
  run<2, 64>("cta_group::2 M=256 N=64 K=16", 2000);
  run<1, 128>("cta_group::1 M=128 N=128 K=16", 2000);
  run<2, 128>("cta_group::2 M=256 N=128 K=16", 2000);
  return 0;
}
