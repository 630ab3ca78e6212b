// ubench_queue.cu -- depth of the tcgen05.mma issue queue and the issue-side cost of
// tcgen05.commit / mbarrier try_wait (standalone experiment for K1's MMA warp):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2006_11267_b200/csrc \
//        -o scripts/_ubench_queue scripts/ubench_queue.cu && scripts/_ubench_queue
#include <cstdio>

#include "tc_util.cuh"

using namespace ciq::tc;

// out[0] = clk to issue NB MMAs into an idle pipe; out[1] = clk until they complete;
// out[2] = clk of 16 commits (no MMAs in flight); out[3] = clk of 16 try_waits on a completed phase
template <int NB>
__global__ void __launch_bounds__(128, 1) q_depth(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bars[16], done_bar;
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 32 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&done_bar, 1);
    for (int i = 0; i < 16; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tb = tbase_s;
  if (warp == 0) {
    constexpr uint32_t idesc = idesc_f16(128, 64, 0, 1);
    const uint64_t dv = smem_desc(smem_u32(smem), 8 * 128, 128);
    long long t0 = clock64();
#pragma unroll
    for (int k = 0; k < NB; ++k) mma_ts_warp(tb + 128 * (k & 1), tb + 384 + 8 * (k & 7), dv, idesc, 1u);
    long long t1 = clock64();
    mma_commit_warp(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    // commits with nothing in flight
    long long t3 = clock64();
#pragma unroll
    for (int i = 0; i < 16; ++i) mma_commit_warp(&bars[i]);
    long long t4 = clock64();
    for (int i = 0; i < 16; ++i) mbar_wait(&bars[i], 0);  // all complete by now (or soon)
    long long t5 = clock64();
#pragma unroll
    for (int i = 0; i < 16; ++i) mbar_wait(&bars[i], 0);  // completed phase: pure try_wait cost
    long long t6 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
      out[2] = t4 - t3;
      out[3] = t6 - t5;
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    fence_after_sync();
    tmem_dealloc<512>(tb);
  }
}

template <int NB>
void run(long long* out, long long* h) {
  const int smem = 33 * 1024;
  cudaFuncSetAttribute(q_depth<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  q_depth<NB><<<1, 128, smem>>>(out);
  q_depth<NB><<<1, 128, smem>>>(out);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, out, 4 * sizeof(long long), cudaMemcpyDeviceToHost);
  printf("NB=%3d  issue %6lld clk (%5.1f/MMA)  complete %6lld clk  16 commits %5lld clk  16 done try_waits %5lld clk (%s)\n",
         NB, h[0], (double)h[0] / NB, h[1], h[2], h[3], cudaGetErrorString(e));
}

int main() {
  long long *out, h[4];
  cudaMalloc(&out, 4 * sizeof(long long));
  run<1>(out, h);
  run<2>(out, h);
  run<4>(out, h);
  run<8>(out, h);
  run<12>(out, h);
  run<16>(out, h);
  run<24>(out, h);
  run<32>(out, h);
  run<64>(out, h);
  return 0;
}
