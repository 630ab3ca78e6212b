// ubench_smsp.cu -- does a tcgen05.mma issuer blocked on a full tensor queue slow down the
// ex2-bound epilogue warps that share its SM sub-partition?  16 "epilogue" warps (ex2 + fp16 split
// on registers, TMEM lane quarter = warp % 4) run for a fixed time while warp 1 issues TS MMAs
// (M=128 N=64 K=16) either (0) not at all, (1) back to back (queue always full), (2) in batches of
// 8 with a commit + mbarrier wait per batch (never more than ~8 in flight), (3) batches of 4.
// Prints epilogue chunks completed per warp, grouped by SMSP.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2006_11267_b200/csrc -o /tmp/ubs scripts/ubench_smsp.cu
#include <cstdio>

#include "tc_util.cuh"

using namespace ciq::tc;

template <int MODE>
__global__ void __launch_bounds__(640, 1) k(long long* out, int* mma_count, long long dur) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase_s;
  __shared__ volatile int stop;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < 16384 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); stop = 0; }
  if (warp == 0) tmem_alloc<512>(&tbase_s);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tb = tbase_s;
  const long long t0 = clock64();
  __shared__ uint64_t rb[4];
  if (threadIdx.x == 32) { for (int i = 0; i < 4; ++i) mbar_init(&rb[i], 1); fence_mbar_init(); }
  __syncwarp();
  if (MODE == 6 && warp == 2) {  // second issuer on SMSP 2, back to back
    constexpr uint32_t idesc = idesc_f16(128, 64, 0, 1);
    const uint64_t dv = smem_desc(smem_u32(smem), 8 * 128, 128);
    while (clock64() - t0 < dur) {
#pragma unroll
      for (int i = 0; i < 8; ++i) mma_ts_warp(tb + 384, tb + 256 + 8 * (i & 7), dv, idesc, 1u);
    }
  }
  if (warp == 1) {
    constexpr uint32_t idesc = idesc_f16(128, 64, 0, 1);
    const uint64_t dv = smem_desc(smem_u32(smem), 8 * 128, 128);
    int n = 0;
    uint32_t ph = 0;
    while (clock64() - t0 < dur) {
      if (MODE == 4 || MODE == 5 || MODE == 7) {  // batches of B, at most D batches in flight
        constexpr int B = MODE == 4 ? 8 : (MODE == 5 ? 6 : 12);
        constexpr int D = MODE == 5 ? 3 : 2;
        const int i = n / B;
        if (i >= D) mbar_wait(&rb[(i - D) & 3], ((i - D) >> 2) & 1);
#pragma unroll
        for (int m = 0; m < B; ++m) mma_ts_warp(tb + 448, tb + 256 + 8 * (m & 7), dv, idesc, 1u);
        mma_commit_warp(&rb[i & 3]);
        n += B;
      } else if (MODE == 1 || MODE == 6) {
#pragma unroll
        for (int i = 0; i < 8; ++i) mma_ts_warp(tb + 448, tb + 256 + 8 * (i & 7), dv, idesc, 1u);
        n += 8;
      } else if (MODE == 2 || MODE == 3) {
        constexpr int B = MODE == 2 ? 8 : 4;
#pragma unroll
        for (int i = 0; i < B; ++i) mma_ts_warp(tb + 448, tb + 256 + 8 * (i & 7), dv, idesc, 1u);
        mma_commit_warp(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
        n += B;
      }
    }
    if (lane == 0) mma_count[blockIdx.x] = n;
    mma_commit_warp(&bar);
    mbar_wait(&bar, ph);
    stop = 1;
  } else if (warp >= 4) {
    uint32_t acc = 0;
    float s0 = -0.01f * lane;
    long long cnt = 0;
    while (clock64() - t0 < dur) {
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        const float k0 = ex2_approx(s0 - c * 1e-3f), k1 = ex2_approx(s0 - (c + 1) * 1e-3f);
        const uint32_t h = pack_half2(k0, k1);
        const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&h));
        hi[c / 2] = h;
        lo[c / 2] = pack_half2(k0 - hf.x, k1 - hf.y);
      }
#pragma unroll
      for (int m = 0; m < 16; ++m) acc ^= hi[m] ^ lo[m];
      s0 += 1e-6f;
      ++cnt;
    }
    if (lane == 0) out[blockIdx.x * 16 + warp - 4] = cnt + (acc == 0x12345678u);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) { fence_after_sync(); tmem_dealloc<512>(tb); }
}

template <int MODE>
void run(const char* name) {
  long long* out;
  int* mc;
  cudaMalloc(&out, 148 * 16 * 8);
  cudaMalloc(&mc, 148 * 4);
  const int smem = 16384 + 1024;
  const long long dur = 2000000;
  k<MODE><<<148, 640, smem>>>(out, mc, dur);
  k<MODE><<<148, 640, smem>>>(out, mc, dur);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148 * 16];
  int m[148];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  cudaMemcpy(m, mc, sizeof(m), cudaMemcpyDeviceToHost);
  double smsp[4] = {0, 0, 0, 0}, mm = 0;
  for (int b = 0; b < 148; ++b) {
    for (int w = 0; w < 16; ++w) smsp[(w + 4) % 4] += h[b * 16 + w];
    mm += m[b];
  }
  printf("%-40s epilogue elem/clk per SMSP: %.3f %.3f %.3f %.3f   MMA/clk*32: %.2f  (%s)\n", name,
         smsp[0] * 1024 / 148 / dur, smsp[1] * 1024 / 148 / dur, smsp[2] * 1024 / 148 / dur,
         smsp[3] * 1024 / 148 / dur, mm / 148 / dur * 32, cudaGetErrorString(e));
}

int main() {
  run<0>("no MMAs");
  run<1>("MMAs back to back (queue full)");
  run<2>("MMAs in batches of 8 + commit/wait");
  run<3>("MMAs in batches of 4 + commit/wait");
  run<4>("batches of 8, 2 in flight");
  run<5>("batches of 6, 3 in flight");
  run<7>("batches of 12, 2 in flight");
  run<6>("two issuers (SMSP 1, 2) back to back");
  return 0;
}
