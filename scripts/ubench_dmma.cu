// DMMA (mma.sync m8n8k4 f64) vs DFMA throughput on one B200 (microbenchmark for the fp64 route's
// M MVM).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 ubench_dmma.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma_k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c[16] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) c[u] = fma(a, b, c[u]);
  }
  double s = 0;
  for (int u = 0; u < 16; ++u) s += c[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    const int iters = 20000, blocks = 148 * 2;
    dmma_k<<<blocks, 32 * warps>>>(out, 10);
    cudaEventRecord(e0);
    dmma_k<<<blocks, 32 * warps>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * warps * blocks;
    printf("DMMA m8n8k4: %d warps/CTA x %d CTAs: %.2f TFLOP/s\n", warps, blocks, flops / ms / 1e9);
    dfma_k<<<blocks, 32 * warps>>>(out, 10);
    cudaEventRecord(e0);
    dfma_k<<<blocks, 32 * warps>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * 32.0 * iters * warps * blocks;
    printf("DFMA:        %d warps/CTA x %d CTAs: %.2f TFLOP/s\n", warps, blocks, flops / ms / 1e9);
  }
  return 0;
}
