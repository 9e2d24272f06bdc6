// Microbenchmark: fp64 tensor-core (mma.sync m8n8k4 f64) throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void mixed_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2], f[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = f[t] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
#pragma unroll
      for (int u = 0; u < 4; ++u) f[t] = fma(f[t], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + f[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 8 * 256);
  int iters = 4096;
  for (int warps = 4; warps <= 16; warps *= 2) {
    int blocks = 148 * 4;
    dmma_loop<<<blocks, warps * 32>>>(out, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dmma_loop<<<blocks, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * blocks * warps;  // per warp per mma: 8x8x4 FMA
    printf("warps/block %d: %.2f TFLOP/s fp64 mma\n", warps, flops / ms / 1e9);
  }
  {
    int blocks = 148 * 4, warps = 8;
    mixed_loop<<<blocks, warps * 32>>>(out, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mixed_loop<<<blocks, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fm = 2.0 * 256 * 8 * (double)iters * blocks * warps;
    double fv = 2.0 * 32 * 8 * 4 * (double)iters * blocks * warps;
    printf("mixed: mma %.2f + dfma %.2f = %.2f TFLOP/s\n", fm / ms / 1e9, fv / ms / 1e9,
           (fm + fv) / ms / 1e9);
  }
  return 0;
}
