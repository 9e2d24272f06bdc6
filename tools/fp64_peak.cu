// FP64 DFMA throughput microbenchmark: measures the FP64-pipe peak used as the
// roofline denominator for the SOE scan kernels (not in MEASURED_PEAKS.json).
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void sincos_loop(double* out, int iters, double step) {
  double th = threadIdx.x * 1e-3 + blockIdx.x;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    double s, c;
    sincos(th, &s, &c);
    acc += s * c;
    th += step;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void exp_loop(double* out, int iters, double step) {
  double x = -(threadIdx.x * 1e-4);
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += exp(x);
    x -= step;
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void erfc_loop(double* out, int iters, double step) {
  double x = (threadIdx.x * 1e-4);
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += erfc(x);
    x += step;
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int dev = 0;
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("device %s sms %d clock_khz %d regs/sm %d smem/sm %zu\n", p.name, sms, clk_khz,
         p.regsPerMultiprocessor, p.sharedMemPerMultiprocessor);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int tpb : {256, 512, 1024}) {
      int blocks = sms * (2048 / tpb);
      dfma_loop<8><<<blocks, tpb>>>(out, 100, 1.0000001, 1e-7);
      cudaEventRecord(e0);
      dfma_loop<8><<<blocks, tpb>>>(out, iters, 1.0000001, 1e-7);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * (double)iters * blocks * tpb;
      printf("dfma tpb=%d blocks=%d: %.3f ms  %.2f TFLOP/s  (%.1f DFMA/clk/SM at nominal clock)\n", tpb, blocks, ms,
             flops / ms / 1e9, flops / 2 / (ms * 1e-3) / sms / (clk_khz * 1e3));
    }
  }
  {
    int blocks = sms * 8, tpb = 256;
    int it = 4000;
    sincos_loop<<<blocks, tpb>>>(out, 10, 0.01);
    cudaEventRecord(e0);
    sincos_loop<<<blocks, tpb>>>(out, it, 0.0137);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("sincos: %.3f ms  %.3f Gsincos/s\n", ms, (double)it * blocks * tpb / ms / 1e6);
    exp_loop<<<blocks, tpb>>>(out, 10, 0.01);
    cudaEventRecord(e0);
    exp_loop<<<blocks, tpb>>>(out, it, 1e-4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("exp: %.3f ms  %.3f Gexp/s\n", ms, (double)it * blocks * tpb / ms / 1e6);
    erfc_loop<<<blocks, tpb>>>(out, 10, 0.01);
    cudaEventRecord(e0);
    erfc_loop<<<blocks, tpb>>>(out, it, 1e-4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("erfc: %.3f ms  %.3f Gerfc/s\n", ms, (double)it * blocks * tpb / ms / 1e6);
  }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
