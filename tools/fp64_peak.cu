// FP64 peak microbenchmark for the roofline denominator ("P64 must be
// measured on the box").  DFMA throughput with 8 independent chains per thread and
// register operands, full-machine grid (148 SMs x 2048 threads), CUDA events.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, double a, double b, int iters) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 512, blocks = sms * 4, iters = 1 << 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7, iters);
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8.0 * iters * (double)threads * blocks;
  printf("{\"fp64_dfma_tflops\": %.3f, \"sms\": %d, \"clock_mhz_attr\": %.0f, \"ms\": %.3f, "
         "\"dfma_per_clk_per_sm_at_attr_clock\": %.2f}\n",
         flops / (best * 1e-3) / 1e12, sms, clk / 1e3, best,
         flops / 2 / (best * 1e-3) / sms / (clk * 1e3));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
