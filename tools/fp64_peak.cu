// FP64 peak microbenchmarks for the roofline denominator ("P64 must be
// measured on the box").  Full-machine grids (148 SMs x 2048 threads), CUDA events,
// best of 10 after 3 warm-ups.
//   dfma : 8 independent DFMA chains per thread, register operands
//   dmma : mma.sync m8n8k4 f64 (DMMA), 4 independent accumulators per warp
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

__global__ void dmma_loop(double* out, double a0, int iters) {
  double a = a0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
  double c[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

template <class F>
static float best_ms(F launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) launch();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 512, blocks = sms * 4, iters = 1 << 16;
  const float t1 = best_ms([&] { dfma_loop<<<blocks, threads>>>(out, 0.999999, 1e-7, iters); });
  const double f1 = 2.0 * 8.0 * iters * (double)threads * blocks;
  const int it2 = 1 << 14;
  const float t2 = best_ms([&] { dmma_loop<<<blocks, threads>>>(out, 0.5, it2); });
  const double f2 = 2.0 * 256.0 * 4.0 * it2 * (double)(threads / 32) * blocks;
  printf("{\"fp64_dfma_tflops\": %.3f, \"fp64_dmma_tflops\": %.3f, \"sms\": %d, \"clock_mhz_attr\": %.0f, "
         "\"dfma_per_clk_per_sm_at_attr_clock\": %.2f, \"dmma_fma_per_clk_per_sm_at_attr_clock\": %.2f}\n",
         f1 / (t1 * 1e-3) / 1e12, f2 / (t2 * 1e-3) / 1e12, sms, clk / 1e3,
         f1 / 2 / (t1 * 1e-3) / sms / (clk * 1e3), f2 / 2 / (t2 * 1e-3) / sms / (clk * 1e3));
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
