#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 2) k(double* p) { extern __shared__ double s[]; __shared__ int x[64]; x[threadIdx.x % 64] = 1; s[threadIdx.x] = p[threadIdx.x] + x[3]; __syncthreads(); p[threadIdx.x] = s[255 - threadIdx.x]; }
int main() {
  int v; cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0); printf("smem/SM %d\n", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0); printf("smem/block optin %d\n", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrReservedSharedMemoryPerBlock, 0); printf("reserved/block %d\n", v);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  for (int co = -1; co <= 100; co += 101) {
    if (co == 100) cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    for (int b = 96 * 1024; b <= 118 * 1024; b += 2048) {
      int n; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, 256, b); printf("carveout %d dyn %d -> %d blocks\n", co, b, n);
    }
  }
}
