// TMA (cp.async.bulk.tensor) + mbarrier helpers shared by the fused kernels, and the
// host-side encoder of 2-D tile descriptors over element-major [rows][Kp] fp64 arrays.
#pragma once
#include <utility>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace sdrt {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
// 2-D tile {E columns (elements), box rows} at (x = first element, y = first row)
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// the same with an L2 evict-first policy: for tiles read once and dead afterwards (R_int)
__device__ __forceinline__ void tma_load_2d_ef(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], "
      "[%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// rows per TMA box: the largest divisor of the row count that is <= 256
__host__ __device__ constexpr int tma_box_rows(int rows) {
  int b = rows < 256 ? rows : 256;
  while (rows % b) --b;
  return b;
}

// whole tile [ROWS][E] of one array, issued by one thread, completing on bar
template <int ROWS, int E, bool EF = false>
__device__ __forceinline__ void tma_tile(double* dst, const CUtensorMap* map, int64_t e0, uint64_t* bar) {
  constexpr int BR = tma_box_rows(ROWS);
#pragma unroll
  for (int r = 0; r < ROWS; r += BR) {
    if constexpr (EF) tma_load_2d_ef(dst + r * E, map, (int)e0, r, bar);
    else tma_load_2d(dst + r * E, map, (int)e0, r, bar);
  }
}

// host: descriptor of a [rows][Kp] fp64 array, boxes of E x tma_box_rows(rows)
inline void encode_tile_map(CUtensorMap* map, const void* ptr, int rows, int E, int64_t Kp) {
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      throw std::runtime_error("CUDA: cuTensorMapEncodeTiled unavailable");
    enc = (EncodeFn)fn;
  }
  cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)Kp * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)E, (cuuint32_t)tma_box_rows(rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("CUDA: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

// small per-context cache: descriptor of array ptr
template <class Cache>
inline const CUtensorMap& cached_tile_map(Cache* t, const void* ptr) {
  for (int i = 0; i < 8; ++i)
    if (t->ptr[i] == ptr) return t->map[i];
  const int i = t->next;
  t->next = (t->next + 1) % 8;
  encode_tile_map(&t->map[i], ptr, t->rows, t->E, t->Kp);
  t->ptr[i] = ptr;
  return t->map[i];
}


// ---- programmatic dependent launch (SDRT_PDL): a stage kernel is launched with
// programmatic stream serialization, so its CTAs are scheduled while the previous
// kernel drains; pdl_wait() (first statement of the kernel) blocks until that kernel has
// completed and its writes are visible.  Kernels without pdl_wait are launched normally.
#ifndef SDRT_PDL
#define SDRT_PDL 1
#endif
__device__ __forceinline__ void pdl_wait() {
#if SDRT_PDL
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

#define CUDA_LAUNCH_OK(x)                                                                     \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                     Args&&... args) {
#if SDRT_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
#else
  k<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
  return cudaGetLastError();
#endif
}

}  // namespace sdrt
