// Host-side helpers shared by the C-ABI translation units: error state,
// TMA tensor-map encoding (driver entry point, no libcuda link), launch checks.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "../../include/sparseft_b200.h"

namespace lx {

void set_error(const char* fmt, ...);

#define LX_CHECK_CUDA(expr)                                                          \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      ::lx::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
      return LX_ERR_CUDA;                                                           \
    }                                                                               \
  } while (0)

#define LX_REQUIRE(cond, code, ...)   \
  do {                                \
    if (!(cond)) {                    \
      ::lx::set_error(__VA_ARGS__);   \
      return (code);                  \
    }                                 \
  } while (0)

// 2D bf16 tensor map: dims {inner, outer}, row stride in elements, box {box_inner, box_outer}, 128B swizzle.
int make_tmap_bf16_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
                      uint32_t box_inner, uint32_t box_outer);

// same with an explicit swizzle (CU_TENSOR_MAP_SWIZZLE_*)
int make_tmap_bf16_2d_sw(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
                         uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz);

int num_sms();

// Programmatic dependent launch on (LX_PDL=0 disables): see pdl_wait_trigger in ptx.cuh.
bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);  // errors surface in launch_check
}

inline int launch_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s launch failed: %s", what, cudaGetErrorString(e));
    return LX_ERR_CUDA;
  }
  return LX_OK;
}

}  // namespace lx
