// common.cuh -- host-side helpers shared by the kernel translation units:
// TMA tensor-map encoding through the driver entry point, launch checking,
// and the SM count.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <utility>

namespace fsvd {

struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

#define FSVD_CUDA_CHECK(expr)                                                          \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      throw ::fsvd::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_));     \
  } while (0)

// Counts every kernel this library launches (fsvd_kernel_launch_count).
void note_launch();
void check_launch(const char* what);

int num_sms();

// FSVD_NO_PDL=1 turns programmatic dependent launch off (developer traces).
bool pdl_enabled();
// Launch with programmatic stream serialization (see ptx::pdl_wait).
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  FSVD_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

enum class TmaSwizzle { None, B32, B64, B128 };

// Row-major 2-D tensor [rows, cols] with leading dimension ld (elements);
// the box is [box_rows, box_cols] (box_cols * elem_bytes <= swizzle width).
CUtensorMap make_tmap_2d(const void* base, CUtensorMapDataType dtype, int elem_bytes,
                         uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows,
                         uint32_t box_cols, TmaSwizzle swz);

inline CUtensorMap tmap_bf16(const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                             uint32_t box_rows, uint32_t box_cols, TmaSwizzle swz) {
  return make_tmap_2d(base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rows, cols, ld, box_rows,
                      box_cols, swz);
}

inline TmaSwizzle swizzle_for_row_bytes(uint32_t row_bytes) {
  return row_bytes >= 128 ? TmaSwizzle::B128 : row_bytes == 64 ? TmaSwizzle::B64
                                                                : TmaSwizzle::B32;
}

}  // namespace fsvd
