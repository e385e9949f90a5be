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
// dynamic-schedule counters for kernels launched on stream s (see common.cu)
int* sched_counter(cudaStream_t s);
bool sched_enabled(const char* env);
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

#ifdef FSVD_TRACE
// per-CTA timeline of the last launch of a kernel in this translation unit
// (ptx::globaltimer_ns): [cta][entry, after pdl_wait, exit (ns), clock64 after
// pdl_wait, clock64 at exit, smid, -, -]; the clock64 / ns ratio is the SM
// clock the CTA ran at
#define FSVD_CTA_TIMES(tu)                                                              \
  namespace {                                                                          \
  __device__ unsigned long long g_cta_t[4096 * 8];                                     \
  }                                                                                    \
  extern "C" __attribute__((visibility("default"))) int fsvd_debug_cta_times_##tu(      \
      unsigned long long* host, int n) {                                                \
    return static_cast<int>(cudaMemcpyFromSymbol(host, g_cta_t, sizeof(unsigned long long) * n)); \
  }
#define CTA_T(slot)                                                                     \
  do {                                                                                  \
    if (threadIdx.x == 0 && blockIdx.x < 4096) {                                        \
      unsigned long long* e_ = g_cta_t + blockIdx.x * 8;                                \
      e_[(slot)] = ::fsvd::ptx::globaltimer_ns();                                       \
      if ((slot) == 0) e_[5] = ::fsvd::ptx::smid();                                     \
      if ((slot) >= 1) e_[2 + (slot)] = clock64();                                      \
    }                                                                                   \
  } while (0)
#else
#define FSVD_CTA_TIMES(tu)
#define CTA_T(slot) do { } while (0)
#endif

enum class TmaSwizzle { None, B32, B64, B128 };

// Row-major 2-D tensor [rows, cols] with leading dimension ld (elements);
// the box is [box_rows, box_cols] (box_cols * elem_bytes <= swizzle width).
CUtensorMap make_tmap_2d(const void* base, CUtensorMapDataType dtype, int elem_bytes,
                         uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows,
                         uint32_t box_cols, TmaSwizzle swz);

// [d2][d1][d0] elements, d0 contiguous, ld1 / ld2 the strides of d1 / d2 in
// elements; box {box0, box1, 1}
CUtensorMap make_tmap_3d(const void* base, CUtensorMapDataType dtype, int elem_bytes,
                         uint64_t d0, uint64_t d1, uint64_t d2, uint64_t ld1, uint64_t ld2,
                         uint32_t box0, uint32_t box1, TmaSwizzle swz);
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
