// common.cu -- TMA descriptor encoding, launch accounting, device queries,
// dynamic-schedule counters.
#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

namespace fsvd {

namespace {
std::atomic<uint64_t> g_launches{0};

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled is unavailable (driver too old?)");
  return fn;
}
}  // namespace

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(); }

void check_launch(const char* what) {
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FSVD_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    FSVD_CUDA_CHECK(cudaGetDevice(&dev));
    FSVD_CUDA_CHECK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  }
  return n;
}

CUtensorMap make_tmap_2d(const void* base, CUtensorMapDataType dtype, int elem_bytes,
                         uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows,
                         uint32_t box_cols, TmaSwizzle swz) {
  CUtensorMap map;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * static_cast<uint64_t>(elem_bytes)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle s = swz == TmaSwizzle::B128  ? CU_TENSOR_MAP_SWIZZLE_128B
                         : swz == TmaSwizzle::B64 ? CU_TENSOR_MAP_SWIZZLE_64B
                         : swz == TmaSwizzle::B32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                  : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = encode_fn()(&map, dtype, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, s, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) +
                    ") rows=" + std::to_string(rows) + " cols=" + std::to_string(cols) +
                    " ld=" + std::to_string(ld) + " box=" + std::to_string(box_rows) + "x" +
                    std::to_string(box_cols));
  return map;
}

CUtensorMap make_tmap_3d(const void* base, CUtensorMapDataType dtype, int elem_bytes,
                         uint64_t d0, uint64_t d1, uint64_t d2, uint64_t ld1, uint64_t ld2,
                         uint32_t box0, uint32_t box1, TmaSwizzle swz) {
  CUtensorMap map;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {ld1 * static_cast<uint64_t>(elem_bytes),
                           ld2 * static_cast<uint64_t>(elem_bytes)};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUtensorMapSwizzle s = swz == TmaSwizzle::B128  ? CU_TENSOR_MAP_SWIZZLE_128B
                         : swz == TmaSwizzle::B64 ? CU_TENSOR_MAP_SWIZZLE_64B
                         : swz == TmaSwizzle::B32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                  : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = encode_fn()(&map, dtype, 3, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, s, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw CudaError("cuTensorMapEncodeTiled (3d) failed (" + std::to_string(static_cast<int>(r)) +
                    ") dims=" + std::to_string(d0) + "x" + std::to_string(d1) + "x" +
                    std::to_string(d2));
  return map;
}

// Per-(device, stream) work counters of the dynamic tile / item schedules
// ([next, CTAs done]; zero between launches: the last CTA out resets them).
// One slot serves every kernel on a stream: a kernel touches it only after
// griddepcontrol.wait, i.e. after the previous kernel has finished.
// Allocated on first use; null (static schedule) while the stream is being
// captured, or past 64 streams.
int* sched_counter(cudaStream_t s) {
  // a captured graph may be replayed on another stream next to eager work on
  // this one: captured launches keep the static schedule
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  FSVD_CUDA_CHECK(cudaStreamIsCapturing(s, &cap));
  if (cap != cudaStreamCaptureStatusNone) return nullptr;
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, int*> slots;
  static std::map<int, std::pair<int*, int>> pools;
  int dev = 0;
  FSVD_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  const auto f = slots.find({dev, s});
  if (f != slots.end()) return f->second;
  auto& pool = pools[dev];
  constexpr int kSlots = 64, kStride = 32;  // 128 B apart
  if (pool.first == nullptr) {
    FSVD_CUDA_CHECK(cudaMalloc(&pool.first, kSlots * kStride * sizeof(int)));
    FSVD_CUDA_CHECK(cudaMemset(pool.first, 0, kSlots * kStride * sizeof(int)));
    FSVD_CUDA_CHECK(cudaDeviceSynchronize());
  }
  if (pool.second >= kSlots) return nullptr;
  int* p = pool.first + kStride * pool.second++;
  slots[{dev, s}] = p;
  return p;
}

bool sched_enabled(const char* env) {
  const char* e = getenv(env);  // developer A/B switches: =0 keeps the static schedule
  return !(e && e[0] == '0');
}

}  // namespace fsvd
