// planes.cu -- split-plane elementwise kernels of the fp32 policy.
//
// The fp32 policy runs the same tcgen05 kernels as bf16 (K1 / K2 / K3 with
// their X3 template flag): every fp32 activation lives in HBM as three bf16
// planes (kernels.cuh: hi, mid, lo; v = hi + mid + lo to fp32 resolution), so
// an MMA operand carries v's full 24-bit significand and each product takes
// six bf16 passes into an fp32 accumulator.  A [T, N] activation occupies
// 6*T*N bytes (hi plane, mid plane, lo plane); fp32 packs on the tensor cores
// have es = 6 for the workspace planner.
//
// This file holds the conversions at the API boundary (fp32 <-> planes) and
// the row kernels between the GEMMs: residual + LayerNorm (encoder.cpp:38-50,
// tensor.cpp:88-102) and the pre-LN residual add, all computing in fp32.
#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace fsvd {
namespace {

__device__ __forceinline__ void split1(float v, bf16& hi, bf16& mid, bf16& lo) {
  hi = __float2bfloat16_rn(v);
  const float r = v - __bfloat162float(hi);
  mid = __float2bfloat16_rn(r);
  lo = __float2bfloat16_rn(r - __bfloat162float(mid));
}
__device__ __forceinline__ void split1(float v, const PlanesOut& y, int64_t i) {
  split1(v, y.hi[i], y.mid[i], y.lo[i]);
}
__device__ __forceinline__ float join1(const Planes& a, int64_t i) {
  return (__bfloat162float(a.hi[i]) + __bfloat162float(a.mid[i])) + __bfloat162float(a.lo[i]);
}

__global__ void k_split_planes(const float* __restrict__ src, PlanesOut y, int64_t n) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    split1(src[i], y, i);
}

__global__ void k_merge_planes(Planes a, float* __restrict__ dst, int64_t n) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = join1(a, i);
}

// y = gamma * ((a + b) - mean) / sqrt(var + eps) + beta per row, fp32, biased
// variance; one warp per row, up to 32*VPL values in registers.  In place
// (y == a or y == b) is allowed: a row is read completely before it is written.
// Rows are stored with `pitch` >= d columns (zero-padded model dimension):
// statistics over the first d, all pitch columns written (gamma = beta = 0 there).
template <int VPL>
__global__ void __launch_bounds__(256)
    k_ln_planes(Planes a, Planes b, const float* __restrict__ gamma,
                const float* __restrict__ beta, float eps, PlanesOut y, int rows, int d,
                int pitch) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const int64_t base = (int64_t)warp * pitch;
  float v[VPL];
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = lane + 32 * i;
    v[i] = 0.0f;
    if (c < pitch) {
      v[i] = join1(a, base + c);
      if (b.hi) v[i] += join1(b, base + c);
      if (c < d) s += v[i];
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float inv_d = 1.0f / static_cast<float>(d);
  const float mean = s * inv_d;
  float q = 0.0f;
#pragma unroll
  for (int i = 0; i < VPL; ++i)
    if (lane + 32 * i < d) {
      const float t = v[i] - mean;
      q = fmaf(t, t, q);
    }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float inv = 1.0f / sqrtf(q * inv_d + eps);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = lane + 32 * i;
    if (c < pitch)
      split1(gamma[c] * ((v[i] - mean) * inv) + beta[c], y, base + c);
  }
}

// Rows wider than the register path: three strided sweeps.
__global__ void __launch_bounds__(256)
    k_ln_planes_wide(Planes a, Planes b, const float* __restrict__ gamma,
                     const float* __restrict__ beta, float eps, PlanesOut y, int rows, int d,
                     int pitch) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const int64_t base = (int64_t)warp * pitch;
  auto val = [&](int c) {
    float t = join1(a, base + c);
    if (b.hi) t += join1(b, base + c);
    return t;
  };
  float s = 0.0f;
  for (int c = lane; c < d; c += 32) s += val(c);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / static_cast<float>(d);
  float q = 0.0f;
  for (int c = lane; c < d; c += 32) {
    const float t = val(c) - mean;
    q = fmaf(t, t, q);
  }
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float inv = 1.0f / sqrtf(q / static_cast<float>(d) + eps);
  // in place is not allowed here (a later value of the row is re-read)
  for (int c = lane; c < pitch; c += 32)
    split1(gamma[c] * ((val(c) - mean) * inv) + beta[c], y, base + c);
}

__global__ void k_add_planes(Planes a, Planes b, PlanesOut y, int64_t n) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    split1(join1(a, i) + join1(b, i), y, i);
}

// Host fp32 rows [rows, d] <-> device activations [rows, pitch] in the
// pack's storage form (0: bf16, 1: fp32, 2: split planes), zero padding.
__global__ void k_rows_in(const float* __restrict__ src, int rows, int d, int pitch, int form,
                          void* __restrict__ dst) {
  const int64_t n = (int64_t)rows * pitch;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / pitch;
    const int c = static_cast<int>(i - r * pitch);
    const float v = c < d ? src[r * d + c] : 0.0f;
    if (form == 1) {
      static_cast<float*>(dst)[i] = v;
    } else if (form == 0) {
      static_cast<bf16*>(dst)[i] = __float2bfloat16_rn(v);
    } else {
      bf16* h = static_cast<bf16*>(dst);
      split1(v, h[i], h[n + i], h[2 * n + i]);
    }
  }
}
__global__ void k_rows_out(const void* __restrict__ src, int rows, int d, int pitch, int form,
                           float* __restrict__ dst) {
  const int64_t n = (int64_t)rows * d, np = (int64_t)rows * pitch;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / d;
    const int64_t j = r * pitch + (i - r * d);
    if (form == 1) dst[i] = static_cast<const float*>(src)[j];
    else if (form == 0) dst[i] = __bfloat162float(static_cast<const bf16*>(src)[j]);
    else {
      const bf16* h = static_cast<const bf16*>(src);
      dst[i] = join1(Planes{h, h + np, h + 2 * np}, j);
    }
  }
}

int ew_grid(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return static_cast<int>(g < 8 * 148 ? (g > 0 ? g : 1) : 8 * 148);
}

}  // namespace

void rows_to_device(const float* src, int rows, int d, int pitch, int form, void* dst,
                    cudaStream_t s) {
  const int64_t n = (int64_t)rows * pitch;
  if (n == 0) return;
  k_rows_in<<<ew_grid(n), 256, 0, s>>>(src, rows, d, pitch, form, dst);
  check_launch("k_rows_in");
}
void rows_from_device(const void* src, int rows, int d, int pitch, int form, float* dst,
                      cudaStream_t s) {
  const int64_t n = (int64_t)rows * d;
  if (n == 0) return;
  k_rows_out<<<ew_grid(n), 256, 0, s>>>(src, rows, d, pitch, form, dst);
  check_launch("k_rows_out");
}

void split_planes(const float* src, const PlanesOut& y, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  launch_pdl(k_split_planes, dim3(ew_grid(n)), dim3(256), 0, s, src, y, n);
  check_launch("k_split_planes");
}

void merge_planes(const Planes& a, float* dst, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  launch_pdl(k_merge_planes, dim3(ew_grid(n)), dim3(256), 0, s, a, dst, n);
  check_launch("k_merge_planes");
}

void ln_planes(const Planes& a, const Planes* b, const float* gamma, const float* beta, float eps,
               const PlanesOut& y, int rows, int d, cudaStream_t s, int pitch) {
  const Planes bb = b ? *b : Planes{nullptr, nullptr, nullptr};
  const dim3 grid((rows + 7) / 8);
  if (pitch <= 0) pitch = d;
  if (pitch <= 32 * 32) {
    launch_pdl(k_ln_planes<32>, grid, dim3(256), 0, s, a, bb, gamma, beta, eps, y, rows, d, pitch);
    check_launch("k_ln_planes");
  } else if (pitch <= 64 * 32) {
    launch_pdl(k_ln_planes<64>, grid, dim3(256), 0, s, a, bb, gamma, beta, eps, y, rows, d, pitch);
    check_launch("k_ln_planes");
  } else {
    if (y.hi == a.hi || (b && y.hi == b->hi))
      throw CudaError("ln_planes: rows wider than 2048 cannot run in place");
    launch_pdl(k_ln_planes_wide, grid, dim3(256), 0, s, a, bb, gamma, beta, eps, y, rows, d,
               pitch);
    check_launch("k_ln_planes_wide");
  }
}

void add_planes(const Planes& a, const Planes& b, const PlanesOut& y, int64_t n, cudaStream_t s) {
  if (n == 0) return;
  launch_pdl(k_add_planes, dim3(ew_grid(n)), dim3(256), 0, s, a, b, y, n);
  check_launch("k_add_planes");
}

}  // namespace fsvd
