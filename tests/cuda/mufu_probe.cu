// Developer probe: MUFU ex2 throughput per SM for f32, f16x2 and bf16x2
// operands (exponentials per clock per SM), and the f16x2 / bf16x2 accuracy
// against exp2f on [-16, 8].
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

template <int MODE>
__global__ void k_ex2(float* out, long long* clk, int iters) {
  uint32_t v[8];
  for (int i = 0; i < 8; ++i) v[i] = 0x3c003c00u ^ (threadIdx.x * 7 + i);  // ~1.0 halves
  float f[8];
  for (int i = 0; i < 8; ++i) f[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
      if (MODE == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
      if (MODE == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[i]));
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += f[i] + __uint_as_float(v[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

__global__ void k_acc(float* err16, float* err_bf) {
  // x on a grid over [-16, 8]
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  float x = -16.0f + 24.0f * i / (gridDim.x * blockDim.x);
  float ref = exp2f(x);
  __half2 h = __floats2half2_rn(x, x);
  uint32_t hv = *reinterpret_cast<uint32_t*>(&h), ho;
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(ho) : "r"(hv));
  __half2 hr = *reinterpret_cast<__half2*>(&ho);
  float y16 = __low2float(hr);
  __nv_bfloat162 b = __floats2bfloat162_rn(x, x);
  uint32_t bv = *reinterpret_cast<uint32_t*>(&b), bo;
  asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(bo) : "r"(bv));
  __nv_bfloat162 br = *reinterpret_cast<__nv_bfloat162*>(&bo);
  float ybf = __low2float(br);
  err16[i] = fabsf(y16 - ref) / ref;
  err_bf[i] = fabsf(ybf - ref) / ref;
}

int main() {
  float* out; long long* clk;
  cudaMalloc(&out, 148 * 4 * 1024 * 4);
  cudaMalloc(&clk, 148 * 4 * 8);
  const int iters = 4096;
  long long h[148 * 4];
  const char* names[3] = {"f32   ", "f16x2 ", "bf16x2"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k_ex2<0><<<148 * 2, 512>>>(out, clk, iters);
      if (mode == 1) k_ex2<1><<<148 * 2, 512>>>(out, clk, iters);
      if (mode == 2) k_ex2<2><<<148 * 2, 512>>>(out, clk, iters);
    }
    cudaDeviceSynchronize();
    cudaMemcpy(h, clk, 148 * 2 * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < 148 * 2; ++i) mx = h[i] > mx ? h[i] : mx;
    // 2 CTAs x 512 threads per SM, 8 instr per iter; f16x2 / bf16x2 give 2 exps per lane
    double instr_per_clk = 2.0 * 512 * 8 * iters / mx;
    printf("%s: %.1f lane-instr/clk/SM, %.1f exps/clk/SM\n", names[mode], instr_per_clk,
           instr_per_clk * (mode ? 2 : 1));
  }
  float *e16, *ebf;
  const int n = 256 * 1024;
  cudaMalloc(&e16, n * 4); cudaMalloc(&ebf, n * 4);
  k_acc<<<1024, 256>>>(e16, ebf);
  static float a[256 * 1024], b[256 * 1024];
  cudaMemcpy(a, e16, n * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(b, ebf, n * 4, cudaMemcpyDeviceToHost);
  double m16 = 0, mbf = 0, s16 = 0, sbf = 0;
  for (int i = 0; i < n; ++i) { m16 = fmax(m16, a[i]); mbf = fmax(mbf, b[i]); s16 += a[i]; sbf += b[i]; }
  printf("rel err vs exp2f on [-16, 8] (input rounding included): f16x2 max %.2e mean %.2e | bf16x2 max %.2e mean %.2e\n",
         m16, s16 / n, mbf, sbf / n);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
