// Developer probe: does a concurrent HBM-bound TMA stream slow an L2-hot one?
// warp 0 streams [64 x 64] boxes of a 1 MB (L2-resident) matrix; warp 1
// (optional) streams [128 x 64] boxes of a 2 GB matrix (HBM).  Reports the
// hot stream's bytes/clk and mean issue->land latency.
#include <cstdio>
#include <vector>
#include <algorithm>

#include "../../paper_2508_01506_b200/csrc/common.cuh"
#include "../../paper_2508_01506_b200/csrc/ptx.cuh"

using namespace fsvd;
using namespace fsvd::ptx;

__global__ void __launch_bounds__(64, 1) k_mix(const __grid_constant__ CUtensorMap hot,
                                              const __grid_constant__ CUtensorMap cold,
                                              int cold_on, int iters, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t fh[6], fc[4];
  __shared__ long long lat_sum;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 6; ++i) mbar_init(&fh[i], 1);
    for (int i = 0; i < 4; ++i) mbar_init(&fc[i], 1);
    lat_sum = 0;
    fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (warp == 0 && lane == 0) {
    long long issue[6];
    long long lsum = 0;
    for (int i = 0; i < iters; ++i) {
      const int s = i % 6;
      if (i >= 6) {
        mbar_wait(&fh[s], ((i / 6) - 1) & 1);
        lsum += clock64() - issue[s];
      }
      issue[s] = clock64();
      mbar_arrive_expect_tx(&fh[s], 8192);
      tma_load_2d(&hot, &fh[s], smem + s * 8192, 0, ((blockIdx.x * 3 + i) % 128) * 64);
    }
    lat_sum = lsum / (iters - 6);
  }
  if (warp == 1 && lane == 0 && cold_on) {
    uint8_t* cs = smem + 6 * 8192;
    for (int i = 0; i < iters / 2; ++i) {
      const int s = i % 4;
      if (i >= 4) mbar_wait(&fc[s], ((i / 4) - 1) & 1);
      mbar_arrive_expect_tx(&fc[s], 16384);
      tma_load_2d(&cold, &fc[s], cs + s * 16384, 0, (int)(((long long)blockIdx.x * 1000003 + i * 128) % (1 << 23)) & ~127);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = lat_sum;
  }
}

int main() {
  void *hotm, *coldm;
  cudaMalloc(&hotm, 8192 * 128);             // 8192 rows x 64 bf16 = 1 MB
  cudaMalloc(&coldm, (size_t)(1 << 23) * 128);  // 8M rows x 128 B = 1 GB
  cudaMemset(hotm, 0, 8192 * 128);
  cudaMemset(coldm, 0, (size_t)(1 << 23) * 128);
  long long* d;
  cudaMalloc(&d, 2 * 148 * sizeof(long long));
  cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  CUtensorMap th = tmap_bf16(hotm, 8192, 64, 64, 64, 64, TmaSwizzle::B128);
  CUtensorMap tc = tmap_bf16(coldm, 1 << 23, 64, 64, 128, 64, TmaSwizzle::B128);
  for (int grid : {1, 128})
    for (int cold_on : {0, 1}) {
      const int iters = 3000;
      for (int rep = 0; rep < 2; ++rep) k_mix<<<grid, 64, 6 * 8192 + 4 * 16384 + 1024>>>(th, tc, cold_on, iters, d);
      cudaDeviceSynchronize();
      std::vector<long long> h(2 * grid);
      cudaMemcpy(h.data(), d, 2 * grid * sizeof(long long), cudaMemcpyDeviceToHost);
      std::vector<long long> cyc, lat;
      for (int i = 0; i < grid; ++i) { cyc.push_back(h[2 * i]); lat.push_back(h[2 * i + 1]); }
      std::sort(cyc.begin(), cyc.end());
      std::sort(lat.begin(), lat.end());
      printf("grid %3d cold %d : hot %.1f B/clk, hot latency %lld cyc (median)\n", grid, cold_on,
             (double)iters * 8192 / cyc[grid / 2], lat[grid / 2]);
    }
  return 0;
}
