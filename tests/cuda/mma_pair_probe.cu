// Developer probe: tcgen05.mma.cta_group::2 (M = 256) issue/throughput vs
// cta_group::1 (M = 128), SS operands, per-SM cycles per MMA instruction.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "../../paper_2508_01506_b200/csrc/common.cuh"
#include "../../paper_2508_01506_b200/csrc/ptx.cuh"

using namespace fsvd;
using namespace fsvd::ptx;

template <bool PAIR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_probe(int n, int iters, long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  for (int i = threadIdx.x; i < (128 + 256) * 64 * 2 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if (PAIR) tmem_alloc_pair<512>(&tslot);
    else tmem_alloc<512>(&tslot);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1 && (!PAIR || rank == 0)) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 128 * 128);
    const uint32_t idesc = idesc_bf16(PAIR ? 256 : 128, n);
    const uint64_t ad = desc_kmajor(a, 128), bd = desc_kmajor(b, 128);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 4) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (PAIR) mma_bf16_ss_pair(tmem, ad + 2 * k, bd + 2 * k, idesc, 1);
          else mma_bf16_ss(tmem, ad + 2 * k, bd + 2 * k, idesc, 1);
        }
      }
      __syncwarp();
    }
    if (elect_one()) {
      if (PAIR) mma_commit_pair(&bar, 0x1);
      else mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (lane == 0) cycles[blockIdx.x / 2] = t1 - t0;
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    if (PAIR) tmem_free_pair<512>(tmem);
    else tmem_free<512>(tmem);
  }
}

int main() {
  const int blocks = 148, smem = 1024 + (128 + 256) * 128;
  cudaFuncSetAttribute(k_probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long* d;
  cudaMalloc(&d, blocks * sizeof(long long));
  std::vector<long long> h(blocks / 2);
  for (int pair : {0, 1})
    for (int n : {64, 128, 256}) {
      const int iters = 4096;
      if (pair) k_probe<true><<<blocks, 128, smem>>>(n, iters, d);
      else k_probe<false><<<blocks, 128, smem>>>(n, iters, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
      std::sort(h.begin(), h.end());
      const double c = (double)h[h.size() / 2] / iters;
      // per SM: 128 rows x n x 16 MACs per instruction either way
      printf("pair=%d N=%3d: %.1f cycles/instr (ideal %.0f)\n", pair, n, c, 128.0 * n / 256.0);
    }
  return 0;
}
