// Developer probe: tcgen05.mma throughput (SS, M=128, K=16 bf16) vs N, and the
// cost of commit+wait round trips, measured with clock64 on every SM.
#include <cstdio>
#include <vector>

#include "../../paper_2508_01506_b200/csrc/common.cuh"
#include "../../paper_2508_01506_b200/csrc/ptx.cuh"

using namespace fsvd;
using namespace fsvd::ptx;

// whole warp executes; one elected lane issues (no C++-level divergence)
__device__ __forceinline__ void mma_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}

// mode 0: commit + wait own MMAs every `sync_every`; 1: commit only (to a
// second barrier, never waited); 2: wait on an already-completed barrier +
// tcgen05 fence (no drain); 3: fence only.
__global__ void __launch_bounds__(128, 1) k_probe(int n, int iters, int sync_every, int mode,
                                                  int use_elect, long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bar2, done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < (128 + 256) * 64 * 2 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    mbar_init(&done, 1);
    mbar_arrive(&done);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tslot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 128 * 128);
    const uint32_t idesc = idesc_bf16(128, n);
    uint32_t phase = 0;
    long long t0 = clock64();
    const bool leader = use_elect ? elect_one() : (lane == 0);
    if (use_elect == 5 || use_elect == 6) {
      // warp-uniform loop, precomputed descriptors; 5: one elect per 4 MMAs,
      // 6: one elect per 16 MMAs
      const uint64_t ad = desc_kmajor(a, 128), bd = desc_kmajor(b, 128);
      const int per = use_elect == 5 ? 4 : 16;
      for (int i = 0; i < iters; i += per) {
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (k < per) mma_bf16_ss(tmem, ad + 2 * (k & 3), bd + 2 * (k & 3), idesc, 1);
        }
        __syncwarp();
      }
    } else if (use_elect == 4) {
      if (lane == 0) {
        uint64_t ad[4], bd[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          ad[k] = desc_kmajor(a + k * 32, 128);
          bd[k] = desc_kmajor(b + k * 32, 128);
        }
        for (int i = 0; i < iters; i += 4) {
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_bf16_ss(tmem, ad[k], bd[k], idesc, 1);
          if (sync_every && ((i + 4) & (sync_every - 1)) == 0) {
            if (mode == 0) {
              mma_commit(&bar);
              mbar_wait(&bar, phase);
              phase ^= 1;
            } else if (mode == 1) {
              mma_commit(&bar2);
            } else if (mode == 2) {
              mbar_wait(&done, 0);
              tc_fence_after();
            }
          }
        }
      }
      __syncwarp();
    } else if (use_elect == 3) {
      if (lane == 0) {
        for (int i = 0; i < iters; ++i) {
          mma_bf16_ss(tmem, desc_kmajor(a + (i & 3) * 32, 128), desc_kmajor(b + (i & 3) * 32, 128),
                      idesc, 1);
          if (sync_every && ((i + 1) & (sync_every - 1)) == 0) {
            if (mode == 0) {
              mma_commit(&bar);
              mbar_wait(&bar, phase);
              phase ^= 1;
            } else if (mode == 1) {
              mma_commit(&bar2);
            } else if (mode == 2) {
              mbar_wait(&done, 0);
              tc_fence_after();
            } else {
              tc_fence_after();
            }
          }
        }
      }
      __syncwarp();
    } else
    for (int i = 0; i < iters; ++i) {
      if (use_elect == 2)
        mma_warp(tmem, desc_kmajor(a + (i & 3) * 32, 128), desc_kmajor(b + (i & 3) * 32, 128),
                 idesc, 1);
      else if (leader)
        mma_bf16_ss(tmem, desc_kmajor(a + (i & 3) * 32, 128), desc_kmajor(b + (i & 3) * 32, 128),
                    idesc, 1);
      if (sync_every && ((i + 1) & (sync_every - 1)) == 0) {
        if (mode == 0) {
          if (use_elect == 2) commit_warp(&bar);
          else if (leader) mma_commit(&bar);
          __syncwarp();
          mbar_wait(&bar, phase);
          phase ^= 1;
        } else if (mode == 1) {
          if (use_elect == 2) commit_warp(&bar2);
          else if (leader) mma_commit(&bar2);
          __syncwarp();
        } else if (mode == 2) {
          mbar_wait(&done, 0);
          tc_fence_after();
        } else {
          tc_fence_after();
        }
      }
    }
    if (lane == 0) mma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, phase);
    long long t1 = clock64();
    if (lane == 0) cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_free<512>(tmem);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const int blocks = 148, smem = 1024 + (128 + 256) * 128;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long* d;
  cudaMalloc(&d, blocks * sizeof(long long));
  std::vector<long long> h(blocks);
  for (int el : {4, 5, 6})
  for (int mode : {0})
  for (int sync : {0}) {
    if (sync == 0 && mode > 0) continue;
    for (int n : {32, 64, 128, 192, 256}) {
      const int iters = 4096;
      k_probe<<<blocks, 128, smem>>>(n, iters, sync, mode, el, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h.data(), d, blocks * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (auto c : h) avg += c;
      avg /= blocks;
      const double ideal = 128.0 * n / 256.0;  // cycles per K=16 instruction at 4096 MAC/clk
      printf("elect=%d mode=%d sync_every=%2d N=%3d  %.1f cycles/instr (ideal %.0f)  eff %.2f\n", el, mode, sync, n,
             avg / iters, ideal, ideal / (avg / iters));
      (void)mode;
    }
  }
  return 0;
}
