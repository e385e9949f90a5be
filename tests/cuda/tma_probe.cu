// Developer probe: per-SM TMA load throughput from an L2-resident matrix.
// One CTA per SM; one thread streams boxes of [box_rows x 64] bf16 (SW128)
// into a ring of `depth` slots and re-issues as soon as each slot lands (no
// consumer), so the rate is what the TMA path delivers.  Variants: box rows,
// ring depth, number of CTAs reading the SAME lines vs. distinct lines.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "../../paper_2508_01506_b200/csrc/common.cuh"
#include "../../paper_2508_01506_b200/csrc/ptx.cuh"

using namespace fsvd;
using namespace fsvd::ptx;

__global__ void __launch_bounds__(128, 1) k_tma(const __grid_constant__ CUtensorMap tm, int box_rows,
                                               int depth, int iters, int rows_total, int same,
                                               int prefetch, long long* cycles) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem0 = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t fulls[4][16];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t* full = fulls[w];
  const int bytes = box_rows * 128;
  uint8_t* smem = smem0 + w * depth * bytes;
  if (lane == 0) {
    if (prefetch) tma_prefetch(&tm);
    for (int i = 0; i < depth; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int nbox_rows = rows_total / box_rows;  // rows_total = span actually read
  const int start = same ? 0 : (blockIdx.x * 7) % nbox_rows;
  long long t0 = clock64();
  if (lane == 0) {
    for (int i = 0; i < depth; ++i) {
      mbar_arrive_expect_tx(&full[i], bytes);
      const int r = ((start + i) % nbox_rows) * box_rows;
      tma_load_2d(&tm, &full[i], smem + i * bytes, 0, r);
    }
    for (int i = depth; i < iters; ++i) {
      const int s = i % depth;
      mbar_wait(&full[s], ((i / depth) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], bytes);
      const int r = ((start + i) % nbox_rows) * box_rows;
      tma_load_2d(&tm, &full[s], smem + s * bytes, 0, r);
    }
    for (int i = iters; i < iters + depth; ++i) {
      const int s = i % depth;
      mbar_wait(&full[s], ((i / depth) - 1) & 1);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = (t1 - t0) / nw;
}

int main() {
  const int rows_total = 8192 * 64;  // 64 MB; the kernel reads the first `span` rows
  void* mat;
  cudaMalloc(&mat, (size_t)rows_total * 64 * 2);
  cudaMemset(mat, 0, (size_t)rows_total * 64 * 2);
  long long* d_cyc;
  cudaMalloc(&d_cyc, 148 * sizeof(long long));
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("span_rows box_rows depth grid warps same : B/clk per SM (median CTA), chip B/clk\n");
  const int pf = 1;
  for (int span : {8192, 8192 * 64})
   for (int same : {0, 1})
    for (int grid : {74, 148})
    for (int nw : {2, 4})
      for (int box_rows : {128, 256})
        for (int depth : {3}) {
          if (nw * depth * box_rows * 128 > 190 * 1024) continue;
          CUtensorMap tm = tmap_bf16(mat, rows_total, 64, 64, box_rows, 64, TmaSwizzle::B128);
          const int iters = 2000 * 64 / box_rows;
          for (int rep = 0; rep < 2; ++rep)
            k_tma<<<grid, 32 * nw, nw * depth * box_rows * 128 + 1024>>>(
                tm, box_rows, depth, iters, span, same, pf, d_cyc);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
          }
          std::vector<long long> c(grid);
          cudaMemcpy(c.data(), d_cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
          std::sort(c.begin(), c.end());
          const double bytes = (double)iters * box_rows * 128;
          printf("%6d %4d %3d %4d %d %d : %6.1f B/clk  chip %7.0f B/clk\n", span, box_rows, depth,
                 grid, nw, same, bytes / c[c.size() / 2], grid * bytes / c[c.size() - 1]);
        }
  (void)nsm;
  return 0;
}
