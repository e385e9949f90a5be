// Standalone K1 check: tcgen05 GEMM vs a double-precision host reference.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../../paper_2508_01506_b200/csrc/common.cuh"
#include "../../paper_2508_01506_b200/csrc/kernels.cuh"
using namespace fsvd;
static float frand(uint64_t& s) { s = s * 6364136223846793005ULL + 1442695040888963407ULL; return ((s >> 40) & 0xFFFFFF) / float(1 << 24) * 2.f - 1.f; }
int run(int M, int N, int K, bool use_bias, int act) {
  uint64_t seed = M * 131 + N * 7 + K;
  std::vector<bf16> A(size_t(M) * K), B(size_t(N) * K); std::vector<float> bias(N);
  std::vector<float> Af(A.size()), Bf(B.size());
  for (size_t i = 0; i < A.size(); ++i) { A[i] = __float2bfloat16(frand(seed)); Af[i] = __bfloat162float(A[i]); }
  for (size_t i = 0; i < B.size(); ++i) { B[i] = __float2bfloat16(frand(seed)); Bf[i] = __bfloat162float(B[i]); }
  for (auto& b : bias) b = frand(seed);
  bf16 *dA, *dB, *dC; float* dbias;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dC, size_t(M) * N * 2); cudaMalloc(&dbias, N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dbias, bias.data(), N * 4, cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, size_t(M) * N * 2);
  gemm_bf16(dA, K, dB, K, dC, N, M, N, K, use_bias ? dbias : nullptr, act, 0);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<bf16> C(size_t(M) * N); cudaMemcpy(C.data(), dC, C.size() * 2, cudaMemcpyDeviceToHost);
  double worst = 0, ref_max = 0;
  for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) {
    double acc = use_bias ? bias[j] : 0;
    for (int k = 0; k < K; ++k) acc += double(Af[size_t(i) * K + k]) * Bf[size_t(j) * K + k];
    if (act == 0) acc = 0.5 * acc * (1 + erf(acc / sqrt(2.0)));
    double got = __bfloat162float(C[size_t(i) * N + j]);
    worst = fmax(worst, fabs(got - acc)); ref_max = fmax(ref_max, fabs(acc));
  }
  // time it
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) gemm_bf16(dA, K, dB, K, dC, N, M, N, K, use_bias ? dbias : nullptr, act, 0);
  cudaEventRecord(a); int it = 20;
  for (int w = 0; w < it; ++w) gemm_bf16(dA, K, dB, K, dC, N, M, N, K, use_bias ? dbias : nullptr, act, 0);
  cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); ms /= it;
  double tf = 2.0 * M * N * K / (ms * 1e-3) / 1e12;
  printf("M=%d N=%d K=%d bias=%d act=%d  max|err|=%.4g  rel=%.3g  %.3f ms %.1f TFLOP/s %s\n", M, N, K, use_bias, act, worst, worst / ref_max, ms, tf, worst / ref_max < 1e-2 ? "OK" : "FAIL");
  cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dbias);
  return worst / ref_max < 1e-2 ? 0 : 1;
}
int main(int argc, char** argv) { setvbuf(stdout, NULL, _IONBF, 0);
  if (argc == 4) return run(atoi(argv[1]), atoi(argv[2]), atoi(argv[3]), false, 3);
  int fails = 0;
  fails += run(128, 64, 64, false, 3);
  fails += run(128, 128, 128, false, 3);
  fails += run(256, 256, 256, true, 3);
  fails += run(200, 192, 768, true, 0);
  fails += run(1000, 1152, 768, false, 3);
  fails += run(333, 104, 40, true, 3);
  fails += run(16384, 1152, 768, false, 3);
  fails += run(16384, 384, 768, false, 3);
  fails += run(16384, 768, 384, true, 3);
  fails += run(8192, 8192, 8192 / 8, false, 3);
  printf("%s\n", fails ? "SOME FAILED" : "ALL OK");
  return fails;
}
