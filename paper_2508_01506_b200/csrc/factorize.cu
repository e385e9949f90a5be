// factorize.cu -- batched rank-r factorization on the device (SURVEY 8(f)
// row 2): the reference's factor_rank_r (svd.cpp:325-456) for every matrix
// of a model in one run.
//
// The reference runs one-sided cyclic Jacobi in fp64 per matrix, serially,
// after a Householder QR for tall inputs, then recovers v_j = Op^T u_j /
// sigma_j, applies the even split and the sign convention.  Here every
// matrix of the batch is oriented tall (A or A^T, M >= N), widened to fp64
// column-major in HBM, and orthogonalized by a one-sided BLOCK Jacobi:
//
//   * the N columns are cut into nb blocks of w columns; a sweep pairs the
//     blocks by the circle method (nb - 1 steps of nb/2 disjoint pairs), so
//     one launch per step runs nb/2 independent CTAs per matrix, all
//     matrices of the batch side by side;
//   * a visit CTA stages the 2w columns of its block pair in shared memory
//     (<= 200 KB) and rotates every cross pair (w rounds of w disjoint
//     pairs, one warp group per pair); at step 0 it also rotates the pairs
//     inside both blocks, so a sweep touches every column pair exactly once;
//   * the rotation is the reference's (svd.cpp:65-87): skip when either norm
//     is below 1e-30 of the largest initial column norm or when
//     |c| <= 1e-15 sqrt(|p|^2 |q|^2); otherwise the small-angle tangent.
//     Norms and the dot product are recomputed exactly at every visit;
//   * sweeps stop per matrix when a sweep rotates nothing (cap 60, as the
//     reference).
//
// Finalisation follows factor_tall (svd.cpp:345-407): exact column norms,
// stable descending order, zero factors below 1e-15 sigma_max, v from the
// pre-rotation operand, the sign convention on the left factor of the final
// orientation (svd.cpp:391-407, 437-449), the even sqrt(sigma) split, fp32
// outputs.  The QR precondition of the reference only changes how fast
// Jacobi converges, not what it converges to, so it is not reproduced.
#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "errors.hpp"
#include "factorize.hpp"

namespace fsvd {
namespace {

constexpr int kVisitThreads = 512;                // 16 warps
constexpr int kVisitWarps = kVisitThreads / 32;
constexpr size_t kColBytes = 200 * 1024;          // staged columns per visit CTA
constexpr double kPairTol = 1.0e-15;              // svd.cpp:22
constexpr int kMaxSweeps = 60;                    // svd.cpp:23
constexpr int kMaxW = 16;

struct DevJob {
  double* work;                 // oriented operand, column-major M x npad
  const float* a;               // compact row-major m x n input
  double* x;                    // left vectors of the operand, x[j*M + i]
  double* y;                    // right vectors, y[j*N + k]
  double* sigma;                // npad column norms
  const int* src;               // r source columns, descending sigma
  const double* sr;             // r singular values (0: zero factor)
  float* u;                     // m x r
  float* v;                     // r x n
  unsigned long long* maxsq;    // largest initial column |.|^2 (double bits)
  unsigned* rot;                // rotations this sweep
  int m, n, M, N, r, wide, w, nb, npad;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Oriented operand element (i, j): A for tall inputs, A^T for wide ones.
__device__ __forceinline__ double op_at(const DevJob& J, int i, int j) {
  return J.wide ? static_cast<double>(J.a[static_cast<size_t>(j) * J.n + i])
                : static_cast<double>(J.a[static_cast<size_t>(i) * J.n + j]);
}

__global__ void k_widen(const DevJob* jobs) {
  const DevJob& J = jobs[blockIdx.y];
  const size_t total = static_cast<size_t>(J.M) * J.npad;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(e / J.M), i = static_cast<int>(e % J.M);
    J.work[e] = j < J.N ? op_at(J, i, j) : 0.0;
  }
}

// Column norms^2 (warp per column); `max_only` folds them into J.maxsq,
// otherwise sigma[j] = sqrt(norm^2) for every padded column.
__global__ void k_colnorms(const DevJob* jobs, int max_only) {
  const DevJob& J = jobs[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int j = blockIdx.x * wpb + warp; j < J.npad; j += gridDim.x * wpb) {
    const double* c = J.work + static_cast<size_t>(j) * J.M;
    double s = 0.0;
    for (int i = lane; i < J.M; i += 32) s = fma(c[i], c[i], s);
    s = warp_sum(s);
    if (lane == 0) {
      if (max_only)
        atomicMax(J.maxsq, static_cast<unsigned long long>(__double_as_longlong(s)));
      else
        J.sigma[j] = sqrt(s);
    }
  }
}

// One block-pair visit: blockIdx.x = pair slot of step `step`, blockIdx.y
// indexes `ids` (the active jobs of one block-count class).
__global__ void __launch_bounds__(kVisitThreads, 1)
    k_visit(const DevJob* jobs, const int* ids, int step, int full) {
  const DevJob& J = jobs[ids[blockIdx.y]];
  const int L = J.nb - 1, k = blockIdx.x, w = J.w, M = J.M;
  const int bp = k == 0 ? step : (step + k) % L;
  const int bq = k == 0 ? L : (step - k + L) % L;
  extern __shared__ double cols[];
  __shared__ double red[kVisitWarps][3];

  for (int c = 0; c < 2 * w; ++c) {
    const int gc = c < w ? bp * w + c : bq * w + (c - w);
    const double* g = J.work + static_cast<size_t>(gc) * M;
    for (int i = threadIdx.x; i < M; i += kVisitThreads) cols[c * M + i] = g[i];
  }
  __syncthreads();

  const double floor_sq = __longlong_as_double(static_cast<long long>(*J.maxsq)) * 1.0e-30;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = max(1, kVisitWarps / w);      // warps per column pair
  const int slot = warp / G, gw = warp % G;
  const int gt = gw * 32 + lane, gthreads = G * 32;
  unsigned nrot = 0;
  const int rounds = full ? 2 * w - 1 : w;
  for (int t = 0; t < rounds; ++t) {
    int p = -1, q = -1;
    if (slot < w) {
      if (full) {  // circle method over all 2w staged columns
        const int L2 = 2 * w - 1;
        p = slot == 0 ? t : (t + slot) % L2;
        q = slot == 0 ? L2 : (t - slot + L2) % L2;
      } else {     // cross pairs only
        p = slot;
        q = w + (slot + t) % w;
      }
    }
    if (p >= 0) {
      const double* cp = cols + p * M;
      const double* cq = cols + q * M;
      double c = 0.0, sp = 0.0, sq = 0.0;
      for (int i = gt; i < M; i += gthreads) {
        const double a = cp[i], b = cq[i];
        c = fma(a, b, c);
        sp = fma(a, a, sp);
        sq = fma(b, b, sq);
      }
      c = warp_sum(c);
      sp = warp_sum(sp);
      sq = warp_sum(sq);
      if (lane == 0) {
        red[warp][0] = c;
        red[warp][1] = sp;
        red[warp][2] = sq;
      }
    }
    __syncthreads();
    if (p >= 0) {
      double c = 0.0, sp = 0.0, sq = 0.0;
      for (int g = 0; g < G; ++g) {
        c += red[slot * G + g][0];
        sp += red[slot * G + g][1];
        sq += red[slot * G + g][2];
      }
      const bool live = sp > floor_sq && sq > floor_sq;
      if (live && fabs(c) > kPairTol * sqrt(sp * sq)) {
        const double zeta = (sq - sp) / (2.0 * c);
        const double tn = copysign(1.0 / (fabs(zeta) + sqrt(1.0 + zeta * zeta)), zeta);
        const double cs = 1.0 / sqrt(1.0 + tn * tn);
        const double sn = cs * tn;
        double* cp = cols + p * M;
        double* cq = cols + q * M;
        for (int i = gt; i < M; i += gthreads) {
          const double xp = cp[i], xq = cq[i];
          cp[i] = cs * xp - sn * xq;
          cq[i] = sn * xp + cs * xq;
        }
        ++nrot;
      }
    }
    __syncthreads();
  }

  for (int c = 0; c < 2 * w; ++c) {
    const int gc = c < w ? bp * w + c : bq * w + (c - w);
    double* g = J.work + static_cast<size_t>(gc) * M;
    for (int i = threadIdx.x; i < M; i += kVisitThreads) g[i] = cols[c * M + i];
  }
  if (gt == 0 && nrot) atomicAdd(J.rot, nrot);
}

// x[:, jj] = work[:, src[jj]] / sigma (zero factor: 0).
__global__ void k_left(const DevJob* jobs) {
  const DevJob& J = jobs[blockIdx.y];
  const size_t total = static_cast<size_t>(J.M) * J.r;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int jj = static_cast<int>(e / J.M), i = static_cast<int>(e % J.M);
    const double s = J.sr[jj];
    J.x[e] = s > 0.0 ? J.work[static_cast<size_t>(J.src[jj]) * J.M + i] / s : 0.0;
  }
}

// y[:, jj] = Op^T x[:, jj] / sigma_jj against the pre-rotation operand
// (svd.cpp:368-379): a [N x M] . [M x r] fp64 product, 32 x 32 output tiles.
constexpr int kRT = 32;
__global__ void __launch_bounds__(256) k_right(const DevJob* jobs) {
  const DevJob& J = jobs[blockIdx.z];
  const int k0 = blockIdx.x * kRT, j0 = blockIdx.y * kRT;
  if (k0 >= J.N || j0 >= J.r) return;
  __shared__ double so[kRT][kRT + 1];  // [i][k]
  __shared__ double sx[kRT][kRT + 1];  // [i][jj]
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // ty 0..7
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int i0 = 0; i0 < J.M; i0 += kRT) {
    for (int e = threadIdx.x; e < kRT * kRT; e += 256) {
      const int ii = e / kRT, cc = e % kRT;
      const int i = i0 + ii;
      so[ii][cc] = (i < J.M && k0 + cc < J.N) ? op_at(J, i, k0 + cc) : 0.0;
      sx[ii][cc] = (i < J.M && j0 + cc < J.r) ? J.x[static_cast<size_t>(j0 + cc) * J.M + i] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int ii = 0; ii < kRT; ++ii) {
      const double o = so[ii][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(o, sx[ii][ty + 8 * q], acc[q]);
    }
    __syncthreads();
  }
  const int kk = k0 + tx;
  if (kk >= J.N) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int jj = j0 + ty + 8 * q;
    if (jj >= J.r) continue;
    const double s = J.sr[jj];
    J.y[static_cast<size_t>(jj) * J.N + kk] = s > 0.0 ? acc[q] / s : 0.0;
  }
}

// Sign convention + even split + fp32 outputs, one CTA per (factor, job).
__global__ void __launch_bounds__(256) k_output(const DevJob* jobs) {
  const DevJob& J = jobs[blockIdx.y];
  const int jj = blockIdx.x;
  if (jj >= J.r) return;
  // final orientation: tall -> U = x, V = y; wide -> U = y, V = x
  const double* uc = J.wide ? J.y + static_cast<size_t>(jj) * J.N : J.x + static_cast<size_t>(jj) * J.M;
  const double* vr = J.wide ? J.x + static_cast<size_t>(jj) * J.M : J.y + static_cast<size_t>(jj) * J.N;
  __shared__ double smag[256];
  __shared__ int sarg[256];
  double best = 0.0;
  int arg = 0;
  for (int i = threadIdx.x; i < J.m; i += 256) {
    const double mg = fabs(uc[i]);
    if (mg > best) {  // strided scan keeps the first index per thread
      best = mg;
      arg = i;
    }
  }
  smag[threadIdx.x] = best;
  sarg[threadIdx.x] = arg;
  __syncthreads();
  for (int s = 128; s; s >>= 1) {
    if (threadIdx.x < s) {
      const double ob = smag[threadIdx.x + s];
      const int oa = sarg[threadIdx.x + s];
      if (ob > smag[threadIdx.x] || (ob == smag[threadIdx.x] && ob > 0.0 && oa < sarg[threadIdx.x])) {
        smag[threadIdx.x] = ob;
        sarg[threadIdx.x] = oa;
      }
    }
    __syncthreads();
  }
  const double flip = uc[sarg[0]] < 0.0 ? -1.0 : 1.0;
  const double f = flip * sqrt(J.sr[jj]);
  for (int i = threadIdx.x; i < J.m; i += 256)
    J.u[static_cast<size_t>(i) * J.r + jj] = static_cast<float>(f * uc[i]);
  for (int k = threadIdx.x; k < J.n; k += 256)
    J.v[static_cast<size_t>(jj) * J.n + k] = static_cast<float>(f * vr[k]);
}

int g_last_sweeps = 0;

size_t al(size_t b) { return (b + 255) & ~size_t(255); }

}  // namespace

int last_factor_sweeps() { return g_last_sweeps; }

void check_factor_job(size_t m, size_t n, size_t r) {
  if (r == 0) fail(Kind::Rank, "factorization rank must be at least 1");
  if (r > std::min(m, n)) fail(Kind::Rank, "factorization rank exceeds min(m, n)");
}

void factor_rank_r_batch(const std::vector<FactorJob>& jobs) {
  for (const FactorJob& j : jobs) {
    check_factor_job(j.m, j.n, j.r);
    if (!j.a || !j.u || !j.v) fail(Kind::Config, "null matrix or output pointer");
    if (j.lda < j.n) fail(Kind::Shape, "leading dimension smaller than the column count");
    if (std::max(j.m, j.n) * 2 * sizeof(double) > kColBytes)
      fail(Kind::Config, "matrix dimension " + std::to_string(std::max(j.m, j.n)) +
                             " exceeds the device factorizer's column budget (12800)");
  }
  g_last_sweeps = 0;
  if (jobs.empty()) return;

  // ---- geometry and arena layout
  const size_t nj = jobs.size();
  std::vector<DevJob> dj(nj);
  std::vector<size_t> off_a(nj), off_w(nj), off_x(nj), off_y(nj), off_s(nj), off_src(nj),
      off_sr(nj), off_u(nj), off_v(nj);
  size_t bytes = al(nj * sizeof(unsigned long long)) + al(nj * sizeof(unsigned));
  const size_t off_max = 0, off_rot = al(nj * sizeof(unsigned long long));
  for (size_t t = 0; t < nj; ++t) {
    const FactorJob& j = jobs[t];
    DevJob& d = dj[t];
    d.m = static_cast<int>(j.m);
    d.n = static_cast<int>(j.n);
    d.r = static_cast<int>(j.r);
    d.wide = j.m < j.n;
    d.M = std::max(d.m, d.n);
    d.N = std::min(d.m, d.n);
    const int wcap = static_cast<int>(kColBytes / (2 * sizeof(double) * d.M));
    d.w = std::max(1, std::min({kMaxW, wcap, (d.N + 1) / 2}));
    d.nb = (d.N + d.w - 1) / d.w;
    d.nb += d.nb & 1;
    d.npad = d.nb * d.w;
    off_a[t] = bytes;   bytes += al(j.m * j.n * sizeof(float));
    off_w[t] = bytes;   bytes += al(static_cast<size_t>(d.M) * d.npad * sizeof(double));
    off_x[t] = bytes;   bytes += al(static_cast<size_t>(d.M) * d.r * sizeof(double));
    off_y[t] = bytes;   bytes += al(static_cast<size_t>(d.N) * d.r * sizeof(double));
    off_s[t] = bytes;   bytes += al(d.npad * sizeof(double));
    off_src[t] = bytes; bytes += al(d.r * sizeof(int));
    off_sr[t] = bytes;  bytes += al(d.r * sizeof(double));
    off_u[t] = bytes;   bytes += al(j.m * j.r * sizeof(float));
    off_v[t] = bytes;   bytes += al(j.r * j.n * sizeof(float));
  }
  const size_t off_jobs = bytes;
  bytes += al(nj * sizeof(DevJob));
  const size_t off_ids = bytes;
  bytes += al(nj * sizeof(int));

  uint8_t* base = nullptr;
  cudaStream_t s = nullptr;
  FSVD_CUDA_CHECK(cudaMalloc(&base, bytes));
  struct Cleanup {
    uint8_t* p;
    cudaStream_t* s;
    ~Cleanup() {
      if (*s) cudaStreamDestroy(*s);
      cudaFree(p);
    }
  } cleanup{base, &s};
  FSVD_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  FSVD_CUDA_CHECK(cudaMemsetAsync(base, 0, off_a.front(), s));
  for (size_t t = 0; t < nj; ++t) {
    DevJob& d = dj[t];
    const FactorJob& j = jobs[t];
    d.a = reinterpret_cast<const float*>(base + off_a[t]);
    d.work = reinterpret_cast<double*>(base + off_w[t]);
    d.x = reinterpret_cast<double*>(base + off_x[t]);
    d.y = reinterpret_cast<double*>(base + off_y[t]);
    d.sigma = reinterpret_cast<double*>(base + off_s[t]);
    d.src = reinterpret_cast<const int*>(base + off_src[t]);
    d.sr = reinterpret_cast<const double*>(base + off_sr[t]);
    d.u = reinterpret_cast<float*>(base + off_u[t]);
    d.v = reinterpret_cast<float*>(base + off_v[t]);
    d.maxsq = reinterpret_cast<unsigned long long*>(base + off_max) + t;
    d.rot = reinterpret_cast<unsigned*>(base + off_rot) + t;
    FSVD_CUDA_CHECK(cudaMemcpy2DAsync(base + off_a[t], j.n * sizeof(float), j.a,
                                      j.lda * sizeof(float), j.n * sizeof(float), j.m,
                                      cudaMemcpyHostToDevice, s));
  }
  DevJob* djobs = reinterpret_cast<DevJob*>(base + off_jobs);
  int* dids = reinterpret_cast<int*>(base + off_ids);
  FSVD_CUDA_CHECK(cudaMemcpyAsync(djobs, dj.data(), nj * sizeof(DevJob), cudaMemcpyHostToDevice, s));

  const int sms = num_sms();
  const unsigned gy = static_cast<unsigned>(nj);
  k_widen<<<dim3(2 * sms, gy), 256, 0, s>>>(djobs);
  check_launch("k_widen");
  k_colnorms<<<dim3(sms, gy), 256, 0, s>>>(djobs, 1);
  check_launch("k_colnorms");

  // ---- Jacobi sweeps, jobs grouped by block count so each launch is dense
  size_t smem = 0;
  for (const DevJob& d : dj)
    smem = std::max(smem, static_cast<size_t>(2 * d.w) * d.M * sizeof(double));
  FSVD_CUDA_CHECK(cudaFuncSetAttribute(k_visit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
  std::vector<char> active(nj, 1);
  std::vector<unsigned> rot(nj);
  int sweeps = 0;
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    std::map<int, std::vector<int>> classes;  // nb -> active job ids
    for (size_t t = 0; t < nj; ++t)
      if (active[t] && dj[t].nb >= 2) classes[dj[t].nb].push_back(static_cast<int>(t));
    if (classes.empty()) break;
    std::vector<int> ids;
    std::vector<std::pair<int, std::pair<int, int>>> spans;  // nb, (offset, count)
    for (auto& kv : classes) {
      spans.push_back({kv.first, {static_cast<int>(ids.size()), static_cast<int>(kv.second.size())}});
      ids.insert(ids.end(), kv.second.begin(), kv.second.end());
    }
    FSVD_CUDA_CHECK(cudaMemcpyAsync(dids, ids.data(), ids.size() * sizeof(int),
                                    cudaMemcpyHostToDevice, s));
    int max_steps = 0;
    for (auto& sp : spans) max_steps = std::max(max_steps, sp.first - 1);
    for (int step = 0; step < max_steps; ++step)
      for (auto& sp : spans) {
        if (step >= sp.first - 1) continue;
        size_t sm_bytes = 0;
        for (int c = 0; c < sp.second.second; ++c) {
          const DevJob& d = dj[ids[sp.second.first + c]];
          sm_bytes = std::max(sm_bytes, static_cast<size_t>(2 * d.w) * d.M * sizeof(double));
        }
        k_visit<<<dim3(sp.first / 2, sp.second.second), kVisitThreads, sm_bytes, s>>>(
            djobs, dids + sp.second.first, step, step == 0);
        check_launch("k_visit");
      }
    ++sweeps;
    FSVD_CUDA_CHECK(cudaMemcpyAsync(rot.data(), base + off_rot, nj * sizeof(unsigned),
                                    cudaMemcpyDeviceToHost, s));
    FSVD_CUDA_CHECK(cudaStreamSynchronize(s));
    for (size_t t = 0; t < nj; ++t)
      if (rot[t] == 0) active[t] = 0;
    FSVD_CUDA_CHECK(cudaMemsetAsync(base + off_rot, 0, nj * sizeof(unsigned), s));
  }
  g_last_sweeps = sweeps;

  // ---- exact norms, descending order, zero factors (svd.cpp:345-366)
  k_colnorms<<<dim3(sms, gy), 256, 0, s>>>(djobs, 0);
  check_launch("k_colnorms");
  std::vector<std::vector<double>> sig(nj);
  for (size_t t = 0; t < nj; ++t) {
    sig[t].resize(dj[t].npad);
    FSVD_CUDA_CHECK(cudaMemcpyAsync(sig[t].data(), dj[t].sigma, dj[t].npad * sizeof(double),
                                    cudaMemcpyDeviceToHost, s));
  }
  FSVD_CUDA_CHECK(cudaStreamSynchronize(s));
  for (size_t t = 0; t < nj; ++t) {
    const DevJob& d = dj[t];
    std::vector<int> order(d.N);
    std::iota(order.begin(), order.end(), 0);
    const std::vector<double>& sg = sig[t];
    std::stable_sort(order.begin(), order.end(), [&](int i, int j) { return sg[i] > sg[j]; });
    const double zero_tol = sg[order[0]] * 1.0e-15;
    std::vector<int> src(d.r);
    std::vector<double> sr(d.r);
    for (int jj = 0; jj < d.r; ++jj) {
      src[jj] = order[jj];
      const double v = sg[order[jj]];
      sr[jj] = (v <= zero_tol || v == 0.0) ? 0.0 : v;
    }
    FSVD_CUDA_CHECK(cudaMemcpyAsync(base + off_src[t], src.data(), d.r * sizeof(int),
                                    cudaMemcpyHostToDevice, s));
    FSVD_CUDA_CHECK(cudaMemcpyAsync(base + off_sr[t], sr.data(), d.r * sizeof(double),
                                    cudaMemcpyHostToDevice, s));
  }
  int maxN = 0, maxr = 0;
  for (const DevJob& d : dj) {
    maxN = std::max(maxN, d.N);
    maxr = std::max(maxr, d.r);
  }
  k_left<<<dim3(sms, gy), 256, 0, s>>>(djobs);
  check_launch("k_left");
  k_right<<<dim3((maxN + kRT - 1) / kRT, (maxr + kRT - 1) / kRT, gy), 256, 0, s>>>(djobs);
  check_launch("k_right");
  k_output<<<dim3(maxr, gy), 256, 0, s>>>(djobs);
  check_launch("k_output");
  for (size_t t = 0; t < nj; ++t) {
    const FactorJob& j = jobs[t];
    FSVD_CUDA_CHECK(cudaMemcpyAsync(j.u, base + off_u[t], j.m * j.r * sizeof(float),
                                    cudaMemcpyDeviceToHost, s));
    FSVD_CUDA_CHECK(cudaMemcpyAsync(j.v, base + off_v[t], j.r * j.n * sizeof(float),
                                    cudaMemcpyDeviceToHost, s));
  }
  FSVD_CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace fsvd
