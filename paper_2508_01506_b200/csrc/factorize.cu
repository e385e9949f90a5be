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
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <map>
#include <numeric>
#include <vector>

#include "common.cuh"
#include "errors.hpp"
#include "factorize.hpp"
#include "ptx.cuh"

namespace fsvd {
namespace {

constexpr int kVisitThreads = 256;                // 8 warps
constexpr int kVisitWarps = kVisitThreads / 32;
constexpr int kVisitCtasPerSm = 4;
constexpr size_t kColBytes = 50 * 1024;           // staged columns per visit CTA
constexpr double kPairTol = 1.0e-15;              // svd.cpp:22
constexpr int kMaxSweeps = 60;                    // svd.cpp:23
constexpr int kMaxW = 16;
constexpr int kMaxCluster = 8;

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
  int ld;                       // column stride of `work` (M padded to a multiple of 2 cs)
  int cs, mc;                   // visit cluster size, rows per cluster CTA (ld / cs)
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
  const size_t total = static_cast<size_t>(J.ld) * J.npad;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(e / J.ld), i = static_cast<int>(e % J.ld);
    J.work[e] = (j < J.N && i < J.M) ? op_at(J, i, j) : 0.0;
  }
}

// Column norms^2 (warp per column); `max_only` folds them into J.maxsq,
// otherwise sigma[j] = sqrt(norm^2) for every padded column.
__global__ void k_colnorms(const DevJob* jobs, int max_only) {
  const DevJob& J = jobs[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  for (int j = blockIdx.x * wpb + warp; j < J.npad; j += gridDim.x * wpb) {
    const double* c = J.work + static_cast<size_t>(j) * J.ld;
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

// One block-pair visit.  A cluster of cs CTAs shares the visit, each holding
// mc = ld / cs consecutive ROWS of the 2w staged columns: dot products are
// per-CTA partial sums exchanged through distributed shared memory and added
// in rank order (so every CTA derives the same rotation), rotations are
// applied to the local rows.  Column norms^2 are summed exactly at visit
// start and then updated by the rotation identities (svd.cpp:85-87).
// Small slices (<= 50 KB) keep four visit CTAs resident per SM: a round is a
// short latency chain (dot, reduction, exchange, rotation), so throughput
// comes from several visits interleaving on an SM.  Warps own one column
// pair per round (w <= 8: G = 8/w warps share a pair; w > 8: a warp
// interleaves two pairs).  blockIdx.x / cs = pair slot of step `step`;
// blockIdx.y indexes `ids` (the active jobs of one (nb, cs) class).
__global__ void __launch_bounds__(kVisitThreads, kVisitCtasPerSm)
    k_visit(const DevJob* jobs, const int* ids, int step, int full) {
  const DevJob& J = jobs[ids[blockIdx.y]];
  const int cs = J.cs;
  const int rank = cs > 1 ? static_cast<int>(ptx::cluster_rank()) : 0;
  const int L = J.nb - 1, k = blockIdx.x / cs, w = J.w, M = J.mc;  // rows held here
  const int bp = k == 0 ? step : (step + k) % L;
  const int bq = k == 0 ? L : (step - k + L) % L;
  const size_t row0 = static_cast<size_t>(rank) * M;
  extern __shared__ __align__(128) double cols[];
  __shared__ double red[kVisitWarps][2];
  __shared__ double cred[2][kMaxCluster][kMaxW];   // [round parity][source rank][slot]
  __shared__ double cnorm[kMaxCluster][2 * kMaxW];
  __shared__ double sqn[2 * kMaxW];
  __shared__ uint64_t landed;
  const uint32_t col_bytes = static_cast<uint32_t>(M * sizeof(double));
  auto sync_all = [&]() {
    if (cs > 1) ptx::cluster_sync_all(); else __syncthreads();
  };
  // value v into slot `idx` of array `arr` ([kMaxCluster][width]) of every CTA
  auto broadcast = [&](double* arr, int width, int idx, double v) {
    const uint32_t local = ptx::smem_u32(arr + rank * width + idx);
    for (int dst = 0; dst < cs; ++dst)
      asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ptx::mapa_shared(local, dst)), "d"(v)
                   : "memory");
  };

  // the 2w column slices arrive by bulk copies (one thread issues, all wait)
  if (threadIdx.x == 0) {
    ptx::mbar_init(&landed, 1);
    ptx::fence_barrier_init();
    ptx::mbar_arrive_expect_tx(&landed, 2 * w * col_bytes);
    for (int c = 0; c < 2 * w; ++c) {
      const int gc = c < w ? bp * w + c : bq * w + (c - w);
      ptx::bulk_load(cols + c * M, J.work + static_cast<size_t>(gc) * J.ld + row0, col_bytes,
                     &landed);
    }
  }
  // every CTA of the cluster is resident (and its barrier initialised) before
  // any distributed-shared-memory store below
#ifdef FSVD_TRACE
  const bool tr = blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0;
  long long tt0 = clock64(), tt1 = 0, tacc[5] = {0, 0, 0, 0, 0};
#define FAC_T(i) do { if (tr) { const long long n_ = clock64(); tacc[i] += n_ - tt1; tt1 = n_; } } while (0)
#else
#define FAC_T(i) do { } while (0)
#endif
  sync_all();
  ptx::mbar_wait(&landed, 0);
#ifdef FSVD_TRACE
  if (tr) { tt1 = clock64(); printf("[visit] cs %d w %d M %d load %lld\n", cs, w, M, tt1 - tt0); }
#endif

  const double floor_sq = __longlong_as_double(static_cast<long long>(*J.maxsq)) * 1.0e-30;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M2 = M / 2;  // rows as double2 (mc is even)
  const double2* cols2c = reinterpret_cast<const double2*>(cols);
  double2* cols2 = reinterpret_cast<double2*>(cols);

  // exact norms^2 of the staged columns, summed over the cluster
  for (int c = warp; c < 2 * w; c += kVisitWarps) {
    const double2* x = cols2c + c * M2;
    double a0 = 0.0, a1 = 0.0;
    for (int i = lane; i < M2; i += 32) {
      a0 = fma(x[i].x, x[i].x, a0);
      a1 = fma(x[i].y, x[i].y, a1);
    }
    const double a = warp_sum(a0 + a1);
    if (lane == 0) broadcast(&cnorm[0][0], 2 * kMaxW, c, a);
  }
  sync_all();
  if (threadIdx.x < 2 * w) {
    double a = 0.0;
    for (int rr = 0; rr < cs; ++rr) a += cnorm[rr][threadIdx.x];
    sqn[threadIdx.x] = a;
  }
  __syncthreads();
  FAC_T(4);

  // pair ownership
  const int G = w >= kVisitWarps ? 1 : kVisitWarps / w;  // warps per pair
  const int P = w > kVisitWarps ? 2 : 1;                  // pairs per warp
  const int slot0 = warp / G, gw = warp % G;
  const int gt = gw * 32 + lane, gthreads = G * 32;
  unsigned nrot = 0;
  const int rounds = full ? 2 * w - 1 : w;
  for (int t = 0; t < rounds; ++t) {
    int p[2] = {-1, -1}, q[2] = {-1, -1};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int slot = slot0 + e * kVisitWarps;
      if (e >= P || slot >= w || (G > 1 && slot0 >= w)) continue;
      if (full) {  // circle method over all 2w staged columns
        const int L2 = 2 * w - 1;
        p[e] = slot == 0 ? t : (t + slot) % L2;
        q[e] = slot == 0 ? L2 : (t - slot + L2) % L2;
      } else {     // cross pairs only
        p[e] = slot;
        q[e] = w + (slot + t) % w;
      }
    }
    // partial dot products of this CTA's rows (both pairs interleaved)
    {
      double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      const double2* a0 = cols2c + max(p[0], 0) * M2;
      const double2* b0 = cols2c + max(q[0], 0) * M2;
      const double2* a1 = cols2c + max(p[1], 0) * M2;
      const double2* b1 = cols2c + max(q[1], 0) * M2;
      if (p[1] >= 0) {
#pragma unroll 2
        for (int i = gt; i < M2; i += gthreads) {
          const double2 x0 = a0[i], y0 = b0[i], x1 = a1[i], y1 = b1[i];
          c[0][0] = fma(x0.x, y0.x, c[0][0]);
          c[0][1] = fma(x0.y, y0.y, c[0][1]);
          c[1][0] = fma(x1.x, y1.x, c[1][0]);
          c[1][1] = fma(x1.y, y1.y, c[1][1]);
        }
      } else if (p[0] >= 0) {
#pragma unroll 4
        for (int i = gt; i < M2; i += gthreads) {
          const double2 x0 = a0[i], y0 = b0[i];
          c[0][0] = fma(x0.x, y0.x, c[0][0]);
          c[0][1] = fma(x0.y, y0.y, c[0][1]);
        }
      }
      const double s0 = warp_sum(c[0][0] + c[0][1]);
      const double s1 = warp_sum(c[1][0] + c[1][1]);
      if (lane == 0) {
        red[warp][0] = s0;
        red[warp][1] = s1;
      }
    }
    FAC_T(0);
    __syncthreads();
    const int buf = t & 1;
    // one thread per slot sums its warps and broadcasts the CTA partial
    if (threadIdx.x < w) {
      const int slot = threadIdx.x;
      const int e = slot >= kVisitWarps ? 1 : 0;
      const int w0 = (slot - e * kVisitWarps) * G;
      double v = 0.0;
      for (int g = 0; g < G; ++g) v += red[w0 + g][e];
      broadcast(&cred[buf][0][0], kMaxW, slot, v);
    }
    sync_all();
    FAC_T(1);
    double np[2] = {-1.0, -1.0}, nq[2] = {0.0, 0.0};  // norms after this round
    double rc[2] = {1.0, 1.0}, rs[2] = {0.0, 0.0};
    bool act[2] = {false, false};
    // rotation parameters of both pairs first (independent latency chains):
    // the reference's small-angle rotation (svd.cpp:65-70) in the algebraically
    // equal form t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2))
    //              = 2c sign(d) / (|d| + sqrt(d^2 + 4c^2)),  d = |q|^2 - |p|^2
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (p[e] < 0) continue;
      const int slot = slot0 + e * kVisitWarps;
      double c = 0.0;
      for (int rr = 0; rr < cs; ++rr) c += cred[buf][rr][slot];
      const double sp = sqn[p[e]], sq = sqn[q[e]];
      const bool live = sp > floor_sq && sq > floor_sq;
      if (!live || c * c <= kPairTol * kPairTol * (sp * sq)) continue;
      const double d = sq - sp;
      const double tn = copysign(2.0 * c, d == 0.0 ? c : d * c) /
                        (fabs(d) + sqrt(fma(d, d, 4.0 * c * c)));
      rc[e] = rsqrt(fma(tn, tn, 1.0));
      rs[e] = rc[e] * tn;
      np[e] = fmax(sp - tn * c, 0.0);
      nq[e] = sq + tn * c;
      act[e] = true;
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (!act[e]) continue;
      const double cs_ = rc[e], sn = rs[e];
      double2* cp = cols2 + p[e] * M2;
      double2* cq = cols2 + q[e] * M2;
#pragma unroll 4
      for (int i = gt; i < M2; i += gthreads) {
        const double2 xp = cp[i], xq = cq[i];
        cp[i] = make_double2(cs_ * xp.x - sn * xq.x, cs_ * xp.y - sn * xq.y);
        cq[i] = make_double2(sn * xp.x + cs_ * xq.x, sn * xp.y + cs_ * xq.y);
      }
      ++nrot;
    }
    FAC_T(2);
    __syncthreads();  // every thread has read sqn[] of this round
    if (gt == 0) {
#pragma unroll
      for (int e = 0; e < 2; ++e)
        if (np[e] >= 0.0) {
          sqn[p[e]] = np[e];
          sqn[q[e]] = nq[e];
        }
    }
    FAC_T(3);
  }
#ifdef FSVD_TRACE
  if (tr) printf("[visit] rounds %d dots %lld xchg %lld rot %lld tail %lld norms %lld total %lld\n", rounds,
                 tacc[0], tacc[1], tacc[2], tacc[3], tacc[4], clock64() - tt0);
#endif

  if (rank == 0 && gt == 0 && nrot) atomicAdd(J.rot, nrot);
  // rotated slices leave by bulk stores (generic writes fenced to the async proxy)
  ptx::fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int c = 0; c < 2 * w; ++c) {
      const int gc = c < w ? bp * w + c : bq * w + (c - w);
      ptx::bulk_store(J.work + static_cast<size_t>(gc) * J.ld + row0, cols + c * M, col_bytes);
    }
    ptx::tma_store_commit();
    ptx::tma_store_wait<0>();
  }
  // no CTA may leave while a peer can still write into its shared memory
  if (cs > 1) ptx::cluster_sync_all();
}

// x[:, jj] = work[:, src[jj]] / sigma (zero factor: 0).
__global__ void k_left(const DevJob* jobs) {
  const DevJob& J = jobs[blockIdx.y];
  const size_t total = static_cast<size_t>(J.M) * J.r;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int jj = static_cast<int>(e / J.M), i = static_cast<int>(e % J.M);
    const double s = J.sr[jj];
    J.x[e] = s > 0.0 ? J.work[static_cast<size_t>(J.src[jj]) * J.ld + i] / s : 0.0;
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
    if ((std::max(j.m, j.n) + 2 * kMaxCluster) * 2 * sizeof(double) > kColBytes * kMaxCluster)
      fail(Kind::Config, "matrix dimension " + std::to_string(std::max(j.m, j.n)) +
                             " exceeds the device factorizer's column budget (" +
                             std::to_string(kColBytes * kMaxCluster / 16 - 2 * kMaxCluster) + ")");
  }
  g_last_sweeps = 0;
  if (jobs.empty()) return;

  // FSVD_FACTOR_PROFILE=1: phase wall times on stderr (developer aid)
  const bool prof = std::getenv("FSVD_FACTOR_PROFILE") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* what, cudaStream_t st) {
    if (!prof) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[factorize] %-10s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
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
    // widest block (<= 16 columns) whose 2w-column slices fit one CTA per
    // cluster rank, smallest cluster first
    d.w = 0;
    for (int w = std::min(kMaxW, std::max(1, (d.N + 1) / 2)); w >= 1 && !d.w; --w)
      for (int cs = 1; cs <= kMaxCluster; cs *= 2) {
        const int ld = (d.M + 2 * cs - 1) / (2 * cs) * (2 * cs);
        if (static_cast<size_t>(2 * w) * (ld / cs) * sizeof(double) <= kColBytes) {
          d.w = w;
          d.cs = cs;
          d.ld = ld;
          d.mc = ld / cs;
          break;
        }
      }
    d.nb = (d.N + d.w - 1) / d.w;
    d.nb += d.nb & 1;
    d.npad = d.nb * d.w;
    off_a[t] = bytes;   bytes += al(j.m * j.n * sizeof(float));
    off_w[t] = bytes;   bytes += al(static_cast<size_t>(d.ld) * d.npad * sizeof(double));
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

  phase("upload", s);
  const int sms = num_sms();
  const unsigned gy = static_cast<unsigned>(nj);
  k_widen<<<dim3(2 * sms, gy), 256, 0, s>>>(djobs);
  check_launch("k_widen");
  k_colnorms<<<dim3(sms, gy), 256, 0, s>>>(djobs, 1);
  check_launch("k_colnorms");

  // ---- Jacobi sweeps, jobs grouped by block count so each launch is dense
  size_t smem = 0;
  for (const DevJob& d : dj)
    smem = std::max(smem, static_cast<size_t>(2 * d.w) * d.mc * sizeof(double));
  FSVD_CUDA_CHECK(cudaFuncSetAttribute(k_visit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
  phase("widen", s);
  std::vector<char> active(nj, 1);
  std::vector<unsigned> rot(nj);
  int sweeps = 0;
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    std::map<std::pair<int, int>, std::vector<int>> classes;  // (nb, cs) -> active job ids
    for (size_t t = 0; t < nj; ++t)
      if (active[t] && dj[t].nb >= 2)
        classes[{dj[t].nb, dj[t].cs}].push_back(static_cast<int>(t));
    if (classes.empty()) break;
    std::vector<int> ids;
    struct Span { int nb, cs, off, count; };
    std::vector<Span> spans;
    for (auto& kv : classes) {
      spans.push_back({kv.first.first, kv.first.second, static_cast<int>(ids.size()),
                       static_cast<int>(kv.second.size())});
      ids.insert(ids.end(), kv.second.begin(), kv.second.end());
    }
    FSVD_CUDA_CHECK(cudaMemcpyAsync(dids, ids.data(), ids.size() * sizeof(int),
                                    cudaMemcpyHostToDevice, s));
    int max_steps = 0;
    for (const Span& sp : spans) max_steps = std::max(max_steps, sp.nb - 1);
    for (int step = 0; step < max_steps; ++step)
      for (const Span& sp : spans) {
        if (step >= sp.nb - 1) continue;
        size_t sm_bytes = 0;
        for (int c = 0; c < sp.count; ++c) {
          const DevJob& d = dj[ids[sp.off + c]];
          sm_bytes = std::max(sm_bytes, static_cast<size_t>(2 * d.w) * d.mc * sizeof(double));
        }
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(sp.cs);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(static_cast<unsigned>(sp.nb / 2 * sp.cs), static_cast<unsigned>(sp.count));
        cfg.blockDim = dim3(kVisitThreads);
        cfg.dynamicSmemBytes = sm_bytes;
        cfg.stream = s;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        FSVD_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_visit, static_cast<const DevJob*>(djobs),
                                           static_cast<const int*>(dids + sp.off), step,
                                           static_cast<int>(step == 0)));
        check_launch("k_visit");
      }
    ++sweeps;
    FSVD_CUDA_CHECK(cudaMemcpyAsync(rot.data(), base + off_rot, nj * sizeof(unsigned),
                                    cudaMemcpyDeviceToHost, s));
    FSVD_CUDA_CHECK(cudaStreamSynchronize(s));
    for (size_t t = 0; t < nj; ++t)
      if (rot[t] == 0) active[t] = 0;
    FSVD_CUDA_CHECK(cudaMemsetAsync(base + off_rot, 0, nj * sizeof(unsigned), s));
    phase("sweep", s);
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
  phase("order", s);
  k_left<<<dim3(sms, gy), 256, 0, s>>>(djobs);
  check_launch("k_left");
  k_right<<<dim3((maxN + kRT - 1) / kRT, (maxr + kRT - 1) / kRT, gy), 256, 0, s>>>(djobs);
  check_launch("k_right");
  k_output<<<dim3(maxr, gy), 256, 0, s>>>(djobs);
  check_launch("k_output");
  phase("finalize", s);
  for (size_t t = 0; t < nj; ++t) {
    const FactorJob& j = jobs[t];
    FSVD_CUDA_CHECK(cudaMemcpyAsync(j.u, base + off_u[t], j.m * j.r * sizeof(float),
                                    cudaMemcpyDeviceToHost, s));
    FSVD_CUDA_CHECK(cudaMemcpyAsync(j.v, base + off_v[t], j.r * j.n * sizeof(float),
                                    cudaMemcpyDeviceToHost, s));
  }
  FSVD_CUDA_CHECK(cudaStreamSynchronize(s));
  phase("download", s);
}

}  // namespace fsvd
