// simt.cu -- CUDA-core kernels: the fp32 precision policy (<= 1e-4 parity
// mode) and every shape outside the tensor-core tilings, plus the row-wise
// residual+LayerNorm kernel (K5) and dtype conversions.
//
// Storage type T is float or bf16; arithmetic is always fp32.  The attention
// and FFN kernels follow the reference's dataflow literally (head-width tile
// reconstruction with the bias preloaded, online softmax in base e, bias
// after the up-projection GEMM, ascending feature blocks), so the fp32 policy
// reproduces the reference to ~1e-6.
#include <float.h>

#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace fsvd {
namespace {

template <typename T>
__device__ __forceinline__ float ld(const T* p) {
  if constexpr (sizeof(T) == 4) return __ldg(reinterpret_cast<const float*>(p));
  else return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ T cvt(float v) {
  if constexpr (sizeof(T) == 4) return v;
  else return __float2bfloat16(v);
}

// --------------------------------------------------------------------- GEMM
// C[M,N] = A[M,K] B[K,N] (+bias) (act); 64x64 tile, 256 threads, 4x4 per thread.
template <typename T>
__global__ void __launch_bounds__(256) k_simt_gemm(const T* __restrict__ A, int64_t lda,
                                                   const T* __restrict__ B, int64_t ldb,
                                                   T* __restrict__ C, int64_t ldc, int M, int N,
                                                   int K, const float* __restrict__ bias,
                                                   int act) {
  __shared__ float sa[16][64 + 4];
  __shared__ float sb[16][64];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int r = e >> 4, c = e & 15;  // A tile: 64 rows x 16 k
      const int gm = m0 + r, gk = k0 + c;
      sa[c][r] = (gm < M && gk < K) ? ld(A + (int64_t)gm * lda + gk) : 0.0f;
      const int kr = e >> 6, nc = e & 63;  // B tile: 16 k x 64 cols
      const int bk = k0 + kr, bn = n0 + nc;
      sb[kr][nc] = (bk < K && bn < N) ? ld(B + (int64_t)bk * ldb + bn) : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sa[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sb[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float v = acc[i][j];
      if (bias) v += bias[gn];
      C[(int64_t)gm * ldc + gn] = cvt<T>(ptx::apply_act(v, act));
    }
  }
}

// ---------------------------------------------------------------- attention
// Reference dataflow (attention.cpp:249-267, :92-137): per (b, h, 32-row query
// tile) rebuild Q = (b_q + P_q V_q) / sqrt(dh), then for each 32-key tile K, V
// the same way, scores, online softmax (exp), acc += p V, out = acc / l.
constexpr int AQ = 32, AK = 32;

template <typename T>
__global__ void __launch_bounds__(256) k_simt_attention(const T* __restrict__ P, int64_t ldp,
                                                        const T* __restrict__ V,
                                                        const float* __restrict__ bias,
                                                        T* __restrict__ ctx, int seq, int heads,
                                                        int groups, int rank, int d_model) {
  extern __shared__ float sm[];
  const int dh = d_model / heads, gd = d_model / groups, hpg = heads / groups;
  const int qt = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int g = h / hpg, hc = (h % hpg) * dh;
  float* sv = sm;                    // [3][rank][dh]
  float* sq = sv + 3 * rank * dh;    // [AQ][dh]
  float* sk = sq + AQ * dh;          // [AK][dh]
  float* svv = sk + AK * dh;         // [AK][dh]
  float* ss = svv + AK * dh;         // [AQ][AK+1]
  float* sacc = ss + AQ * (AK + 1);  // [AQ][dh]
  float* smax = sacc + AQ * dh;      // [AQ]
  float* ssum = smax + AQ;           // [AQ]
  float* salpha = ssum + AQ;         // [AQ]
  const int tid = threadIdx.x;
  for (int e = tid; e < 3 * rank * dh; e += blockDim.x) {
    const int mat = e / (rank * dh), rr = (e / dh) % rank, dd = e % dh;
    sv[e] = ld(V + ((int64_t)(mat * groups + g) * rank + rr) * gd + hc + dd);
  }
  __syncthreads();
  const float scale = 1.0f / sqrtf(static_cast<float>(dh));
  const int64_t row0 = (int64_t)b * seq;
  const int q0 = qt * AQ;
  // load one reconstructed tile: dst[i][dd] = bias + sum_r P[i][r] V[r][dd]
  auto load = [&](int mat, int t0, int rows, float* dst) {
    const float* vm = sv + mat * rank * dh;
    const float* bm = bias + mat * d_model + g * gd + hc;
    for (int e = tid; e < rows * dh; e += blockDim.x) {
      const int i = e / dh, dd = e % dh;
      float acc = bm[dd];
      const int t = t0 + i;
      if (t < seq) {
        const T* prow = P + (row0 + t) * ldp + (int64_t)(mat * groups + g) * rank;
        for (int rr = 0; rr < rank; ++rr) acc = fmaf(ld(prow + rr), vm[rr * dh + dd], acc);
      }
      dst[i * dh + dd] = acc;
    }
  };
  load(0, q0, AQ, sq);
  for (int e = tid; e < AQ * dh; e += blockDim.x) {
    sq[e] *= scale;
    sacc[e] = 0.0f;
  }
  if (tid < AQ) {
    smax[tid] = -INFINITY;
    ssum[tid] = 0.0f;
  }
  __syncthreads();
  for (int n0 = 0; n0 < seq; n0 += AK) {
    const int nlen = min(AK, seq - n0);
    load(1, n0, AK, sk);
    load(2, n0, AK, svv);
    __syncthreads();
    for (int e = tid; e < AQ * AK; e += blockDim.x) {
      const int i = e / AK, j = e % AK;
      float acc = 0.0f;
      for (int dd = 0; dd < dh; ++dd) acc = fmaf(sq[i * dh + dd], sk[j * dh + dd], acc);
      ss[i * (AK + 1) + j] = acc;
    }
    __syncthreads();
    if (tid < AQ) {
      const int i = tid;
      float tmax = -INFINITY;
      for (int j = 0; j < nlen; ++j) tmax = fmaxf(tmax, ss[i * (AK + 1) + j]);
      const float m_new = fmaxf(smax[i], tmax);
      const float alpha = expf(smax[i] - m_new);
      float part = 0.0f;
      for (int j = 0; j < AK; ++j) {
        const float p = j < nlen ? expf(ss[i * (AK + 1) + j] - m_new) : 0.0f;
        ss[i * (AK + 1) + j] = p;
        part += p;
      }
      ssum[i] = ssum[i] * alpha + part;
      smax[i] = m_new;
      salpha[i] = alpha;
    }
    __syncthreads();
    for (int e = tid; e < AQ * dh; e += blockDim.x) {
      const int i = e / dh, dd = e % dh;
      float acc = sacc[e] * salpha[i];
      for (int j = 0; j < nlen; ++j) acc = fmaf(ss[i * (AK + 1) + j], svv[j * dh + dd], acc);
      sacc[e] = acc;
    }
    __syncthreads();
  }
  for (int e = tid; e < AQ * dh; e += blockDim.x) {
    const int i = e / dh, dd = e % dh;
    if (q0 + i < seq)
      ctx[(row0 + q0 + i) * d_model + h * dh + dd] = cvt<T>(sacc[e] / ssum[i]);
  }
}

// ---------------------------------------------------------------- FFN stream
// Reference dataflow (ffn.cpp:84-104): per 16-row tile, for ascending feature
// blocks h = act(P V_up[:, blk] + b_up[blk]); z += h U_down[blk, :].
// FUSED additionally computes P = X U_up first and out = b_dn + Z V_dn last
// (ffn.cpp:158-185), keeping P and Z in shared memory.
constexpr int FRW = 16;  // rows per CTA
constexpr int FBF = 32;  // features per block

template <typename T, bool FUSED>
__global__ void __launch_bounds__(256) k_simt_ffn(const T* __restrict__ x, const T* __restrict__ p,
                                                  const T* __restrict__ up_u,
                                                  const T* __restrict__ up_v,
                                                  const float* __restrict__ up_b,
                                                  const T* __restrict__ dn_u,
                                                  const T* __restrict__ dn_v,
                                                  const float* __restrict__ dn_b,
                                                  T* __restrict__ z_out, T* __restrict__ out,
                                                  int Tn, int d_model, int rank, int d_ff,
                                                  int act) {
  extern __shared__ float sm[];
  float* sp = sm;                 // [FRW][rank]
  float* sz = sp + FRW * rank;    // [FRW][rank]
  float* sh = sz + FRW * rank;    // [FRW][FBF]
  const int tid = threadIdx.x;
  const int r0 = blockIdx.x * FRW;
  if (FUSED) {
    for (int e = tid; e < FRW * rank; e += blockDim.x) {
      const int i = e / rank, j = e % rank;
      float acc = 0.0f;
      if (r0 + i < Tn)
        for (int k = 0; k < d_model; ++k)
          acc = fmaf(ld(x + (int64_t)(r0 + i) * d_model + k), ld(up_u + (int64_t)k * rank + j), acc);
      sp[e] = acc;
    }
  } else {
    for (int e = tid; e < FRW * rank; e += blockDim.x) {
      const int i = e / rank;
      sp[e] = (r0 + i < Tn) ? ld(p + (int64_t)r0 * rank + e) : 0.0f;
    }
  }
  for (int e = tid; e < FRW * rank; e += blockDim.x) sz[e] = 0.0f;
  __syncthreads();
  for (int f0 = 0; f0 < d_ff; f0 += FBF) {
    const int flen = min(FBF, d_ff - f0);
    for (int e = tid; e < FRW * FBF; e += blockDim.x) {
      const int i = e / FBF, j = e % FBF;
      float acc = 0.0f;
      if (j < flen) {
        for (int k = 0; k < rank; ++k)
          acc = fmaf(sp[i * rank + k], ld(up_v + (int64_t)k * d_ff + f0 + j), acc);
        acc = ptx::apply_act(acc + up_b[f0 + j], act);
      }
      sh[e] = acc;
    }
    __syncthreads();
    for (int e = tid; e < FRW * rank; e += blockDim.x) {
      const int i = e / rank, j = e % rank;
      float acc = sz[e];
      for (int f = 0; f < flen; ++f)
        acc = fmaf(sh[i * FBF + f], ld(dn_u + (int64_t)(f0 + f) * rank + j), acc);
      sz[e] = acc;
    }
    __syncthreads();
  }
  if (!FUSED) {
    for (int e = tid; e < FRW * rank; e += blockDim.x) {
      const int i = e / rank;
      if (r0 + i < Tn) z_out[(int64_t)r0 * rank + e] = cvt<T>(sz[e]);
    }
  } else {
    for (int e = tid; e < FRW * d_model; e += blockDim.x) {
      const int i = e / d_model, j = e % d_model;
      if (r0 + i >= Tn) continue;
      float acc = dn_b[j];
      for (int k = 0; k < rank; ++k) acc = fmaf(sz[i * rank + k], ld(dn_v + (int64_t)k * d_model + j), acc);
      out[(int64_t)(r0 + i) * d_model + j] = cvt<T>(acc);
    }
  }
}

// ---------------------------------------------------------------- K5 LayerNorm
// y = gamma * ((a + b) - mean) / sqrt(var + eps) + beta, one warp per row,
// biased variance (tensor.cpp:88-102).  Rows up to 32*VPL values stay in
// registers; wider rows take the strided path.
// Rows have `pitch` >= d stored columns (the tensor-core layouts pad the
// model dimension with zeros): statistics over the first d, the normalised
// value written to all pitch columns (gamma = beta = 0 in the padding -> 0).
template <typename T, int VPL>
__global__ void k_resid_ln(const T* a, const T* b,
                           const float* __restrict__ gamma, const float* __restrict__ beta,
                           float eps, T* y, int rows, int d, int pitch) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const int64_t base = (int64_t)warp * pitch;
  const float inv_d = 1.0f / static_cast<float>(d);
  if (pitch <= 32 * VPL) {
    float v[VPL];
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = lane + 32 * i;
      v[i] = 0.0f;
      if (c < pitch) v[i] = ld(a + base + c) + (b ? ld(b + base + c) : 0.0f);
      if (c < d) s += v[i];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mean = s * inv_d;
    float q = 0.0f;
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = lane + 32 * i;
      if (c < d) {
        const float t = v[i] - mean;
        q += t * t;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float inv = 1.0f / sqrtf(q * inv_d + eps);
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = lane + 32 * i;
      if (c < pitch) y[base + c] = cvt<T>(gamma[c] * ((v[i] - mean) * inv) + beta[c]);
    }
  } else {
    float s = 0.0f;
    for (int c = lane; c < d; c += 32) s += ld(a + base + c) + (b ? ld(b + base + c) : 0.0f);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mean = s * inv_d;
    float q = 0.0f;
    for (int c = lane; c < d; c += 32) {
      const float t = ld(a + base + c) + (b ? ld(b + base + c) : 0.0f) - mean;
      q += t * t;
    }
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float inv = 1.0f / sqrtf(q * inv_d + eps);
    for (int c = lane; c < pitch; c += 32) {
      const float t = ld(a + base + c) + (b ? ld(b + base + c) : 0.0f);
      y[base + c] = cvt<T>(gamma[c] * ((t - mean) * inv) + beta[c]);
    }
  }
}

// bf16 fast path: d % 8 == 0 and d <= 32 * 8 * V8; each lane owns V8 16-byte
// chunks of the row.
template <int V8>
__global__ void __launch_bounds__(256) k_resid_ln_bf16x8(const bf16* a,
                                                       const bf16* b,
                                                       const float* __restrict__ gamma,
                                                       const float* __restrict__ beta, float eps,
                                                       bf16* y, int rows, int d) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const int64_t base = (int64_t)warp * d;
  const int nch = d >> 3;
  float v[V8][8];
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < V8; ++i) {
    const int c = lane + 32 * i;
#pragma unroll
    for (int k = 0; k < 8; ++k) v[i][k] = 0.0f;
    if (c < nch) {
      const uint4 av = __ldg(reinterpret_cast<const uint4*>(a + base) + c);
      const __nv_bfloat162* ap = reinterpret_cast<const __nv_bfloat162*>(&av);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(ap[k]);
        v[i][2 * k] = f.x;
        v[i][2 * k + 1] = f.y;
      }
      if (b) {
        const uint4 bv = __ldg(reinterpret_cast<const uint4*>(b + base) + c);
        const __nv_bfloat162* bp = reinterpret_cast<const __nv_bfloat162*>(&bv);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(bp[k]);
          v[i][2 * k] += f.x;
          v[i][2 * k + 1] += f.y;
        }
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) s += v[i][k];
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float inv_d = 1.0f / static_cast<float>(d);
  const float mean = s * inv_d;
  float q = 0.0f;
#pragma unroll
  for (int i = 0; i < V8; ++i)
    if (lane + 32 * i < nch)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float t = v[i][k] - mean;
        q = fmaf(t, t, q);
      }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float inv = rsqrtf(q * inv_d + eps);
#pragma unroll
  for (int i = 0; i < V8; ++i) {
    const int c = lane + 32 * i;
    if (c >= nch) continue;
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma) + 2 * c);
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma) + 2 * c + 1);
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(beta) + 2 * c);
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(beta) + 2 * c + 1);
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    const float be[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      w[k] = ptx::pack_bf16(fmaf(g[2 * k], (v[i][2 * k] - mean) * inv, be[2 * k]),
                            fmaf(g[2 * k + 1], (v[i][2 * k + 1] - mean) * inv, be[2 * k + 1]));
    reinterpret_cast<uint4*>(y + base)[c] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <typename T>
__global__ void k_add(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ y,
                      int64_t n) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = cvt<T>(ld(a + i) + ld(b + i));
}

template <typename T>
__global__ void k_convert(const float* __restrict__ src, T* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = cvt<T>(src[i]);
}
template <typename T>
__global__ void k_to_f32(const T* __restrict__ src, float* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = ld(src + i);
}

int elementwise_grid(int64_t n) {
  int64_t g = (n + 255) / 256;
  const int64_t cap = 8LL * num_sms();
  return static_cast<int>(g < cap ? (g > 0 ? g : 1) : cap);
}

template <typename T>
void launch_ln(const T* a, const T* b, const float* gamma, const float* beta, float eps, T* y,
               int rows, int d, cudaStream_t s, int pitch) {
  const int threads = 256;
  const int grid = (rows * 32 + threads - 1) / threads;
  if (pitch <= 0) pitch = d;
  if constexpr (sizeof(T) == 2) {
    if (pitch == d && d % 8 == 0 && d <= 32 * 8 * 4) {
      if (d <= 32 * 8 * 2)
        launch_pdl(k_resid_ln_bf16x8<2>, dim3(grid), dim3(threads), 0, s, a, b, gamma, beta, eps, y,
                   rows, d);
      else
        launch_pdl(k_resid_ln_bf16x8<4>, dim3(grid), dim3(threads), 0, s, a, b, gamma, beta, eps, y,
                   rows, d);
      check_launch("k_resid_ln_bf16x8");
      return;
    }
  }
  // in place (y == a or b) needs the register path: pitch <= 1024
  if (pitch <= 32 * 8)
    k_resid_ln<T, 8><<<grid, threads, 0, s>>>(a, b, gamma, beta, eps, y, rows, d, pitch);
  else if (pitch <= 32 * 24)
    k_resid_ln<T, 24><<<grid, threads, 0, s>>>(a, b, gamma, beta, eps, y, rows, d, pitch);
  else
    k_resid_ln<T, 32><<<grid, threads, 0, s>>>(a, b, gamma, beta, eps, y, rows, d, pitch);
  check_launch("k_resid_ln");
}

}  // namespace

template <typename T>
void simt_gemm(const T* A, int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc, int M, int N,
               int K, const float* bias, int act, cudaStream_t s) {
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  k_simt_gemm<T><<<grid, 256, 0, s>>>(A, lda, B, ldb, C, ldc, M, N, K, bias, act);
  check_launch("k_simt_gemm");
}

template <typename T>
void simt_attention(const AttnSimtArgs& a, cudaStream_t s) {
  const int dh = a.d_model / a.heads;
  const size_t smem =
      sizeof(float) * (3 * a.rank * dh + AQ * dh + 2 * AK * dh + AQ * (AK + 1) + AQ * dh + 3 * AQ);
  static bool attr = false;
  if (!attr) {
    FSVD_CUDA_CHECK(cudaFuncSetAttribute(k_simt_attention<T>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  if (smem > 227 * 1024) throw CudaError("simt_attention: head too large for shared memory");
  dim3 grid((a.seq + AQ - 1) / AQ, a.heads, a.batch);
  k_simt_attention<T><<<grid, 256, smem, s>>>(
      static_cast<const T*>(a.P), 3LL * a.groups * a.rank, static_cast<const T*>(a.v), a.bias,
      static_cast<T*>(a.ctx), a.seq, a.heads, a.groups, a.rank, a.d_model);
  check_launch("k_simt_attention");
}

template <typename T, bool FUSED>
void launch_simt_ffn(const T* x, const T* p, const T* up_u, const T* up_v, const float* up_b,
                     const T* dn_u, const T* dn_v, const float* dn_b, T* z, T* out, int Tn, int d,
                     int rank, int d_ff, int act, cudaStream_t s) {
  const size_t smem = sizeof(float) * (2 * FRW * rank + FRW * FBF);
  if (smem > 227 * 1024) throw CudaError("simt_ffn: FFN rank too large for shared memory");
  static bool attr = false;
  if (!attr) {
    FSVD_CUDA_CHECK(cudaFuncSetAttribute(k_simt_ffn<T, FUSED>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  k_simt_ffn<T, FUSED><<<(Tn + FRW - 1) / FRW, 256, smem, s>>>(x, p, up_u, up_v, up_b, dn_u, dn_v,
                                                               dn_b, z, out, Tn, d, rank, d_ff, act);
  check_launch(FUSED ? "k_simt_ffn_fused" : "k_simt_ffn_stream");
}

template <typename T>
void simt_ffn_stream(const FfnSimtArgs& a, cudaStream_t s) {
  launch_simt_ffn<T, false>(nullptr, static_cast<const T*>(a.p), nullptr,
                            static_cast<const T*>(a.up_v), a.up_b, static_cast<const T*>(a.dn_u),
                            nullptr, nullptr, static_cast<T*>(a.z), nullptr, a.T, 0, a.rank,
                            a.d_ff, a.act, s);
}

template <typename T>
void simt_ffn_fused(const T* x, const T* up_u, const T* up_v, const float* up_b, const T* dn_u,
                    const T* dn_v, const float* dn_b, T* out, int Tn, int d, int rank, int d_ff,
                    int act, cudaStream_t s) {
  launch_simt_ffn<T, true>(x, nullptr, up_u, up_v, up_b, dn_u, dn_v, dn_b, nullptr, out, Tn, d,
                           rank, d_ff, act, s);
}

void resid_layernorm_bf16(const bf16* a, const bf16* b, const float* gamma, const float* beta,
                          float eps, bf16* y, int rows, int d, cudaStream_t s, int pitch) {
  launch_ln<bf16>(a, b, gamma, beta, eps, y, rows, d, s, pitch);
}
void resid_layernorm_f32(const float* a, const float* b, const float* gamma, const float* beta,
                         float eps, float* y, int rows, int d, cudaStream_t s, int pitch) {
  launch_ln<float>(a, b, gamma, beta, eps, y, rows, d, s, pitch);
}
void add_bf16(const bf16* a, const bf16* b, bf16* y, int64_t n, cudaStream_t s) {
  launch_pdl(k_add<bf16>, dim3(elementwise_grid(n)), dim3(256), 0, s, a, b, y, n);
  check_launch("k_add");
}
void add_f32(const float* a, const float* b, float* y, int64_t n, cudaStream_t s) {
  launch_pdl(k_add<float>, dim3(elementwise_grid(n)), dim3(256), 0, s, a, b, y, n);
  check_launch("k_add");
}
template <typename T>
void convert_f32(const float* src, T* dst, int64_t n, cudaStream_t s) {
  k_convert<T><<<elementwise_grid(n), 256, 0, s>>>(src, dst, n);
  check_launch("k_convert");
}
template <typename T>
void to_f32(const T* src, float* dst, int64_t n, cudaStream_t s) {
  k_to_f32<T><<<elementwise_grid(n), 256, 0, s>>>(src, dst, n);
  check_launch("k_to_f32");
}

template void simt_gemm<float>(const float*, int64_t, const float*, int64_t, float*, int64_t, int,
                               int, int, const float*, int, cudaStream_t);
template void simt_gemm<bf16>(const bf16*, int64_t, const bf16*, int64_t, bf16*, int64_t, int, int,
                              int, const float*, int, cudaStream_t);
template void simt_attention<float>(const AttnSimtArgs&, cudaStream_t);
template void simt_attention<bf16>(const AttnSimtArgs&, cudaStream_t);
template void simt_ffn_stream<float>(const FfnSimtArgs&, cudaStream_t);
template void simt_ffn_stream<bf16>(const FfnSimtArgs&, cudaStream_t);
template void simt_ffn_fused<float>(const float*, const float*, const float*, const float*,
                                    const float*, const float*, const float*, float*, int, int, int,
                                    int, int, cudaStream_t);
template void simt_ffn_fused<bf16>(const bf16*, const bf16*, const bf16*, const float*, const bf16*,
                                   const bf16*, const float*, bf16*, int, int, int, int, int,
                                   cudaStream_t);
template void convert_f32<float>(const float*, float*, int64_t, cudaStream_t);
template void convert_f32<bf16>(const float*, bf16*, int64_t, cudaStream_t);
template void to_f32<float>(const float*, float*, int64_t, cudaStream_t);
template void to_f32<bf16>(const bf16*, float*, int64_t, cudaStream_t);

}  // namespace fsvd
