// decode.cu -- rank-space KV cache and single-token decode attention
// (the cache the paper's decoder analysis sizes at
// 2 * layers * B * M * r elements, planner.cpp:123-141 / PAPER.md "Decoder
// Memory Cost Analysis").
//
// The cache of one layer is token-major [B, max_seq, 2*G*rp] bf16: for every
// token the group-projected keys P_k (G blocks of rp) then values P_v -- the
// same column block [k_off, v_off + G*rp) the K1 projection writes, so a
// prefill stores it with one strided copy and a decode step appends one row
// per sequence.  Scores stay in rank space exactly as in K2 (Qt already
// carries V_q V_k^T, 1/sqrt(dh) and log2 e; V_v is folded into the output
// projection), so decode attention is a dot of rp-vectors and an rp-wide
// weighted sum per cached token: HBM-bound on the cache read.
//
// k_attn_decode: grid (B*H, splits); a CTA scores one chunk of the cache for
// one (sequence, head) -- scores to shared memory, chunk max, p = 2^(s - m),
// l and O = sum p * P_v in fp32 -- and writes (m, l, O) partials;
// the last CTA of each (sequence, head) to finish merges the splits
// (max-rescaled sums, in split order) into the rank-space output row
// [B, H*rp] consumed by the out-projection + LN1.
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace fsvd {
namespace {

constexpr int kDecThreads = 128;
constexpr int kDecChunk = 512;  // cache rows per CTA (scores staged in smem)

__device__ __forceinline__ float bf2f(uint16_t v) { return __uint_as_float(uint32_t(v) << 16); }

// rows [0, rows) of src (row stride lds elements, rp-wide blocks [c0, c0 +
// width)) -> cache rows b * max_seq + pos0 + m for src row b * rows_per_b + m
__global__ void k_kv_store(const bf16* __restrict__ src, int64_t lds, int c0, int width,
                           int batch, int rows_per_b, bf16* __restrict__ cache, int max_seq,
                           int pos0, const int* __restrict__ pos_dev) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  if (pos_dev) pos0 = *pos_dev;  // graph replay: the position lives on the device
  const int vec = width / 8;  // uint4 per row
  const int64_t total = (int64_t)batch * rows_per_b * vec;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int v = static_cast<int>(e % vec);
    const int64_t r = e / vec;
    const int b = static_cast<int>(r / rows_per_b), m = static_cast<int>(r % rows_per_b);
    const uint4 x = *reinterpret_cast<const uint4*>(src + r * lds + c0 + v * 8);
    *reinterpret_cast<uint4*>(cache + ((int64_t)b * max_seq + pos0 + m) * width + v * 8) = x;
  }
}

template <int RP>
__global__ void __launch_bounds__(kDecThreads)
    k_attn_decode(const bf16* __restrict__ qkv, int64_t ldq, int q_off, const bf16* __restrict__ cache,
                  int max_seq, int heads, int groups, int len, int splits, float* __restrict__ part,
                  bf16* __restrict__ out, int64_t ldo, const int* __restrict__ pos_dev,
                  unsigned* __restrict__ arrivals) {
  const int bh = blockIdx.x, b = bh / heads, h = bh % heads, g = h / (heads / groups);
  ptx::pdl_trigger();
  ptx::pdl_wait();
  if (pos_dev) len = *pos_dev + 1;
  const int chunk = (len + splits - 1) / splits;
  const int k0 = blockIdx.y * chunk, k1 = min(len, k0 + chunk);
  const int width = 2 * groups * RP;
  const bf16* kbase = cache + (int64_t)b * max_seq * width + g * RP;
  const bf16* vbase = kbase + groups * RP;
  // The new token (position len - 1) is read from the projection rows, not
  // the cache: this kernel also appends it (the first head of each group,
  // split 0 writes the group's K and V rows), so no reader races the write.
  const int pos = len - 1;
  const bf16* knew = qkv + (int64_t)b * ldq + q_off + heads * RP + g * RP;
  const bf16* vnew = knew + groups * RP;
  if (blockIdx.y == 0 && h % (heads / groups) == 0 && threadIdx.x < 2 * (RP / 8)) {
    const int half = threadIdx.x / (RP / 8), v8 = threadIdx.x % (RP / 8);
    const uint4 x = reinterpret_cast<const uint4*>(half ? vnew : knew)[v8];
    bf16* dst = const_cast<bf16*>(half ? vbase : kbase) + (int64_t)pos * width;
    reinterpret_cast<uint4*>(dst)[v8] = x;
  }
  __shared__ float q[RP];
  __shared__ float sc[kDecChunk];
  __shared__ float wred[kDecThreads / 32];
  __shared__ float ored[kDecThreads / 32][RP];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < RP)
    q[tid] = bf2f(reinterpret_cast<const uint16_t*>(qkv)[(int64_t)b * ldq + q_off + h * RP + tid]);
  __syncthreads();

  // scores of this chunk (one cache row per thread per pass)
  float mx = -INFINITY;
  for (int j = k0 + tid; j < k1; j += kDecThreads) {
    const uint4* kr = reinterpret_cast<const uint4*>(j == pos ? knew : kbase + (int64_t)j * width);
    float s = 0.0f;
#pragma unroll
    for (int v = 0; v < RP / 8; ++v) {
      const uint4 u = kr[v];
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        s = fmaf(q[8 * v + 2 * e], __uint_as_float(w4[e] << 16), s);
        s = fmaf(q[8 * v + 2 * e + 1], __uint_as_float(w4[e] & 0xffff0000u), s);
      }
    }
    sc[j - k0] = s;
    mx = fmaxf(mx, s);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) wred[warp] = mx;
  __syncthreads();
  float m = wred[0];
#pragma unroll
  for (int w = 1; w < kDecThreads / 32; ++w) m = fmaxf(m, wred[w]);
  __syncthreads();  // wred is reused for the sums

  // p = 2^(s - m); l = sum p; O = sum p * P_v  (lanes own rows, RP accumulators)
  float l = 0.0f, o[RP];
#pragma unroll
  for (int c = 0; c < RP; ++c) o[c] = 0.0f;
  for (int j = k0 + tid; j < k1; j += kDecThreads) {
    const float p = exp2f(sc[j - k0] - m);
    l += p;
    const uint4* vr = reinterpret_cast<const uint4*>(j == pos ? vnew : vbase + (int64_t)j * width);
#pragma unroll
    for (int v = 0; v < RP / 8; ++v) {
      const uint4 u = vr[v];
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        o[8 * v + 2 * e] = fmaf(p, __uint_as_float(w4[e] << 16), o[8 * v + 2 * e]);
        o[8 * v + 2 * e + 1] = fmaf(p, __uint_as_float(w4[e] & 0xffff0000u), o[8 * v + 2 * e + 1]);
      }
    }
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    l += __shfl_xor_sync(0xffffffffu, l, off);
#pragma unroll
    for (int c = 0; c < RP; ++c) o[c] += __shfl_xor_sync(0xffffffffu, o[c], off);
  }
  if (lane == 0) {
    wred[warp] = l;
#pragma unroll
    for (int c = 0; c < RP; ++c) ored[warp][c] = o[c];
  }
  __syncthreads();
  if (tid < RP) {
    float oc = 0.0f, lt = 0.0f;
#pragma unroll
    for (int w = 0; w < kDecThreads / 32; ++w) {
      oc += ored[w][tid];
      lt += wred[w];
    }
    if (splits == 1) {
      out[(int64_t)b * ldo + h * RP + tid] = __float2bfloat16_rn(oc / lt);
    } else {
      float* pp = part + ((int64_t)bh * splits + blockIdx.y) * (RP + 2);
      pp[2 + tid] = oc;
      if (tid == 0) {
        pp[0] = m;
        pp[1] = lt;
      }
    }
  }
  if (splits == 1) return;
  // the last split CTA of this (sequence, head) merges the partials (in split
  // order, whichever CTA arrives last) and re-arms the arrival counter
  __shared__ int last;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    last = atomicAdd(&arrivals[bh], 1u) == static_cast<unsigned>(splits - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (tid < RP) {
    const volatile float* pp = part + (int64_t)bh * splits * (RP + 2);
    float mm = -INFINITY;
    for (int sp = 0; sp < splits; ++sp) mm = fmaxf(mm, pp[sp * (RP + 2)]);
    float l = 0.0f, o = 0.0f;
    for (int sp = 0; sp < splits; ++sp) {
      const volatile float* qp = pp + sp * (RP + 2);
      const float w = qp[1] > 0.0f ? exp2f(qp[0] - mm) : 0.0f;  // empty chunks carry l = 0
      l = fmaf(w, qp[1], l);
      o = fmaf(w, qp[2 + tid], o);
    }
    out[(int64_t)b * ldo + h * RP + tid] = __float2bfloat16_rn(o / l);
  }
  if (tid == 0) arrivals[bh] = 0u;
}

template <int RP>
void launch_decode(const DecodeArgs& a, cudaStream_t s) {
  const int bh = a.batch * a.heads;
  unsigned* arrivals = reinterpret_cast<unsigned*>(a.part + (size_t)bh * a.splits * (RP + 2));
  if (a.splits > 1) FSVD_CUDA_CHECK(cudaMemsetAsync(arrivals, 0, bh * sizeof(unsigned), s));
  launch_pdl(k_attn_decode<RP>, dim3(bh, a.splits), dim3(kDecThreads), 0, s, a.qkv, a.ldq,
             a.q_off, a.cache, a.max_seq, a.heads, a.groups, a.len, a.splits, a.part, a.out, a.ldo,
             a.pos_dev, arrivals);
  check_launch("k_attn_decode");
}

__global__ void k_set_int(int* p, int v) { *p = v; }

// z[i] = bf16(sum_s part[s][i]), splits summed in order
__global__ void k_z_partial_sum(const float* __restrict__ part, int splits, int64_t n,
                                bf16* __restrict__ z) {
  ptx::pdl_trigger();
  ptx::pdl_wait();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.0f;
    for (int sp = 0; sp < splits; ++sp) acc += part[sp * n + i];
    z[i] = __float2bfloat16_rn(acc);
  }
}

}  // namespace

void z_partial_sum_bf16(const float* part, int splits, int64_t n, bf16* z, cudaStream_t s) {
  const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 4 * num_sms()));
  launch_pdl(k_z_partial_sum, dim3(grid), dim3(256), 0, s, part, splits, n, z);
  check_launch("k_z_partial_sum");
}

void set_device_int(int* p, int v, cudaStream_t s) {
  k_set_int<<<1, 1, 0, s>>>(p, v);
  check_launch("k_set_int");
}

int decode_splits(int batch, int heads, int len) {
  // enough CTAs for two per SM, chunks no longer than the score staging
  const int want = (2 * num_sms() + batch * heads - 1) / (batch * heads);
  const int need = (len + kDecChunk - 1) / kDecChunk;
  const int most = (len + 63) / 64;
  return std::max(need, std::min(want, most));
}

size_t decode_partial_bytes(int batch, int heads, int rank_pad, int max_len) {
  return (size_t)batch * heads * decode_splits(batch, heads, max_len) * (rank_pad + 2) *
             sizeof(float) +
         (size_t)batch * heads * sizeof(unsigned);  // split arrival counters
}

void kv_store_bf16(const bf16* src, int64_t lds, int c0, int width, int batch, int rows_per_b,
                   bf16* cache, int max_seq, int pos0, const int* pos_dev, cudaStream_t s) {
  const int64_t total = (int64_t)batch * rows_per_b * (width / 8);
  const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 4 * num_sms()));
  launch_pdl(k_kv_store, dim3(grid), dim3(256), 0, s, src, lds, c0, width, batch, rows_per_b,
             cache, max_seq, pos0, pos_dev);
  check_launch("k_kv_store");
}

void attn_decode_bf16(const DecodeArgs& a, cudaStream_t s) {
  switch (a.rank_pad) {
    case 16: launch_decode<16>(a, s); break;
    case 32: launch_decode<32>(a, s); break;
    case 64: launch_decode<64>(a, s); break;
    default: throw CudaError("attn_decode_bf16: unsupported rank padding");
  }
}

}  // namespace fsvd
