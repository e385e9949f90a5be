// ln_epi.cuh -- residual + LayerNorm epilogue shared by the row-complete
// tensor-core kernels (K6 k_gemm_ln, K4 k_ffn with the fused LN2).
//
// The producing MMA writes 64-column pieces of a 128-row output tile into a
// double-buffered TMEM accumulator (columns [0, 64) and [64, 128)).  For each
// piece the epilogue (8 warps, two per TMEM lane quadrant, each owning 32 of
// the 64 columns) adds the bias, rounds to bf16 -- the value the unfused
// pipeline stores for the sublayer output --, adds the bf16 residual in fp32
// and accumulates shifted row sums of that fp32 sum s.  s itself is parked in
// TMEM as bf16, two per 32-bit column at [128, 128 + N/2), so the whole row
// stays on chip.  Once every piece is in, the two half-row statistics are
// merged (Chan's pairwise update; biased variance, eps inside the square
// root, tensor.cpp:88-102) and a second sweep over the parked values writes
// y = gamma * ((s - mean) * rstd) + beta.  The statistics are exact fp32;
// only the value being normalised carries one extra bf16 rounding (<= 2^-9
// relative), well inside the bf16 policy's tolerance.
//
// Memory traffic is all bulk/asynchronous: a dedicated producer warp TMA-loads
// the residual as [128 x 64] bf16 SW128 boxes into a two-box ring; in the
// second sweep the same two boxes stage the normalised output for TMA stores,
// and gamma / beta are staged once in shared memory the kernel no longer
// needs.  Every CTA visits the pieces in a rotated order (piece_of), so the
// 128 CTAs of a launch do not all read the same weight lines at once.
#pragma once

#include "ptx.cuh"

namespace fsvd {
namespace lnepi {

using namespace ptx;

constexpr int PN = 64;            // output columns per piece
constexpr int kPark = 2 * PN;     // first TMEM column of the parked values
constexpr int kEpiThreads = 256;
constexpr int kMaxN = 2 * (512 - kPark);

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const __nv_bfloat162* p = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 t = __bfloat1622float2(p[k]);
    f[2 * k] = t.x;
    f[2 * k + 1] = t.y;
  }
}
__device__ __forceinline__ float2 unpack_bf16(uint32_t w) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&w);
  return __bfloat1622float2(h);
}
// 32 residual values (16 bf16 pairs) of `row`, columns [half*32, half*32+32)
// of one [128 x 64] SW128 box at shared address `box`.
__device__ __forceinline__ void load_res32(uint32_t box, uint32_t row, uint32_t half,
                                           uint32_t (&r)[16]) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[4 * k]), "=r"(r[4 * k + 1]), "=r"(r[4 * k + 2]), "=r"(r[4 * k + 3])
                 : "r"(box + swz_offset(row, half * 4 + k, 128)));
}
// bf16x2 -> float2 (exact: bf16 is the top half of an fp32)
__device__ __forceinline__ float2 bf2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
__device__ __forceinline__ uint32_t pack2(float2 v) { return pack_bf16(v.x, v.y); }

// Hands a residual box back to the TMA producer.  The generic-proxy reads of
// the box must be complete and ordered before the next TMA (async-proxy)
// write into it: without the proxy fence the arrive was observed to overtake
// the in-flight LDS and the refill raced the read.
__device__ __forceinline__ void release_box(uint64_t* empty) {
  fence_proxy_async_smem();
  mbar_arrive(empty);
}

// Column piece handled at step i by this CTA (rotated per CTA).
__device__ __forceinline__ int piece_of(int i, int NP) {
  const int j = i + static_cast<int>(blockIdx.x % NP);
  return j >= NP ? j - NP : j;
}

// Residual producer (one thread): streams the [128 x N] residual tile at row
// m0, piece order piece_of(), through a ring of `depth` 16 KB boxes.
__device__ __forceinline__ void produce_residual(const CUtensorMap* tm, uint8_t* ring,
                                                 uint64_t* full, uint64_t* empty, int depth,
                                                 int N, int m0) {
  const int NP = N / PN;
  for (int i = 0; i < NP; ++i) {
    const int slot = i % depth;
    mbar_wait(&empty[slot], ((i / depth) & 1) ^ 1);
    mbar_arrive_expect_tx(&full[slot], 128 * 128);
    tma_load_2d(tm, &full[slot], ring + slot * 128 * 128, piece_of(i, NP) * PN, m0);
  }
}

// Runs in all 256 epilogue threads.  `warp_in_epi` = 0..7 (two per lane
// quadrant, quadrant = hardware warp id % 4), `row` = tile row of this thread.
// Arithmetic runs on packed fp32 pairs (FADD2 / FFMA2) to halve the issue
// count of this epilogue, which is instruction-bound.
__device__ __forceinline__ void run(uint32_t tmem, uint32_t quad, uint32_t half, uint32_t row,
                                    int grow, int T, int N, const float* __restrict__ bias,
                                    uint32_t res_ring, uint64_t* res_full, uint64_t* res_empty,
                                    int res_depth, const float* __restrict__ gamma,
                                    const float* __restrict__ beta, float eps,
                                    const CUtensorMap* tmY, int m0, float* gb_smem,
                                    uint64_t* acc_full, uint64_t* acc_empty, uint32_t bar_id) {
  const uint32_t loff = (quad * 32) << 16;
  const int NP = N / PN;

  float2 shift = make_float2(0.0f, 0.0f), S1 = shift, S2 = shift;
  for (int i = 0; i < NP; ++i) {
    const int q = piece_of(i, NP);
    const int c0 = q * PN + half * 32;
    float4 b[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) b[k] = __ldg(reinterpret_cast<const float4*>(bias + c0) + k);
    uint32_t r[16];
    {
      const int slot = i % res_depth;
      mbar_wait(&res_full[slot], (i / res_depth) & 1);
      load_res32(res_ring + slot * 128 * 128, row, half, r);
      release_box(&res_empty[slot]);
    }
    const uint32_t acc = i & 1;
#ifdef LN_TRACE
    if (threadIdx.x == 64) LN_TRACE(200 + i);
#endif
    mbar_wait(&acc_full[acc], (i >> 1) & 1);
    tc_fence_after();
#ifdef LN_TRACE
    if (threadIdx.x == 64) LN_TRACE(232 + i);
#endif
    uint32_t v[32];
    tmem_ld32(tmem + loff + acc * PN + half * 32, v);
    tmem_ld_wait();
    tc_fence_before();
    mbar_arrive(&acc_empty[acc]);
    if (i == 0) {
      const float s00 = bf2(pack2(make_float2(__uint_as_float(v[0]) + b[0].x, 0.0f))).x +
                        bf2(r[0]).x;
      shift = make_float2(-s00, -s00);
    }
    uint32_t park[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float4& bq = b[k >> 1];
      const float2 bb = (k & 1) ? make_float2(bq.z, bq.w) : make_float2(bq.x, bq.y);
      // o: the sublayer output exactly as the unfused path stores it (bf16)
      const float2 o = bf2(pack2(
          __fadd2_rn(make_float2(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1])), bb)));
      const float2 sv = __fadd2_rn(o, bf2(r[k]));
      park[k] = pack2(sv);
      const float2 t = __fadd2_rn(sv, shift);
      S1 = __fadd2_rn(S1, t);
      S2 = __ffma2_rn(t, t, S2);
    }
    tmem_st16(tmem + loff + kPark + q * 32 + half * 16, park);
  }
  tmem_st_wait();
#ifdef LN_TRACE
  if (threadIdx.x == 64) LN_TRACE(300);
#endif
  const float nh = static_cast<float>(NP * 32);
  const float s1 = S1.x + S1.y, s2 = S2.x + S2.y;
  const float mean_h = s1 / nh - shift.x;
  const float m2_h = fmaxf(s2 - s1 * (s1 / nh), 0.0f);
  // exchange with the other half-row thread (same TMEM lane) through columns
  // [0, 4) of the drained accumulator: the last MMA into it has completed and
  // only this lane's own threads touch this lane
  tmem_st2(tmem + loff + 2 * half, __float_as_uint(mean_h), __float_as_uint(m2_h));
  tmem_st_wait();
  tc_fence_before();
  named_bar_sync(bar_id, kEpiThreads);
  tc_fence_after();
  uint32_t mo, m2o;
  tmem_ld2(tmem + loff + 2 * (half ^ 1), mo, m2o);
  tmem_ld_wait();
  const float mean_o = __uint_as_float(mo), m2_o = __uint_as_float(m2o);
  const float delta = mean_o - mean_h;
  const float mean = 0.5f * (mean_h + mean_o);
  const float m2 = m2_h + m2_o + delta * delta * (0.5f * nh);
  const float rstd = rsqrtf(m2 / static_cast<float>(N) + eps);
  // y = gamma * ((s - mean) * rstd) + beta = gamma * (s * rstd + off) + beta
  const float2 rs2 = make_float2(rstd, rstd), off2 = make_float2(-mean * rstd, -mean * rstd);

  // gamma | beta -> shared memory (the caller's region is idle by now)
  const int et = static_cast<int>(threadIdx.x) - 64;  // 0..255 across the epilogue warps
  for (int c = et * 4; c < N; c += kEpiThreads * 4) {
    *reinterpret_cast<float4*>(gb_smem + c) = __ldg(reinterpret_cast<const float4*>(gamma + c));
    *reinterpret_cast<float4*>(gb_smem + N + c) = __ldg(reinterpret_cast<const float4*>(beta + c));
  }
  named_bar_sync(bar_id, kEpiThreads);

  // second sweep: normalise, stage [128 x 64] bf16 boxes in the (drained)
  // residual ring, TMA-store them
  for (int i = 0; i < NP; ++i) {
    const int q = piece_of(i, NP);
    const int c0 = q * PN + half * 32;
    uint32_t park[16];
    tmem_ld16(tmem + loff + kPark + q * 32 + half * 16, park);
    tmem_ld_wait();
    uint32_t w[16];
#pragma unroll
    for (int k = 0; k < 16; k += 2) {
      const float4 g = *reinterpret_cast<const float4*>(gb_smem + c0 + 2 * k);
      const float4 be = *reinterpret_cast<const float4*>(gb_smem + N + c0 + 2 * k);
      const float2 n0 = __ffma2_rn(bf2(park[k]), rs2, off2);
      const float2 n1 = __ffma2_rn(bf2(park[k + 1]), rs2, off2);
      w[k] = pack2(__ffma2_rn(make_float2(g.x, g.y), n0, make_float2(be.x, be.y)));
      w[k + 1] = pack2(__ffma2_rn(make_float2(g.z, g.w), n1, make_float2(be.z, be.w)));
    }
    const uint32_t box = res_ring + (i & 1) * 128 * 128;
    if (i >= 2) {
      // the store issued from this box two pieces ago must have read it
      if (et == 0) tma_store_wait_read<1>();
      named_bar_sync(bar_id, kEpiThreads);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      st_shared_v4(box + swz_offset(row, half * 4 + k, 128), w[4 * k], w[4 * k + 1], w[4 * k + 2],
                   w[4 * k + 3]);
    fence_proxy_async_smem();
    named_bar_sync(bar_id, kEpiThreads);
    if (et == 0) {
      tma_store_2d_u32(tmY, box, q * PN, m0);
      tma_store_commit();
    }
  }
  if (et == 0) tma_store_wait<0>();
  (void)grow;
  (void)T;
}

}  // namespace lnepi
}  // namespace fsvd
