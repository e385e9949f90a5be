// ln_epi.cuh -- residual + LayerNorm epilogue shared by the row-complete
// tensor-core kernels (K6 k_gemm_ln, K4 k_ffn with the fused LN2).
//
// The producing MMA writes PN-column pieces of a 128-row output tile into
// TMEM columns [0, 128): PN = 64 double-buffers two accumulators, PN = 128
// uses one (then MMAs are N = 128, which the tensor pipe runs at full rate
// from shared memory; N = 64 runs at 2/3).  For each piece the epilogue (8
// warps, two per TMEM lane quadrant, each owning PN/2 of the piece's
// columns) adds the bias, rounds to bf16 -- the value the unfused
// pipeline stores for the sublayer output --, adds the bf16 residual in fp32
// and accumulates shifted row sums of that fp32 sum s.  s itself is parked in
// TMEM as fp16, two per 32-bit column at [128, 128 + N/2), so the whole row
// stays on chip.  Once every piece is in, the two half-row statistics are
// merged (Chan's pairwise update; biased variance, eps inside the square
// root, tensor.cpp:88-102) and a second sweep over the parked values writes
// y = gamma * ((s - mean) * rstd) + beta.  The statistics are exact fp32;
// the value being normalised carries one fp16 rounding (<= 2^-11 relative).
// Parking s in bf16 (2^-9) was measured to push the 12-layer cfg2 error to
// 2.4e-2 on some sequences -- large-magnitude features carry |s| many times
// the row's standard deviation -- against 1.0e-2 with fp16 and 1.2e-2 with
// the exact sum (re-reading the residual in the second sweep: +2.3% step
// time).  fp16's range bounds |x + sublayer(x)| by 65504 (a post-LN residual
// stream is renormalised every layer; beyond the range the output turns
// inf / NaN instead of silently wrong).
//
// Memory traffic is all bulk/asynchronous: a dedicated producer warp TMA-loads
// the residual as [128 x 64] bf16 SW128 boxes into a two-box ring; in the
// second sweep the same two boxes stage the normalised output for TMA stores,
// and gamma / beta are staged once in shared memory the kernel no longer
// needs.
#pragma once

#include <cuda_fp16.h>

#include "ptx.cuh"

namespace fsvd {
namespace lnepi {

using namespace ptx;

constexpr int kPark = 128;        // first TMEM column of the parked values
constexpr int kEpiThreads = 256;
constexpr int kMaxN = 2 * (512 - kPark);
constexpr int kBox = 128 * 128;   // one [128 x 64] bf16 SW128 box

// 32 residual values (16 bf16 pairs) of `row`, columns [c, c+32) (c = 0 or
// 32) of one [128 x 64] SW128 box at shared address `box`.
__device__ __forceinline__ void load_res32(uint32_t box, uint32_t row, uint32_t c,
                                           uint32_t (&r)[16]) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[4 * k]), "=r"(r[4 * k + 1]), "=r"(r[4 * k + 2]), "=r"(r[4 * k + 3])
                 : "r"(box + swz_offset(row, (c >> 3) + k, 128)));
}
// bf16x2 -> float2 (exact: bf16 is the top half of an fp32)
__device__ __forceinline__ float2 bf2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
__device__ __forceinline__ uint32_t pack2(float2 v) { return pack_bf16(v.x, v.y); }
// fp16x2 park of the pre-normalisation sum (see the header)
__device__ __forceinline__ uint32_t packh2(float2 v) {
  __half2 h = __floats2half2_rn(v.x, v.y);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float2 h2f(uint32_t w) {
  __half2 h = *reinterpret_cast<__half2*>(&w);
  return __half22float2(h);
}

// Hands a residual box back to the TMA producer.  The generic-proxy reads of
// the box must be complete and ordered before the next TMA (async-proxy)
// write into it: without the proxy fence the arrive was observed to overtake
// the in-flight LDS and the refill raced the read.
__device__ __forceinline__ void release_box(uint64_t* empty) {
  fence_proxy_async_smem();
  mbar_arrive(empty);
}

// Column piece handled at step i: the pieces start at `rot`, which the
// kernels set from the tile's position inside its sequence (FfnTcArgs::
// seq_tiles), so concurrent CTAs read different weight boxes instead of all
// pulling the same box through the same L2 slices at once; the statistics'
// summation order then depends only on the row's place in its sequence, never
// on the batch position.
__device__ __forceinline__ int piece_of(int i, int NP, int rot = 0) {
  const int q = i + rot;
  return q >= NP ? q - NP : q;
}
// Rotation for a CTA whose 128-row tile is `tile` (blockIdx) when a sequence
// holds seq_tiles tiles (0: no rotation), over n steps.
__device__ __forceinline__ int seq_rotation(int tile, int seq_tiles, int n) {
  return seq_tiles > 1 ? (tile % seq_tiles) * n / seq_tiles : 0;
}

// Residual producer (one thread): streams the [128 x N] residual tile at row
// m0 as [128 x 64] boxes, pieces in piece_of() order, through a ring of
// `depth` boxes.
template <int PN>
__device__ __forceinline__ void produce_residual(const CUtensorMap* tm, uint8_t* ring,
                                                 uint64_t* full, uint64_t* empty, int depth,
                                                 int N, int m0, int rot = 0) {
  constexpr int BPP = PN / 64;  // boxes per piece
  const int NP = N / PN;
  for (int b = 0; b < NP * BPP; ++b) {
    const int slot = b % depth;
    mbar_wait(&empty[slot], ((b / depth) & 1) ^ 1);
    mbar_arrive_expect_tx(&full[slot], kBox);
    tma_load_2d(tm, &full[slot], ring + slot * kBox, piece_of(b / BPP, NP, rot) * PN + (b % BPP) * 64,
                m0);
  }
}
// Output boxes of run()'s second sweep: one thread of an otherwise idle warp
// issues the TMA store of every box as soon as its writers have arrived on
// box_full[slot] (box_writer_warps() arrivals), and frees the slot once the
// store has read it.  Box j = (piece j / BPP, 64-column half j % BPP), slot
// j % NBOX, in piece_of() order; the writers run up to NBOX - 1 boxes ahead
// of the store issue.
template <int PN>
constexpr int box_writer_warps() { return kEpiThreads / 64; }  // one group (PN 64) / one half (PN 128)
template <int PN, int NBOX = 2 * (PN / 64)>
__device__ __forceinline__ void store_boxes(const CUtensorMap* tmY, uint32_t out_stage,
                                            uint64_t* box_full, uint64_t* box_free, int N,
                                            int m0, int rot = 0) {
  constexpr int BPP = PN / 64;
  static_assert(NBOX % BPP == 0 && NBOX >= 2 * BPP, "staging slots");
  const int NP = N / PN;
  for (int j = 0; j < NP * BPP; ++j) {
    const int slot = j % NBOX;
    mbar_wait(&box_full[slot], (j / NBOX) & 1);
    tma_store_2d_u32(tmY, out_stage + slot * kBox, piece_of(j / BPP, NP, rot) * PN + (j % BPP) * 64,
                     m0);
    tma_store_commit();
    tma_store_wait_read<1>();  // every store before box j has read its slot
    if (j >= 1) mbar_arrive(&box_free[(j - 1) % NBOX]);
  }
  tma_store_wait<0>();
}
// Arrivals a residual box needs before it can be refilled.
template <int PN>
constexpr int res_box_readers() { return kEpiThreads / 2; }  // one group (PN 64) / one half (PN 128)

// Runs in all 256 epilogue threads: `quad` = TMEM lane quadrant (hardware
// warp id % 4), `half` = which of the two warp groups (pieces i with
// i % 2 == half), `row` = tile row.  The two groups take alternate pieces
// whole, so one group computes piece i while the other waits for / loads
// piece i + 1 -- the epilogue is latency-bound (TMEM load, bias, residual
// box, pack chains) and the two groups' latencies overlap instead of both
// groups stalling on the same piece.
// Accumulator protocol: PN = 64 alternates acc_full/empty[0..1] (buffers at
// columns 0 and 64; buffer i % 2 = the group's own); PN = 128 uses
// acc_full/empty[0] only.  acc_empty takes one group's arrivals per piece:
// acc_drain_arrivals<64>() threads, or in a CTA pair (acc_empty_leader != 0:
// shared::cluster address of the leader's acc_empty[0]) one remote arrive
// per warp of the group from each CTA.  Arithmetic runs on packed fp32 pairs
// (FADD2 / FFMA2).
constexpr int kGroupThreads = kEpiThreads / 2;
// threads that release an accumulator per piece: one group (PN = 64) or all
// epilogue threads (PN = 128)
template <int PN>
constexpr int acc_drain_arrivals() { return PN == 64 ? kGroupThreads : kEpiThreads; }
template <int PN, int NBOX = 2 * (PN / 64)>
__device__ __forceinline__ void run_groups(uint32_t tmem, uint32_t quad, uint32_t half, uint32_t row,
                                    int N, const float* __restrict__ bias, uint32_t res_ring,
                                    uint64_t* res_full, uint64_t* res_empty, int res_depth,
                                    const float* __restrict__ gamma,
                                    const float* __restrict__ beta, float eps,
                                    const CUtensorMap* tmY, int m0, float* gb_smem,
                                    uint32_t out_stage, uint64_t* box_full, uint64_t* box_free,
                                    uint64_t* acc_full, uint64_t* acc_empty,
                                    uint32_t bar_id, uint32_t acc_empty_leader = 0,
                                    bf16* sum_out = nullptr, int rows = 0, int rot = 0) {
  static_assert(PN == 64 || PN == 128, "piece width");
  constexpr int BPP = PN / 64;  // [128 x 64] boxes per piece
  const uint32_t loff = (quad * 32) << 16;
  const int NP = N / PN;
  // gamma / beta for the second sweep: this thread's float4 of each, loaded
  // now so the load latency hides behind the first sweep (N <= kMaxN < 4 *
  // kEpiThreads: at most one float4 per thread)
  static_assert(kMaxN <= 4 * kEpiThreads, "one gamma / beta float4 per epilogue thread");
  const int gb_c = (static_cast<int>(threadIdx.x) - 64) * 4;
  float4 gb_g = make_float4(0.0f, 0.0f, 0.0f, 0.0f), gb_b = gb_g;
  if (gb_c < N) {
    gb_g = __ldg(reinterpret_cast<const float4*>(gamma + gb_c));
    gb_b = __ldg(reinterpret_cast<const float4*>(beta + gb_c));
  }

  float2 shift = make_float2(0.0f, 0.0f), S1 = shift, S2 = shift;
  bool first = true;
  for (int i = static_cast<int>(half); i < NP; i += 2) {
    const int q = piece_of(i, NP, rot);
    const uint32_t acc = PN == 64 ? (i & 1) : 0;
    const uint32_t par = PN == 64 ? ((i >> 1) & 1) : (i & 1);
#ifdef LN_TRACE
    if (threadIdx.x == 64) LN_TRACE(200 + i);
#endif
    mbar_wait(&acc_full[acc], par);
    tc_fence_after();
#ifdef LN_TRACE
    if (threadIdx.x == 64) LN_TRACE(232 + i);
#endif
    // the piece in 64-column boxes: two 32-column TMEM chunks per box
#pragma unroll
    for (int bx = 0; bx < BPP; ++bx) {
      uint32_t v[2][32];
      tmem_ld32(tmem + loff + acc * 64 + bx * 64, v[0]);
      tmem_ld32(tmem + loff + acc * 64 + bx * 64 + 32, v[1]);
      tmem_ld_wait();
      if (bx == BPP - 1) {  // the whole piece is in registers: hand the accumulator back
        tc_fence_before();
        if (acc_empty_leader) {
          // CTA pair: one arrive per warp on the leader CTA's barrier; the
          // signal is "TMEM drained" (no shared-memory data), so no release fence
          __syncwarp();
          if ((threadIdx.x & 31) == 0) mbar_arrive_cluster_relaxed(acc_empty_leader + acc * 8);
        } else {
          mbar_arrive(&acc_empty[acc]);
        }
      }
      // residual box of these 64 columns
      const int rb = i * BPP + bx;
      const int slot = rb % res_depth;
      mbar_wait(&res_full[slot], (rb / res_depth) & 1);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int col = q * PN + bx * 64 + c * 32;  // first output column of the chunk
        float4 b[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) b[k] = __ldg(reinterpret_cast<const float4*>(bias + col) + k);
        uint32_t r[16];
        load_res32(res_ring + slot * kBox, row, c * 32, r);
        if (c == 1) release_box(&res_empty[slot]);
        if (first) {
          const float s00 = bf2(pack2(make_float2(__uint_as_float(v[c][0]) + b[0].x, 0.0f))).x +
                            bf2(r[0]).x;
          shift = make_float2(-s00, -s00);
          first = false;
        }
        uint32_t park[16], sums[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float4& bq = b[k >> 1];
          const float2 bb = (k & 1) ? make_float2(bq.z, bq.w) : make_float2(bq.x, bq.y);
          // o: the sublayer output exactly as the unfused path stores it (bf16)
          const float2 o = bf2(pack2(__fadd2_rn(
              make_float2(__uint_as_float(v[c][2 * k]), __uint_as_float(v[c][2 * k + 1])), bb)));
          const float2 sv = __fadd2_rn(o, bf2(r[k]));
          park[k] = packh2(sv);
          sums[k] = pack2(sv);
          const float2 t = __fadd2_rn(sv, shift);
          S1 = __fadd2_rn(S1, t);
          S2 = __ffma2_rn(t, t, S2);
        }
        tmem_st16(tmem + loff + kPark + col / 2, park);
        if (sum_out != nullptr && m0 + static_cast<int>(row) < rows) {
          // pre-LN residual stream: the un-normalised sum, as the unfused path stores it
          uint4* d = reinterpret_cast<uint4*>(sum_out + (int64_t)(m0 + static_cast<int>(row)) * N + col);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            d[k] = make_uint4(sums[4 * k], sums[4 * k + 1], sums[4 * k + 2], sums[4 * k + 3]);
        }
      }
    }
  }
  tmem_st_wait();
#ifdef LN_TRACE
  if (threadIdx.x == 64) LN_TRACE(300);
#endif
  // this group's elements: its pieces (NP may be odd: group 0 then has one more)
  const int my_pieces = (NP - static_cast<int>(half) + 1) / 2;
  const int ot_pieces = NP - my_pieces;
  const float nh = static_cast<float>(my_pieces * PN), no = static_cast<float>(ot_pieces * PN);
  const float s1 = S1.x + S1.y, s2 = S2.x + S2.y;
  const float mean_h = my_pieces ? s1 / nh - shift.x : 0.0f;
  const float m2_h = my_pieces ? fmaxf(s2 - s1 * (s1 / nh), 0.0f) : 0.0f;
  // exchange with the other group's thread of this row (same TMEM lane)
  // through columns [0, 4) of the drained accumulator: the last MMA into it
  // has completed and only this lane's own threads touch this lane
  tmem_st2(tmem + loff + 2 * half, __float_as_uint(mean_h), __float_as_uint(m2_h));
  tmem_st_wait();
  tc_fence_before();
  named_bar_sync(bar_id, kEpiThreads);
  tc_fence_after();
  uint32_t mo, m2o;
  tmem_ld2(tmem + loff + 2 * (half ^ 1), mo, m2o);
  tmem_ld_wait();
  const float mean_o = __uint_as_float(mo), m2_o = __uint_as_float(m2o);
  // Chan's pairwise merge (counts nh, no)
  const float ntot = nh + no;
  const float delta = mean_o - mean_h;
  const float mean = (nh * mean_h + no * mean_o) / ntot;
  const float m2 = m2_h + m2_o + delta * delta * (nh * no / ntot);
  const float rstd = rsqrtf(m2 / static_cast<float>(N) + eps);
  // y = gamma * ((s - mean) * rstd) + beta = gamma * (s * rstd + off) + beta
  const float2 rs2 = make_float2(rstd, rstd), off2 = make_float2(-mean * rstd, -mean * rstd);

  // gamma | beta -> shared memory (the caller's region is idle by now)
  if (gb_c < N) {
    *reinterpret_cast<float4*>(gb_smem + gb_c) = gb_g;
    *reinterpret_cast<float4*>(gb_smem + N + gb_c) = gb_b;
  }
  named_bar_sync(bar_id, kEpiThreads);
#ifdef LN_TRACE
  if (threadIdx.x == 64) LN_TRACE(301);
#endif

  // second sweep: normalise into [128 x 64] bf16 boxes staged at out_stage;
  // each finished box is handed to the kernel's store thread (store_boxes)
  // through box_full / box_free, so no epilogue thread waits on a TMA store
  // instruction.  Box j of the sweep = (piece j / BPP, 64-column part j % BPP),
  // staging slot j % NBOX; a group fills the boxes of its own pieces.
  for (int i = static_cast<int>(half); i < NP; i += 2) {
    const int q = piece_of(i, NP, rot);
#pragma unroll
    for (int bx = 0; bx < BPP; ++bx) {
      const int j = i * BPP + bx;
      const int slot = j % NBOX;
      const uint32_t box = out_stage + slot * kBox;
      if (j >= NBOX) mbar_wait(&box_free[slot], ((j / NBOX) - 1) & 1);
      uint32_t park[2][16];
      tmem_ld16(tmem + loff + kPark + (q * PN + bx * 64) / 2, park[0]);
      tmem_ld16(tmem + loff + kPark + (q * PN + bx * 64 + 32) / 2, park[1]);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int col = q * PN + bx * 64 + c * 32;
        uint32_t w[16];
#pragma unroll
        for (int k = 0; k < 16; k += 2) {
          const float4 g = *reinterpret_cast<const float4*>(gb_smem + col + 2 * k);
          const float4 be = *reinterpret_cast<const float4*>(gb_smem + N + col + 2 * k);
          const float2 n0 = __ffma2_rn(h2f(park[c][k]), rs2, off2);
          const float2 n1 = __ffma2_rn(h2f(park[c][k + 1]), rs2, off2);
          w[k] = pack2(__ffma2_rn(make_float2(g.x, g.y), n0, make_float2(be.x, be.y)));
          w[k + 1] = pack2(__ffma2_rn(make_float2(g.z, g.w), n1, make_float2(be.z, be.w)));
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
          st_shared_v4(box + swz_offset(row, c * 4 + k, 128), w[4 * k], w[4 * k + 1],
                       w[4 * k + 2], w[4 * k + 3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&box_full[slot]);
    }
#ifdef LN_TRACE
    if (threadIdx.x == 64) LN_TRACE(310 + i);
#endif
  }
#ifdef LN_TRACE
  if (threadIdx.x == 64) LN_TRACE(330);
#endif
}

// Column halves (PN = 128, single accumulator): both warp groups work on
// every piece, each on half of its columns.  Alternating whole pieces between
// the groups needs one accumulator per group -- with a single one a group
// that skips a phase could wait on the wrong parity -- so the single-buffered
// kernels (K6) keep this form.
template <int PN, int NBOX = 2 * (PN / 64)>
__device__ __forceinline__ void run_halves(uint32_t tmem, uint32_t quad, uint32_t half, uint32_t row,
                                    int N, const float* __restrict__ bias, uint32_t res_ring,
                                    uint64_t* res_full, uint64_t* res_empty, int res_depth,
                                    const float* __restrict__ gamma,
                                    const float* __restrict__ beta, float eps,
                                    const CUtensorMap* tmY, int m0, float* gb_smem,
                                    uint32_t out_stage, uint64_t* box_full, uint64_t* box_free,
                                    uint64_t* acc_full, uint64_t* acc_empty,
                                    uint32_t bar_id, uint32_t acc_empty_leader = 0,
                                    bf16* sum_out = nullptr, int rows = 0, int rot = 0) {
  static_assert(PN == 64 || PN == 128, "piece width");
  constexpr int CPT = PN / 64;  // 32-column chunks per thread per piece
  const uint32_t loff = (quad * 32) << 16;
  const int NP = N / PN;
  // gamma / beta for the second sweep: this thread's float4 of each, loaded
  // now so the load latency hides behind the first sweep (N <= kMaxN < 4 *
  // kEpiThreads: at most one float4 per thread)
  static_assert(kMaxN <= 4 * kEpiThreads, "one gamma / beta float4 per epilogue thread");
  const int gb_c = (static_cast<int>(threadIdx.x) - 64) * 4;
  float4 gb_g = make_float4(0.0f, 0.0f, 0.0f, 0.0f), gb_b = gb_g;
  if (gb_c < N) {
    gb_g = __ldg(reinterpret_cast<const float4*>(gamma + gb_c));
    gb_b = __ldg(reinterpret_cast<const float4*>(beta + gb_c));
  }

  float2 shift = make_float2(0.0f, 0.0f), S1 = shift, S2 = shift;
  for (int i = 0; i < NP; ++i) {
    const int q = piece_of(i, NP, rot);
    const uint32_t acc = PN == 64 ? (i & 1) : 0;
    const uint32_t par = PN == 64 ? ((i >> 1) & 1) : (i & 1);
#ifdef LN_TRACE
    if (threadIdx.x == 64) LN_TRACE(200 + i);
#endif
    mbar_wait(&acc_full[acc], par);
    tc_fence_after();
#ifdef LN_TRACE
    if (threadIdx.x == 64) LN_TRACE(232 + i);
#endif
    uint32_t v[CPT][32];
#pragma unroll
    for (int c = 0; c < CPT; ++c)
      tmem_ld32(tmem + loff + acc * 64 + half * (PN / 2) + c * 32, v[c]);
    tmem_ld_wait();
    tc_fence_before();
    if (acc_empty_leader) {
      // CTA pair: one arrive per warp on the leader CTA's barrier; the signal
      // is "TMEM drained" (no shared-memory data), so no release fence
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive_cluster_relaxed(acc_empty_leader + acc * 8);
    } else {
      mbar_arrive(&acc_empty[acc]);
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int col = q * PN + half * (PN / 2) + c * 32;  // first output column
      float4 b[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) b[k] = __ldg(reinterpret_cast<const float4*>(bias + col) + k);
      uint32_t r[16];
      {
        // residual box of this chunk and the 32 columns of it
        const int bx = PN == 64 ? i : 2 * i + static_cast<int>(half);
        const int slot = bx % res_depth;
        if (PN == 64 || c == 0) mbar_wait(&res_full[slot], (bx / res_depth) & 1);
        load_res32(res_ring + slot * kBox, row, PN == 64 ? half * 32 : c * 32, r);
        if (c == CPT - 1) release_box(&res_empty[slot]);
      }
      if (i == 0 && c == 0) {
        const float s00 = bf2(pack2(make_float2(__uint_as_float(v[0][0]) + b[0].x, 0.0f))).x +
                          bf2(r[0]).x;
        shift = make_float2(-s00, -s00);
      }
      uint32_t park[16], sums[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float4& bq = b[k >> 1];
        const float2 bb = (k & 1) ? make_float2(bq.z, bq.w) : make_float2(bq.x, bq.y);
        // o: the sublayer output exactly as the unfused path stores it (bf16)
        const float2 o = bf2(pack2(__fadd2_rn(
            make_float2(__uint_as_float(v[c][2 * k]), __uint_as_float(v[c][2 * k + 1])), bb)));
        const float2 sv = __fadd2_rn(o, bf2(r[k]));
        park[k] = packh2(sv);
          sums[k] = pack2(sv);
        const float2 t = __fadd2_rn(sv, shift);
        S1 = __fadd2_rn(S1, t);
        S2 = __ffma2_rn(t, t, S2);
      }
      tmem_st16(tmem + loff + kPark + col / 2, park);
      if (sum_out != nullptr && m0 + static_cast<int>(row) < rows) {
        // pre-LN residual stream: the un-normalised sum, as the unfused path stores it
        uint4* d = reinterpret_cast<uint4*>(sum_out + (int64_t)(m0 + static_cast<int>(row)) * N + col);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          d[k] = make_uint4(sums[4 * k], sums[4 * k + 1], sums[4 * k + 2], sums[4 * k + 3]);
      }
    }
  }
  tmem_st_wait();
#ifdef LN_TRACE
  if (threadIdx.x == 64) LN_TRACE(300);
#endif
  const float nh = static_cast<float>(N / 2);
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
  if (gb_c < N) {
    *reinterpret_cast<float4*>(gb_smem + gb_c) = gb_g;
    *reinterpret_cast<float4*>(gb_smem + N + gb_c) = gb_b;
  }
  named_bar_sync(bar_id, kEpiThreads);
#ifdef LN_TRACE
  if (threadIdx.x == 64) LN_TRACE(301);
#endif

  // second sweep: normalise, stage [128 x 64] bf16 boxes at out_stage (an
  // idle shared-memory region of 2 boxes for PN = 64, 4 for PN = 128) and
  // TMA-store them.  PN = 64: both halves fill one box per piece (two boxes
  // alternate, 256-thread barriers); PN = 128: each half owns a box per piece
  // and alternates its own two boxes (128-thread barriers, ids bar_id + 1 +
  // half).
  // Each finished [128 x 64] box is handed to the kernel's store thread
  // (store_boxes, below) through box_full / box_free, so no epilogue thread
  // waits on a TMA store instruction: box j of the sweep (piece j / BPP, half
  // j % BPP) lives in staging slot j % NBOX.
  for (int i = 0; i < NP; ++i) {
    const int q = piece_of(i, NP, rot);
    const int j = PN == 64 ? i : 2 * i + static_cast<int>(half);
    const int slot = j % NBOX;
    const uint32_t box = out_stage + slot * kBox;
    if (j >= NBOX) mbar_wait(&box_free[slot], ((j / NBOX) - 1) & 1);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int col = q * PN + half * (PN / 2) + c * 32;
      uint32_t park[16];
      tmem_ld16(tmem + loff + kPark + col / 2, park);
      tmem_ld_wait();
      uint32_t w[16];
#pragma unroll
      for (int k = 0; k < 16; k += 2) {
        const float4 g = *reinterpret_cast<const float4*>(gb_smem + col + 2 * k);
        const float4 be = *reinterpret_cast<const float4*>(gb_smem + N + col + 2 * k);
        const float2 n0 = __ffma2_rn(h2f(park[k]), rs2, off2);
        const float2 n1 = __ffma2_rn(h2f(park[k + 1]), rs2, off2);
        w[k] = pack2(__ffma2_rn(make_float2(g.x, g.y), n0, make_float2(be.x, be.y)));
        w[k + 1] = pack2(__ffma2_rn(make_float2(g.z, g.w), n1, make_float2(be.z, be.w)));
      }
      const uint32_t chunk0 = PN == 64 ? half * 4 : c * 4;  // 16-byte chunk within the box row
#pragma unroll
      for (int k = 0; k < 4; ++k)
        st_shared_v4(box + swz_offset(row, chunk0 + k, 128), w[4 * k], w[4 * k + 1],
                     w[4 * k + 2], w[4 * k + 3]);
    }
    fence_proxy_async_smem();
#ifdef LN_TRACE
    if (threadIdx.x == 64) LN_TRACE(310 + i);
#endif
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&box_full[slot]);
  }
#ifdef LN_TRACE
  if (threadIdx.x == 64) LN_TRACE(330);
#endif
}

// The LayerNorm epilogue: whole pieces per warp group for PN = 64 (double
// buffered: accumulator i % 2 belongs to group i % 2), column halves for
// PN = 128 (single accumulator).
template <int PN, int NBOX = 2 * (PN / 64)>
__device__ __forceinline__ void run(uint32_t tmem, uint32_t quad, uint32_t half, uint32_t row,
                                    int N, const float* __restrict__ bias, uint32_t res_ring,
                                    uint64_t* res_full, uint64_t* res_empty, int res_depth,
                                    const float* __restrict__ gamma,
                                    const float* __restrict__ beta, float eps,
                                    const CUtensorMap* tmY, int m0, float* gb_smem,
                                    uint32_t out_stage, uint64_t* box_full, uint64_t* box_free,
                                    uint64_t* acc_full, uint64_t* acc_empty,
                                    uint32_t bar_id, uint32_t acc_empty_leader = 0,
                                    bf16* sum_out = nullptr, int rows = 0, int rot = 0) {
  if constexpr (PN == 64)
    run_groups<PN, NBOX>(tmem, quad, half, row, N, bias, res_ring, res_full, res_empty, res_depth,
                         gamma, beta, eps, tmY, m0, gb_smem, out_stage, box_full, box_free,
                         acc_full, acc_empty, bar_id, acc_empty_leader, sum_out, rows, rot);
  else
    run_halves<PN, NBOX>(tmem, quad, half, row, N, bias, res_ring, res_full, res_empty, res_depth,
                         gamma, beta, eps, tmY, m0, gb_smem, out_stage, box_full, box_free,
                         acc_full, acc_empty, bar_id, acc_empty_leader, sum_out, rows, rot);
}

}  // namespace lnepi
}  // namespace fsvd
