// gemm_ln_tc.cu -- K6: low-rank projection GEMM with the residual + LayerNorm
// fused into its epilogue.
//
//   y[T, N] = LN( resid + bf16(A[T, K] B[N, K]^T + bias) ) * gamma + beta
//
// Replaces the out-projection + residual_norm pair of the post-LN layer
// (lowrank_output_projection attention.cpp:366-391 followed by
// residual_norm encoder.cpp:38-50 / layer_norm_row tensor.cpp:88-102): the
// [T, d] sublayer output never reaches HBM.  The rounding points equal the
// unfused pipeline's: the projection result is rounded to bf16 (what the
// unfused path stores), the residual sum and the statistics are fp32, the
// variance is biased, eps sits inside the square root.
//
// One CTA owns 128 complete rows, so the LayerNorm statistics never leave
// the SM:
//   * A (the rank-width activation, K <= 512) is TMA-loaded once and stays
//     resident in shared memory as K/64 SW128 atoms;
//   * B (the [N, K] weight) streams through a ring of [64 x 64] bf16 slots;
//   * the output is produced in 64-column pieces into a double-buffered
//     TMEM accumulator (columns [0, 128)); the epilogue adds the bias, rounds
//     to bf16, adds the residual, accumulates shifted row statistics and
//     parks the pre-normalisation row, two bf16 per 32-bit column, in TMEM
//     columns [128, 128 + N/2) -- all N values of a row fit in TMEM (N <= 768);
//   * after the last piece, the two threads of each row combine their
//     statistics (Chan's pairwise update) and a second sweep over the parked
//     values writes normalized rows.
//
// Warps: 0 and 11 TMA producers (A, B; alternating stages), 1 MMA issuer +
// TMEM owner, 2..9 epilogue (two per TMEM lane quadrant; each owns 32 of the
// 64 columns of a piece), 10 residual producer (ln_epi.cuh).
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#ifdef FSVD_TRACE
namespace fsvd { __device__ long long g_trace_ln[1024]; }
#define LN_TRACE(slot) do { if (blockIdx.x == 0) ::fsvd::g_trace_ln[(slot)] = clock64(); } while (0)
#endif
#include "ln_epi.cuh"
#include "ptx.cuh"

namespace fsvd {
FSVD_CTA_TIMES(gemm_ln)
}  // namespace fsvd

namespace fsvd {
namespace {

using namespace ptx;

constexpr int kThreads = 384;
constexpr int kEpi = 256;
constexpr int BMr = 128;            // rows per CTA
// 128-column pieces into one TMEM accumulator.  The FSVD_LN_PN=64 build runs
// 64-column pieces into two accumulators ([0, 64), [64, 128)) so the MMA of
// piece q+1 overlaps the drain of piece q (run_groups): measured slower
// (23.7 vs 17.8 us at cfg2 -- N = 64 MMAs are shared-memory bound and the
// epilogue pays its per-piece latency twelve times instead of six).
#ifndef FSVD_LN_PN
#define FSVD_LN_PN 128
#endif
constexpr int PN = FSVD_LN_PN;      // output columns per piece
constexpr int NACC = PN == 64 ? 2 : 1;
constexpr int ATOM = BMr * 128;     // [128 x 64] bf16 A atom (16 KB)
constexpr int SLOT = PN * 128;      // [128 x 64] bf16 B slot (16 KB)
constexpr int SPS = 1;              // slots per ring stage
constexpr int STAGE = SPS * SLOT;
constexpr int kMaxStages = 12;
constexpr int RS = 2;               // residual ring depth ([128 x 64] bf16 boxes)
constexpr int RBOX = BMr * 128;
constexpr int kBoxes = 4;           // second-sweep output staging boxes (in the B ring; K <= 512 leaves 4 stages)

#ifdef FSVD_TRACE
}  // namespace
extern "C" __attribute__((visibility("default"))) int fsvd_debug_trace_ln_copy(long long* host, int n) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace_ln, sizeof(long long) * n));
}
namespace {
#define LTRACE(slot) LN_TRACE(slot)
#else
#define LTRACE(slot) do { } while (0)
#endif

struct LnBars {
  uint64_t full[kMaxStages], empty[kMaxStages];
  uint64_t a_full, acc_full[2], acc_empty[2], res_full[RS], res_empty[RS];
  uint64_t box_full[kBoxes], box_free[kBoxes];  // second-sweep output boxes (ln_epi.cuh store_boxes)
  uint32_t tmem;
};

__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_ln(const __grid_constant__ CUtensorMap tmA,  // A [T, K]  box 128 x 64
              const __grid_constant__ CUtensorMap tmB,  // B [N, K]  box 64 x 64
              const __grid_constant__ CUtensorMap tmR,  // resid [T, N] box 128 x 64
              const __grid_constant__ CUtensorMap tmY,  // y     [T, N] box 128 x 64
              const float* __restrict__ bias,
              const float* __restrict__ gamma, const float* __restrict__ beta, float eps,
              bf16* y, int T, int N, int K, int stages,
              bf16* sum_out, int seq_tiles) {
  CTA_T(0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays __shared__
  const int KA = K / 64;        // A atoms
  const int NP = N / PN;        // output pieces
  uint8_t* sA = smem;
  uint8_t* ring = sA + KA * ATOM;
  uint8_t* rring = ring + stages * STAGE;
  LnBars* bars = reinterpret_cast<LnBars*>(rring + RS * RBOX);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int m0 = blockIdx.x * BMr;
  const int rot = lnepi::seq_rotation(blockIdx.x, seq_tiles, N / PN);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmR);
    tma_prefetch(&tmY);
    for (int i = 0; i < stages; ++i) {
      mbar_init(&bars->full[i], 1);
      mbar_init(&bars->empty[i], 1);
    }
    mbar_init(&bars->a_full, 1);
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&bars->acc_full[i], 1);
      mbar_init(&bars->acc_empty[i], lnepi::acc_drain_arrivals<PN>());
    }
    for (int i = 0; i < RS; ++i) {
      mbar_init(&bars->res_full[i], 1);
      mbar_init(&bars->res_empty[i], lnepi::res_box_readers<PN>());
    }
    for (int i = 0; i < kBoxes; ++i) {
      mbar_init(&bars->box_full[i], lnepi::box_writer_warps<PN>());
      mbar_init(&bars->box_free[i], 1);
    }
    fence_barrier_init();
  }
  if (threadIdx.x == 0) LTRACE(0);
  if (warp == 1) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) LTRACE(3);
  tc_fence_after();
  pdl_trigger();
  pdl_wait();
  CTA_T(1);
  const uint32_t tmem = bars->tmem;

  if (warp == 0 || warp == 11) {
    // ============================================ TMA producers (A, B)
    // One thread in each of two warps, alternating: a TMA instruction holds
    // its issuing thread for ~250 cycles (tests/cuda/tma_probe.cu).
    if (lane == 0) {
      const int me = warp == 0 ? 0 : 1;
      if (me == 0) mbar_arrive_expect_tx(&bars->a_full, KA * ATOM);
      for (int a = me; a < KA; a += 2) tma_load_2d(&tmA, &bars->a_full, sA + a * ATOM, a * 64, m0);
      uint32_t st = 0, ph = 0;
      const int nslots = NP * KA;
      for (int i = 0; i < nslots; i += SPS) {
        if (((i / SPS) & 1) == me) {
          mbar_wait(&bars->empty[st], ph ^ 1);
          if (i / SPS < 200) LTRACE(400 + i / SPS);
          const int n = (nslots - i) < SPS ? (nslots - i) : SPS;
          mbar_arrive_expect_tx(&bars->full[st], n * SLOT);
          for (int j = 0; j < n; ++j) {
            const int s = i + j, q = lnepi::piece_of(s / KA, NP, rot), a = s % KA;
            tma_load_2d(&tmB, &bars->full[st], ring + st * STAGE + j * SLOT, a * 64, q * PN);
          }
        }
        if (++st == (uint32_t)stages) { st = 0; ph ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ============================================ MMA issuer
    // The whole warp runs the (warp-uniform) loop so descriptors live in
    // uniform registers; one elected lane issues.  N = 64 MMAs take only ~32
    // cycles each, so per-MMA issue overhead must stay below that.
    const uint64_t dhi = desc_hi_kmajor(128);
    constexpr uint32_t idesc = idesc_bf16(BMr, PN);
    const uint64_t da0 = desc_at(dhi, smem_u32(sA));
    const uint64_t db0 = desc_at(dhi, smem_u32(ring));
    LTRACE(1);
    mbar_wait(&bars->a_full, 0);
    tc_fence_after();
    LTRACE(2);
    uint32_t st = 0, ph = 0;
    int in_stage = 0;
    for (int q = 0; q < NP; ++q) {
      // accumulator q % NACC: the epilogue must have drained piece q - NACC
      const int acc = q % NACC;
      if (q >= NACC) {
        mbar_wait(&bars->acc_empty[acc], ((q / NACC) - 1) & 1);
        tc_fence_after();
      }
      LTRACE(16 + q);
      const uint32_t d = tmem + acc * PN;
      for (int a = 0; a < KA; ++a) {
        if (in_stage == 0) {
          mbar_wait(&bars->full[st], ph);
          tc_fence_after();
          if (q * KA + a < 400) LTRACE(600 + (q * KA + a) / SPS);
        }
        // start-address field is in 16-byte units: +2 per 16-element K step
        const uint64_t bd = db0 + ((st * STAGE + in_stage * SLOT) >> 4);
        const uint64_t ad = da0 + ((a * ATOM) >> 4);
        if (elect_one()) {
          mma_bf16_ss(d, ad, bd, idesc, a != 0);
          mma_bf16_ss(d, ad + 2, bd + 2, idesc, 1u);
          mma_bf16_ss(d, ad + 4, bd + 4, idesc, 1u);
          mma_bf16_ss(d, ad + 6, bd + 6, idesc, 1u);
        }
        __syncwarp();
        const bool last = (q == NP - 1) && (a == KA - 1);
        if (++in_stage == SPS || last) {
          if (elect_one()) mma_commit(&bars->empty[st]);
          __syncwarp();
          in_stage = 0;
          if (++st == (uint32_t)stages) { st = 0; ph ^= 1; }
        }
      }
      if (elect_one()) mma_commit(&bars->acc_full[acc]);
      __syncwarp();
      LTRACE(48 + q);
    }
  } else if (warp == 10) {
    // ============================================ residual producer, then the
    // second sweep's store thread (one thread)
    if (lane == 0) {
      lnepi::produce_residual<PN>(&tmR, rring, bars->res_full, bars->res_empty, RS, N, m0, rot);
      lnepi::store_boxes<PN, kBoxes>(&tmY, smem_u32(ring), bars->box_full, bars->box_free, N, m0,
                                     rot);
    }
    __syncwarp();
  } else {
    // ============================================ epilogue (8 warps)
    const uint32_t quad = warp & 3;
    const uint32_t half = (warp - 2) >> 2;  // which 32 columns of each piece
    const uint32_t row = quad * 32 + lane;
    // second sweep: output boxes staged in the B ring, gamma / beta in the A
    // region (both idle once every MMA has completed)
    lnepi::run<PN, kBoxes>(tmem, quad, half, row, N, bias, smem_u32(rring), bars->res_full,
                   bars->res_empty, RS, gamma, beta, eps, &tmY, m0, reinterpret_cast<float*>(sA),
                   smem_u32(ring), bars->box_full, bars->box_free, bars->acc_full,
                   bars->acc_empty, 1, 0, sum_out, T, rot);
  }
  if (threadIdx.x == 64) LTRACE(100);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) LTRACE(101);
  if (warp == 1) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
  CTA_T(2);
}

}  // namespace

bool gemm_ln_supported(int N, int K) {
  return N % PN == 0 && N <= lnepi::kMaxN && K % 64 == 0 && K >= 64 && K <= 512;
}

void gemm_ln_bf16(const bf16* A, int64_t lda, const bf16* B, int64_t ldb, const float* bias,
                  const bf16* resid, const float* gamma, const float* beta, float eps, bf16* y,
                  int T, int N, int K, cudaStream_t s, bf16* sum_out, int seq_tiles) {
  if (!gemm_ln_supported(N, K)) throw CudaError("gemm_ln_bf16: unsupported shape");
  if (gemm_ln_pair_enabled() &&
      gemm_ln_pair_bf16(A, lda, B, ldb, bias, resid, gamma, beta, eps, y, T, N, K, s, sum_out,
                        seq_tiles))
    return;
  const int KA = K / 64;
  int stages =
      (227 * 1024 - 1024 - KA * ATOM - RS * RBOX - static_cast<int>(sizeof(LnBars))) / STAGE;
  stages = stages > kMaxStages ? kMaxStages : stages;
  // the ring doubles as the second sweep's output staging
  if (stages * STAGE < kBoxes * RBOX)
    throw CudaError("gemm_ln_bf16: K too large for the shared-memory ring");
  const int smem = 1024 + KA * ATOM + stages * STAGE + RS * RBOX + static_cast<int>(sizeof(LnBars));
  static int attr = 0;
  if (attr < smem) {
    FSVD_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_ln, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024));
    attr = 227 * 1024;
  }
  const CUtensorMap ta = tmap_bf16(A, T, K, lda, BMr, 64, TmaSwizzle::B128);
  const CUtensorMap tb = tmap_bf16(B, N, K, ldb, PN, 64, TmaSwizzle::B128);
  const CUtensorMap tr = tmap_bf16(resid, T, N, N, BMr, 64, TmaSwizzle::B128);
  const CUtensorMap ty = tmap_bf16(y, T, N, N, BMr, 64, TmaSwizzle::B128);
  static const bool rot_off = [] {
    const char* e = getenv("FSVD_LN_ROT");  // developer A/B switch: 0 = no piece rotation
    return e && e[0] == '0';
  }();
  if (rot_off) seq_tiles = 0;
  const int grid = (T + BMr - 1) / BMr;
  launch_pdl(k_gemm_ln, dim3(grid), dim3(kThreads), smem, s, ta, tb, tr, ty, bias, gamma, beta,
             eps, y, T, N, K, stages, sum_out, seq_tiles);
  check_launch("k_gemm_ln");
}

}  // namespace fsvd
