// gemm_ln2_tc.cu -- K6 on a CTA pair: the out-projection GEMM with the
// residual + LayerNorm epilogue, cta_group::2.
//
//   y[T, N] = LN( resid + bf16(A[T, K] B[N, K]^T + bias) ) * gamma + beta
//
// Same contract and rounding points as k_gemm_ln (gemm_ln_tc.cu: the
// out-projection + residual_norm pair, attention.cpp:366-391 then
// encoder.cpp:38-50), but a cluster of two CTAs on one TPC owns 256 rows:
// each CTA keeps its own 128 rows of A resident and streams only HALF of
// every [128 x 64] weight slot (64 of the piece's 128 output columns); the
// even CTA issues M = 256 MMAs over both CTAs' shared memory.  Per SM this
// halves the weight bytes pulled from L2, and the ring -- now in 8 KB half
// slots -- holds two output pieces instead of one.  Measured on the cfg2
// step: 24.75 µs against k_gemm_ln's 23.96 (ncu launch list), so it stays
// opt-in (FSVD_LN_PAIR=1): K6's first sweep is bound by its LayerNorm
// epilogue (~2.9 K cycles per 128-column piece against 1.5 K of MMA), which
// the pair does not shorten.
//
// Each CTA runs the LayerNorm epilogue (ln_epi.cuh) on its own rows: the
// accumulator is released to the leader's barrier (one relaxed remote arrive
// per warp), residual boxes and output boxes are per CTA.
//
// Barrier ownership (as ffn2_tc.cu): the leader owns full, a_full and
// acc_empty (TMA bytes of both CTAs complete on the leader's full / a_full,
// both CTAs' epilogue warps arrive on its acc_empty); empty and acc_full exist
// in both CTAs and receive multicast commits.
//
// Warps: 0 and 11 TMA producers (A, B half slots; both CTAs), 1 MMA issuer
// (leader) + TMEM owner, 2..9 epilogue, 10 residual producer and store
// thread of the second sweep.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "ln_epi.cuh"
#include "ptx.cuh"

namespace fsvd {
namespace {

using namespace ptx;

constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;
constexpr int BMr = 128;              // rows per CTA (256 per pair)
constexpr int PN = 128;               // output columns per piece (pair MMA N)
constexpr int ATOM = BMr * 128;       // [128 x 64] bf16 A atom (16 KB)
constexpr int HSLOT = (PN / 2) * 128; // this CTA's half of a [128 x 64] weight slot (8 KB)
constexpr int kMaxStages = 16;
constexpr int RS = 2;                 // residual ring depth ([128 x 64] boxes)
constexpr int RBOX = BMr * 128;
constexpr int kBoxes = 4;             // second-sweep output staging boxes (in the ring)

struct Ln2Bars {
  uint64_t full[kMaxStages], empty[kMaxStages];
  uint64_t a_full, acc_full[1], acc_empty[1], res_full[RS], res_empty[RS];
  uint64_t box_full[kBoxes], box_free[kBoxes];
  uint32_t tmem;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_gemm_ln2(const __grid_constant__ CUtensorMap tmA,  // A [T, K]  box 128 x 64
               const __grid_constant__ CUtensorMap tmB,  // B [N, K]  box 64 x 64
               const __grid_constant__ CUtensorMap tmR,  // resid [T, N] box 128 x 64
               const __grid_constant__ CUtensorMap tmY,  // y     [T, N] box 128 x 64
               const float* __restrict__ bias, const float* __restrict__ gamma,
               const float* __restrict__ beta, float eps, int T, int N, int K, int stages,
               bf16* sum_out, int seq_pairs) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays __shared__
  const int KA = K / 64;  // A atoms
  const int NP = N / PN;  // output pieces
  uint8_t* sA = smem;
  uint8_t* ring = sA + KA * ATOM;
  uint8_t* rring = ring + stages * HSLOT;
  Ln2Bars* bars = reinterpret_cast<Ln2Bars*>(rring + RS * RBOX);
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_rank();
  const int m0 = static_cast<int>(blockIdx.x >> 1) * (2 * BMr) + static_cast<int>(rank) * BMr;
  // pieces start at an offset set by the pair tile's place in its sequence
  // (ln_epi.cuh piece_of); both CTAs of the pair use the same one
  const int rot = lnepi::seq_rotation(static_cast<int>(blockIdx.x >> 1), seq_pairs, NP);

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
    mbar_init(&bars->acc_full[0], 1);
    mbar_init(&bars->acc_empty[0], 2 * kEpiWarps);  // one arrive per epilogue warp, both CTAs
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
  if (warp == 1) tmem_alloc_pair<512>(&bars->tmem);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  pdl_trigger();
  pdl_wait();
  const uint32_t tmem = bars->tmem;

  if (warp == 0 || warp == 11) {
    // ============================================ TMA producers (both CTAs)
    if (lane == 0) {
      const int me = warp == 0 ? 0 : 1;
      if (me == 0 && rank == 0) mbar_arrive_expect_tx(&bars->a_full, 2 * KA * ATOM);
      for (int a = me; a < KA; a += 2)
        tma_load_2d_pair(&tmA, &bars->a_full, sA + a * ATOM, a * 64, m0);
      uint32_t st = 0, ph = 0;
      const int nslots = NP * KA;
      for (int i = 0; i < nslots; ++i) {
        if ((i & 1) == me) {
          mbar_wait(&bars->empty[st], ph ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&bars->full[st], 2 * HSLOT);
          const int q = lnepi::piece_of(i / KA, NP, rot), a = i % KA;
          tma_load_2d_pair(&tmB, &bars->full[st], ring + st * HSLOT, a * 64,
                           q * PN + static_cast<int>(rank) * (PN / 2));
        }
        if (++st == static_cast<uint32_t>(stages)) { st = 0; ph ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ============================================ MMA issuer (leader only)
    if (rank == 0) {
      const uint64_t dhi = desc_hi_kmajor(128);
      constexpr uint32_t idesc = idesc_bf16(2 * BMr, PN);
      const uint64_t da0 = desc_at(dhi, smem_u32(sA));
      const uint64_t db0 = desc_at(dhi, smem_u32(ring));
      mbar_wait(&bars->a_full, 0);
      tc_fence_after();
      uint32_t st = 0, ph = 0;
      for (int q = 0; q < NP; ++q) {
        // single accumulator: both CTAs' epilogues must have drained piece q-1
        if (q >= 1) {
          mbar_wait(&bars->acc_empty[0], (q - 1) & 1);
          tc_fence_after();
        }
        for (int a = 0; a < KA; ++a) {
          mbar_wait(&bars->full[st], ph);
          tc_fence_after();
          const uint64_t bd = db0 + ((st * HSLOT) >> 4);
          const uint64_t ad = da0 + ((a * ATOM) >> 4);
          if (elect_one()) {
            mma_bf16_ss_pair(tmem, ad, bd, idesc, a != 0);
            mma_bf16_ss_pair(tmem, ad + 2, bd + 2, idesc, 1u);
            mma_bf16_ss_pair(tmem, ad + 4, bd + 4, idesc, 1u);
            mma_bf16_ss_pair(tmem, ad + 6, bd + 6, idesc, 1u);
            mma_commit_pair(&bars->empty[st], 0x3);
          }
          __syncwarp();
          if (++st == static_cast<uint32_t>(stages)) { st = 0; ph ^= 1; }
        }
        if (elect_one()) mma_commit_pair(&bars->acc_full[0], 0x3);
        __syncwarp();
      }
    }
  } else if (warp == 10) {
    // ============================================ residual producer, then the
    // second sweep's store thread (one thread, own rows)
    if (lane == 0) {
      lnepi::produce_residual<PN>(&tmR, rring, bars->res_full, bars->res_empty, RS, N, m0, rot);
      lnepi::store_boxes<PN, kBoxes>(&tmY, smem_u32(ring), bars->box_full, bars->box_free, N, m0,
                                     rot);
    }
    __syncwarp();
  } else {
    // ============================================ epilogue (8 warps, own rows)
    const uint32_t quad = warp & 3;
    const uint32_t half = (warp - 2) >> 2;
    const uint32_t row = quad * 32 + lane;
    // second sweep: output boxes staged in the ring, gamma / beta in the A
    // region (both idle once every MMA has completed)
    lnepi::run<PN, kBoxes>(tmem, quad, half, row, N, bias, smem_u32(rring), bars->res_full,
                           bars->res_empty, RS, gamma, beta, eps, &tmY, m0,
                           reinterpret_cast<float*>(sA), smem_u32(ring), bars->box_full,
                           bars->box_free, bars->acc_full, bars->acc_empty, 1,
                           mapa_shared(smem_u32(&bars->acc_empty[0]), 0), sum_out, T, rot);
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_free_pair<512>(tmem);
  }
}

}  // namespace

bool gemm_ln_pair_enabled() {
  static const bool on = [] {
    // opt-in (FSVD_LN_PAIR=1): measured level with k_gemm_ln on the cfg2 step
    // (24.75 vs 23.96 µs in the launch list) -- K6's first sweep is bound by
    // its LayerNorm epilogue, not by the weight stream the pair halves
    const char* e = getenv("FSVD_LN_PAIR");
    return e && e[0] == '1';
  }();
  return on;
}

bool gemm_ln_pair_bf16(const bf16* A, int64_t lda, const bf16* B, int64_t ldb, const float* bias,
                       const bf16* resid, const float* gamma, const float* beta, float eps, bf16* y,
                       int T, int N, int K, cudaStream_t s, bf16* sum_out, int seq_tiles) {
  if (T < 2 * BMr || N % PN != 0 || N > lnepi::kMaxN || K % 64 != 0 ||
      K < 64 || K > 512)
    return false;
  const int KA = K / 64;
  int stages =
      (227 * 1024 - 1024 - KA * ATOM - RS * RBOX - static_cast<int>(sizeof(Ln2Bars))) / HSLOT;
  stages = stages > kMaxStages ? kMaxStages : stages;
  if (stages * HSLOT < kBoxes * RBOX) return false;  // the ring stages the output boxes
  const int smem = 1024 + KA * ATOM + stages * HSLOT + RS * RBOX + static_cast<int>(sizeof(Ln2Bars));
  static int attr = 0;
  if (attr < smem) {
    FSVD_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_ln2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024));
    attr = 227 * 1024;
  }
  const CUtensorMap ta = tmap_bf16(A, T, K, lda, BMr, 64, TmaSwizzle::B128);
  const CUtensorMap tb = tmap_bf16(B, N, K, ldb, PN / 2, 64, TmaSwizzle::B128);
  const CUtensorMap tr = tmap_bf16(resid, T, N, N, BMr, 64, TmaSwizzle::B128);
  const CUtensorMap ty = tmap_bf16(y, T, N, N, BMr, 64, TmaSwizzle::B128);
  const int pairs = (T + 2 * BMr - 1) / (2 * BMr);
  const int seq_pairs = seq_tiles % 2 == 0 ? seq_tiles / 2 : 0;
  launch_pdl(k_gemm_ln2, dim3(2 * pairs), dim3(kThreads), smem, s, ta, tb, tr, ty, bias, gamma,
             beta, eps, T, N, K, stages, sum_out, seq_pairs);
  check_launch("k_gemm_ln2");
  return true;
}

}  // namespace fsvd
