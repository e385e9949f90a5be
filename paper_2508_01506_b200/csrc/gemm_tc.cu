// gemm_tc.cu -- K1: persistent tcgen05 GEMM with fused bias/activation epilogue.
//
// C[M,N] = A[M,K] * B[N,K]^T (+ bias[N]) (act), bf16 in/out, fp32 accumulate
// in TMEM.  This is the B200 replacement of the reference's strided fp32
// projection loop gemm_acc_ld (attention.cpp:19-31, ffn.cpp:26-38) wherever
// it is used as a whole-matrix product: X*U (attention.cpp:239-247,
// ffn.cpp:131-134), ctx*U_o / P*V_o + b_o (attention.cpp:381-389) and
// Z*V_down + b_down (ffn.cpp:148-154).  Bias is applied in the epilogue,
// which equals the reference's bias preload up to fp32 rounding order.
//
// Structure (one CTA per SM, persistent over 128 x BN output tiles):
//   warps 0, 10 TMA producers (alternate stages): A [128 x 64] and B [BN x 64]
//               bf16 tiles (SW128) into a STAGES-deep smem ring guarded by
//               full/empty mbarriers.
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma (M=128,
//               N=BN, K=16) into one of two TMEM accumulators.
//   warps 2..9  epilogue: tcgen05.ld 32 columns at a time, bias + act,
//               bf16 pack, swizzled st.shared into a [128 x 64] box, one TMA
//               store per box.
// The double-buffered TMEM accumulator lets tile i's epilogue overlap tile
// i+1's MMAs.
#include <cstdlib>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace fsvd {
FSVD_CTA_TIMES(gemm)
}  // namespace fsvd

namespace fsvd {
namespace {

using namespace ptx;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 352;  // 0 TMA, 1 MMA, 2..9 epilogue, 10 TMA

#ifdef FSVD_TRACE
__device__ long long g_trace_gm[1024];
}  // namespace
extern "C" __attribute__((visibility("default"))) int fsvd_debug_trace_gemm_copy(long long* host, int n) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace_gm, sizeof(long long) * n));
}
namespace {
#define GTRACE(slot) do { if (blockIdx.x == 0 && (slot) < 1024) g_trace_gm[(slot)] = clock64(); } while (0)
#else
#define GTRACE(slot) do { } while (0)
#endif

template <int BN, int STAGES>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  // [128 x 64] bf16 SW128 output staging boxes: two when they fit beside the
  // ring, else one
  static constexpr int CBOX = BM * 64 * 2;
  static constexpr int NCBOX = (1024 + STAGES * (A_BYTES + B_BYTES) + 2 * CBOX + 256 <= 227 * 1024) ? 2 : 1;
  static constexpr int C_BYTES = NCBOX * CBOX;
  static constexpr int TMEM_COLS = (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + C_BYTES + 256;
  static_assert(SMEM <= 227 * 1024, "shared-memory budget");
};

// X3 (fp32 policy): every operand is three bf16 planes v = hi + mid + lo
// (kernels.cuh), and the K loop runs six times over K -- the plane pairs
// (hi,hi) (hi,mid) (mid,hi) (hi,lo) (lo,hi) (mid,mid) -- into the same fp32
// accumulator.  A and B are loaded through ONE map each over the stacked
// planes ([3M, K], [3N, K]; plane p at row offset p*M): rows a tile reads past
// a plane's end only feed output rows / columns the store clips.  The
// epilogue re-splits the fp32 result into three planes (tmC, tmC2, tmC3);
// resid planes are resid_ps elements apart.
__device__ __forceinline__ int x3_plane_a(int seg) { return (0x120100 >> (4 * seg)) & 15; }
__device__ __forceinline__ int x3_plane_b(int seg) { return (0x102010 >> (4 * seg)) & 15; }

// Tile walk.  Tiles are listed full-width first ((m, n) row-major over the
// N / BN full column tiles), then the narrow last column (N % BN wide) of
// every row tile; CTA b takes list positions k * G + (k even ? b : G-1-b)
// (a snake over the size-sorted list), so when N % BN != 0 the narrow tiles
// fill the CTAs that got one full tile fewer.  Narrow tiles run MMAs of
// their own width.
struct TileWalk {
  int num_m, nfull, tiles, G, bid;
  __device__ int pos(int k) const { return k * G + ((k & 1) ? G - 1 - bid : bid); }
  __device__ void at(int p, int bn, int& m0, int& n0) const {
    const int nf = num_m * nfull;
    if (p < nf) {
      m0 = (p / nfull) * BM;
      n0 = (p % nfull) * bn;
    } else {
      m0 = (p - nf) * BM;
      n0 = nfull * bn;
    }
  }
};

template <int BN, int STAGES, bool X3 = false>
__global__ void __launch_bounds__(kThreads, 1)
    k_gemm_bf16(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const float* __restrict__ bias, int act,
                int M, int N, int K, const bf16* resid, int64_t ldr,
                const __grid_constant__ CUtensorMap tmC2, const __grid_constant__ CUtensorMap tmC3,
                int64_t resid_ps, int split_n) {
  using Cfg = GemmCfg<BN, STAGES>;
  CTA_T(0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays __shared__
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * Cfg::A_BYTES;
  uint8_t* sC = sB + STAGES * Cfg::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + Cfg::C_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n;
  const int nk = (K + BK - 1) / BK;
  const int nk3 = X3 ? 6 * nk : nk;  // K blocks of the six plane-pair sweeps
  const TileWalk walk{num_m, N / BN, tiles, static_cast<int>(gridDim.x), static_cast<int>(blockIdx.x)};

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmC);
    if (X3) {
      tma_prefetch(&tmC2);
      tma_prefetch(&tmC3);
    }
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  pdl_wait();
  CTA_T(1);
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == kThreads / 32 - 1) {
    // ---------------- TMA producers (one thread in each of two warps) ----------------
    // A TMA instruction occupies its issuing thread for ~250 cycles whatever
    // the box size (tests/cuda/tma_probe.cu), so two issuers alternate stages.
    if (lane == 0) {
      const int me = warp == 0 ? 0 : 1;
      uint32_t stage = 0, phase = 0;
      int it = 0;
      for (int k = 0; walk.pos(k) < tiles; ++k) {
        int m0, n0;
        walk.at(walk.pos(k), BN, m0, n0);
        for (int kb3 = 0; kb3 < nk3; ++kb3, ++it) {
          if ((it & 1) == me) {
            const int seg = X3 ? kb3 / nk : 0, kb = kb3 - seg * nk;
            const int ra = X3 ? x3_plane_a(seg) * M : 0, rb = X3 ? x3_plane_b(seg) * N : 0;
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], Cfg::A_BYTES + Cfg::B_BYTES);
            tma_load_2d(&tmA, &full[stage], sA + stage * Cfg::A_BYTES, kb * BK, m0 + ra);
            tma_load_2d(&tmB, &full[stage], sB + stage * Cfg::B_BYTES, kb * BK, n0 + rb);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (warp-uniform loop, one elected lane issues) ----------------
    {
      const uint64_t dhi = desc_hi_kmajor(128);
      const uint64_t da = desc_at(dhi, smem_u32(sA)), db = desc_at(dhi, smem_u32(sB));
      uint32_t stage = 0, phase = 0;
      int i = 0;
      for (int k = 0; walk.pos(k) < tiles; ++k, ++i) {
        int m0, n0;
        walk.at(walk.pos(k), BN, m0, n0);
        // narrow last column: an MMA of its own width (rounded up to 16)
        const uint32_t idesc = idesc_bf16(BM, min(BN, (N - n0 + 15) / 16 * 16));
        const uint32_t acc = i & 1, use = i >> 1;
        if (lane == 0) GTRACE(16 + 4 * i);
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        if (lane == 0) GTRACE(17 + 4 * i);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < nk3; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t a0 = da + ((stage * Cfg::A_BYTES) >> 4);
          const uint64_t b0 = db + ((stage * Cfg::B_BYTES) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              mma_bf16_ss(d, a0 + 2 * kk, b0 + 2 * kk, idesc, (kb | kk) != 0);
            mma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit(&tfull[acc]);
        __syncwarp();
        if (lane == 0) GTRACE(18 + 4 * i);
      }
    }
  } else {
    // ---------------- epilogue (8 warps) ----------------
    // Two warps per TMEM lane quadrant, each taking 32 of every 64 columns.
    // Output leaves through [128 x 64] SW128 boxes staged in shared memory
    // (double-buffered) and written by ONE TMA store per box: a TMA
    // instruction costs its thread ~250 cycles whatever the box size.
    const uint32_t q = warp & 3, half = (warp - 2) >> 2;
    const uint32_t row = q * 32 + lane;
    const int et = static_cast<int>(threadIdx.x) - 64;  // 0..255
    const uint32_t s_c = smem_u32(sC);
    uint32_t nbox = 0;
    int i = 0;
    for (int k = 0; walk.pos(k) < tiles; ++k, ++i) {
      int m0, n0;
      walk.at(walk.pos(k), BN, m0, n0);
      const uint32_t acc = i & 1, use = i >> 1;
      if (threadIdx.x == 64) GTRACE(512 + 4 * i);
      mbar_wait(&tfull[acc], use & 1);
      if (threadIdx.x == 64) GTRACE(513 + 4 * i);
      tc_fence_after();
      const uint32_t tbase = tmem + acc * BN + ((q * 32) << 16);
#pragma unroll 1
      for (int b0 = 0; b0 < BN; b0 += 64) {
        if (n0 + b0 >= N) break;
        const int c0 = b0 + static_cast<int>(half) * 32;
        uint32_t r[32];
        tmem_ld32(tbase + c0, r);
        tmem_ld_wait();
        if (b0 + 64 >= BN || n0 + b0 + 64 >= N) {
          // last TMEM read of this tile by this warp: hand the accumulator back
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
        }
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (X3)
          bias_act_chunk_exact<32>(v, bias != nullptr ? bias + n0 + c0 : nullptr, N - (n0 + c0), act);
        else
          bias_act_chunk<32>(v, bias != nullptr ? bias + n0 + c0 : nullptr, N - (n0 + c0), act);
        for (int pl = 0; pl < (X3 ? kPlanes : 1); ++pl) {  // C = A B^T + bias + R (R = sum of planes)
          const bf16* rp = resid == nullptr ? nullptr : resid + pl * resid_ps;
          if (rp == nullptr || m0 + static_cast<int>(row) >= M) continue;
          const uint4* rr = reinterpret_cast<const uint4*>(rp + (int64_t)(m0 + row) * ldr + n0 + c0);
#pragma unroll
          for (int q8 = 0; q8 < 4; ++q8) {
            if (n0 + c0 + 8 * q8 >= N) break;
            const uint4 u = rr[q8];
            const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              v[8 * q8 + 2 * e] += __uint_as_float(w4[e] << 16);
              v[8 * q8 + 2 * e + 1] += __uint_as_float(w4[e] & 0xffff0000u);
            }
          }
        }
#pragma unroll 1
        for (int pl = 0; pl < (X3 ? kPlanes : 1); ++pl) {
          if (X3 && pl > 0) {  // next plane: what the previous planes' rounding left
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] -= bf16_round_f(v[j]);
          }
          const uint32_t box = s_c + (nbox % Cfg::NCBOX) * Cfg::CBOX;
          if (nbox >= Cfg::NCBOX) {
            if (et == 0) {
              if (Cfg::NCBOX == 2) tma_store_wait_read<1>();
              else tma_store_wait_read<0>();
            }
            named_bar_sync(1, kEpiWarps * 32);
          }
#pragma unroll
          for (int c = 0; c < 4; ++c)
            st_shared_v4(box + swz_offset(row, half * 4 + c, 128), pack_bf16(v[8 * c + 0], v[8 * c + 1]),
                         pack_bf16(v[8 * c + 2], v[8 * c + 3]),
                         pack_bf16(v[8 * c + 4], v[8 * c + 5]),
                         pack_bf16(v[8 * c + 6], v[8 * c + 7]));
          fence_proxy_async_smem();
          named_bar_sync(1, kEpiWarps * 32);
          if (et == 0) {
            if (!X3 && split_n > 0 && n0 + b0 >= split_n)  // split output: columns >= split_n
              tma_store_2d_u32(&tmC2, box, n0 + b0 - split_n, m0);
            else
              tma_store_2d_u32(pl == 0 ? &tmC : pl == 1 ? &tmC2 : &tmC3, box, n0 + b0, m0);
            tma_store_commit();
          }
          ++nbox;
        }
      }
      if (threadIdx.x == 64) GTRACE(514 + 4 * i);
    }
    if (et == 0) tma_store_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free<Cfg::TMEM_COLS>(tmem);
  }
  CTA_T(2);
}

// ============================================================================
// CTA-pair variant (cta_group::2): a cluster of two CTAs computes a 256 x BN
// tile; rank r loads its own 128 rows of A and rows [r*BN/2, (r+1)*BN/2) of
// the B tile, the leader (rank 0) issues M = 256 MMAs over both CTAs' shared
// memory, and each CTA drains its own 128 x BN accumulator.  Per SM this
// halves the B bytes pulled from L2 and read from shared memory per FLOP --
// the 1-CTA kernel is L2-fabric bound on the QKV projection.
template <int BN, int STAGES>
struct Gemm2Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;  // this CTA's half
  static constexpr int CBOX = BM * 64 * 2;
  static constexpr int C_BYTES = 2 * CBOX;
  static constexpr int TMEM_COLS = (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
  static constexpr int SMEM = 1024 + STAGES * (A_BYTES + B_BYTES) + C_BYTES + 256;
  static_assert(SMEM <= 227 * 1024, "shared-memory budget");
  static_assert(BN % 32 == 0 && BN <= 256, "pair MMA N");
};

template <int BN, int STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_gemm2_bf16(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmC, const float* __restrict__ bias, int act,
                 int M, int N, int K) {
  using Cfg = Gemm2Cfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays __shared__
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * Cfg::A_BYTES;
  uint8_t* sC = sB + STAGES * Cfg::B_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sC + Cfg::C_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_rank();
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const int num_m = (M + 2 * BM - 1) / (2 * BM), num_n = (N + BN - 1) / BN;
  const int tiles = num_m * num_n;
  const int nk = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmC);
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);   // leader: one arrive.expect_tx for both CTAs' bytes
      mbar_init(&empty[i], 1);  // one multicast commit per use
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kEpiWarps);  // leader: both CTAs' epilogue warps
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<Cfg::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 || warp == kThreads / 32 - 1) {
    // ---------------- TMA producers (both CTAs; two issuers each) ----------------
    if (lane == 0) {
      const int me = warp == 0 ? 0 : 1;
      uint32_t stage = 0, phase = 0;
      int it = 0;
      for (int t = pair; t < tiles; t += npairs) {
        const int m0 = (t / num_n) * 2 * BM + static_cast<int>(rank) * BM;
        const int n0 = (t % num_n) * BN + static_cast<int>(rank) * (BN / 2);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          if ((it & 1) == me) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], 2 * (Cfg::A_BYTES + Cfg::B_BYTES));
            tma_load_2d_pair(&tmA, &full[stage], sA + stage * Cfg::A_BYTES, kb * BK, m0);
            tma_load_2d_pair(&tmB, &full[stage], sB + stage * Cfg::B_BYTES, kb * BK, n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA only) ----------------
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_bf16(2 * BM, BN);
      const uint64_t dhi = desc_hi_kmajor(128);
      const uint64_t da = desc_at(dhi, smem_u32(sA)), db = desc_at(dhi, smem_u32(sB));
      uint32_t stage = 0, phase = 0;
      int i = 0;
      for (int t = pair; t < tiles; t += npairs, ++i) {
        const uint32_t acc = i & 1, use = i >> 1;
        mbar_wait(&tempty[acc], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t a0 = da + ((stage * Cfg::A_BYTES) >> 4);
          const uint64_t b0 = db + ((stage * Cfg::B_BYTES) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              mma_bf16_ss_pair(d, a0 + 2 * k, b0 + 2 * k, idesc, (kb | k) != 0);
            mma_commit_pair(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit_pair(&tfull[acc], 0x3);
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue (8 warps per CTA, own 128 rows) ----------------
    const uint32_t q = warp & 3, half = (warp - 2) >> 2;
    const uint32_t row = q * 32 + lane;
    const int et = static_cast<int>(threadIdx.x) - 64;
    const uint32_t s_c = smem_u32(sC);
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
    uint32_t nbox = 0;
    int i = 0;
    for (int t = pair; t < tiles; t += npairs, ++i) {
      const int m0 = (t / num_n) * 2 * BM + static_cast<int>(rank) * BM, n0 = (t % num_n) * BN;
      const uint32_t acc = i & 1, use = i >> 1;
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
      const uint32_t tbase = tmem + acc * BN + ((q * 32) << 16);
#pragma unroll 1
      for (int b0 = 0; b0 < BN; b0 += 64) {
        if (n0 + b0 >= N) break;
        const int c0 = b0 + static_cast<int>(half) * 32;
        uint32_t r[32];
        tmem_ld32(tbase + c0, r);
        tmem_ld_wait();
        if (b0 + 64 >= BN || n0 + b0 + 64 >= N) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(tempty_leader0 + acc * 8);
        }
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        bias_act_chunk<32>(v, bias != nullptr ? bias + n0 + c0 : nullptr, N - (n0 + c0), act);
        const uint32_t box = s_c + (nbox & 1) * Cfg::CBOX;
        if (nbox >= 2) {
          if (et == 0) tma_store_wait_read<1>();
          named_bar_sync(1, kEpiWarps * 32);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
          st_shared_v4(box + swz_offset(row, half * 4 + c, 128), pack_bf16(v[8 * c + 0], v[8 * c + 1]),
                       pack_bf16(v[8 * c + 2], v[8 * c + 3]),
                       pack_bf16(v[8 * c + 4], v[8 * c + 5]),
                       pack_bf16(v[8 * c + 6], v[8 * c + 7]));
        fence_proxy_async_smem();
        named_bar_sync(1, kEpiWarps * 32);
        if (et == 0) {
          tma_store_2d_u32(&tmC, box, n0 + b0, m0);
          tma_store_commit();
        }
        ++nbox;
      }
    }
    if (et == 0) tma_store_wait<0>();
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_free_pair<Cfg::TMEM_COLS>(tmem);
  }
}

template <int BN, int STAGES>
void launch_gemm2(const bf16* A, int64_t lda, const bf16* B, int64_t ldb, bf16* C, int64_t ldc,
                  int M, int N, int K, const float* bias, int act, cudaStream_t s) {
  using Cfg = Gemm2Cfg<BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    FSVD_CUDA_CHECK(cudaFuncSetAttribute(k_gemm2_bf16<BN, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    attr = true;
  }
  const CUtensorMap ta = tmap_bf16(A, M, K, lda, BM, BK, TmaSwizzle::B128);
  const CUtensorMap tb = tmap_bf16(B, N, K, ldb, BN / 2, BK, TmaSwizzle::B128);
  const CUtensorMap tc = tmap_bf16(C, M, N, ldc, BM, 64, TmaSwizzle::B128);
  const int tiles = ((M + 2 * BM - 1) / (2 * BM)) * ((N + BN - 1) / BN);
  int pairs = num_sms() / 2;
  if (tiles < pairs) pairs = tiles;
  k_gemm2_bf16<BN, STAGES><<<2 * pairs, kThreads, Cfg::SMEM, s>>>(ta, tb, tc, bias, act, M, N, K);
  check_launch("k_gemm2_bf16");
}

template <int BN, int STAGES, bool X3 = false>
void launch_gemm(const bf16* A, int64_t lda, const bf16* B, int64_t ldb, bf16* C, int64_t ldc,
                 int M, int N, int K, const float* bias, int act, cudaStream_t s,
                 const bf16* resid = nullptr, int64_t ldr = 0, bf16* C2 = nullptr,
                 bf16* C3 = nullptr, int64_t resid_ps = 0, int split_n = 0, int64_t ldc2 = 0) {
  using Cfg = GemmCfg<BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    FSVD_CUDA_CHECK(cudaFuncSetAttribute(k_gemm_bf16<BN, STAGES, X3>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    attr = true;
  }
  const int np = X3 ? kPlanes : 1;  // stacked planes behind A and B
  const CUtensorMap ta = tmap_bf16(A, (uint64_t)np * M, K, lda, BM, BK, TmaSwizzle::B128);
  const CUtensorMap tb = tmap_bf16(B, (uint64_t)np * N, K, ldb, BN, BK, TmaSwizzle::B128);
  // split output (non-X3): columns [0, split_n) -> C, [split_n, N) -> C2 (pitch ldc2)
  const bool split = !X3 && split_n > 0;
  const CUtensorMap tc = tmap_bf16(C, M, split ? split_n : N, ldc, BM, 64, TmaSwizzle::B128);
  const CUtensorMap tc2 = X3      ? tmap_bf16(C2, M, N, ldc, BM, 64, TmaSwizzle::B128)
                          : split ? tmap_bf16(C2, M, N - split_n, ldc2, BM, 64, TmaSwizzle::B128)
                                  : tc;
  const CUtensorMap tc3 = X3 ? tmap_bf16(C3, M, N, ldc, BM, 64, TmaSwizzle::B128) : tc;
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  launch_pdl(k_gemm_bf16<BN, STAGES, X3>, dim3(grid), dim3(kThreads), Cfg::SMEM, s, ta, tb, tc,
             bias, act, M, N, K, resid, ldr, tc2, tc3, resid_ps, split ? split_n : 0);
  check_launch("k_gemm_bf16");
}

// Heaviest CTA of the snake walk (TileWalk), in 64-column units of MMA work.
int snake_units(int M, int N, int BN) {
  const int G = num_sms();
  const int num_m = (M + BM - 1) / BM, nfull = N / BN, rem = N % BN;
  const int tiles = num_m * (nfull + (rem ? 1 : 0));
  std::vector<int> load(G, 0);
  for (int p = 0; p < tiles; ++p) {
    const int k = p / G, r = p % G, b = (k & 1) ? G - 1 - r : r;
    load[b] += (p < num_m * nfull ? BN : rem + 63) / 64;
  }
  return *std::max_element(load.begin(), load.end());
}

// N divisible by 192 but not 256 (the folded QKV width 1152 at cfg2): 256-wide
// tiles plus a narrow last column when their snake walk is lighter
// (cfg2: 16 vs 18 units on the busiest CTA).  FSVD_GEMM_SNAKE256=0 keeps 192.
bool prefer_256(int M, int N) {
  static const bool on = [] {
    const char* e = getenv("FSVD_GEMM_SNAKE256");
    return !(e && e[0] == '0');
  }();
  return on && N > 256 && snake_units(M, N, 256) < snake_units(M, N, 192);
}

}  // namespace

bool gemm_bf16_supported(int M, int N, int K, int64_t lda, int64_t ldb, int64_t ldc) {
  // TMA needs 16-byte aligned row pitches; tiles cover any M, N, K tails.
  return M > 0 && N > 0 && K > 0 && lda % 8 == 0 && ldb % 8 == 0 && ldc % 8 == 0 && K % 8 == 0;
}

void gemm_bf16(const bf16* A, int64_t lda, const bf16* B, int64_t ldb, bf16* C, int64_t ldc,
               int M, int N, int K, const float* bias, int act, cudaStream_t s, const bf16* resid,
               int64_t ldr) {
  static const int variant = [] {
    const char* e = getenv("FSVD_GEMM_VARIANT");  // developer A/B switch
    return e ? atoi(e) : 0;
  }();
  if (!resid && variant == 2 && N % 192 == 0) {
    launch_gemm2<192, 6>(A, lda, B, ldb, C, ldc, M, N, K, bias, act, s);
    return;
  }
  if (!resid && variant == 3 && N % 256 == 0) {
    launch_gemm2<256, 6>(A, lda, B, ldb, C, ldc, M, N, K, bias, act, s);
    return;
  }
  if (!resid && variant == 5 && N % 128 == 0) {  // single-CTA 128-wide tiles (wave-quantization probe)
    launch_gemm<128, 6>(A, lda, B, ldb, C, ldc, M, N, K, bias, act, s, resid, ldr);
    return;
  }
  if (!resid && variant == 6 && N % 64 == 0) {
    launch_gemm<64, 8>(A, lda, B, ldb, C, ldc, M, N, K, bias, act, s, resid, ldr);
    return;
  }
  if (!resid && variant == 4 && N % 128 == 0) {
    launch_gemm2<128, 8>(A, lda, B, ldb, C, ldc, M, N, K, bias, act, s);
    return;
  }
  if (M <= 128 && N % 64 == 0 && N >= 128)  // one row tile (decode rows): most CTAs
    launch_gemm<64, 8>(A, lda, B, ldb, C, ldc, M, N, K, bias, act, s, resid, ldr);
  else if (N % 256 == 0 || (N % 192 == 0 && prefer_256(M, N)))
    launch_gemm<256, 4>(A, lda, B, ldb, C, ldc, M, N, K, bias, act, s, resid, ldr);
  else if (N % 192 == 0)
    launch_gemm<192, 4>(A, lda, B, ldb, C, ldc, M, N, K, bias, act, s, resid, ldr);
  else if (N > 1024)
    launch_gemm<256, 4>(A, lda, B, ldb, C, ldc, M, N, K, bias, act, s, resid, ldr);
  else if (N % 128 == 0 || N > 64)
    launch_gemm<128, 6>(A, lda, B, ldb, C, ldc, M, N, K, bias, act, s, resid, ldr);
  else
    launch_gemm<64, 8>(A, lda, B, ldb, C, ldc, M, N, K, bias, act, s, resid, ldr);
}

void gemm_bf16_split(const bf16* A, int64_t lda, const bf16* B, int64_t ldb, bf16* C,
                     int64_t ldc, int split_n, bf16* C2, int64_t ldc2, int M, int N, int K,
                     const float* bias, cudaStream_t s) {
  if (split_n % 64 != 0 || split_n <= 0 || split_n >= N || ldc2 % 8 != 0)
    throw CudaError("gemm_bf16_split: split column must be a positive multiple of 64 below N");
  static const int bn = [] {
    const char* e = getenv("FSVD_SPLIT_BN");  // developer A/B switch
    return e ? atoi(e) : 0;
  }();
  if (bn == 128 && N % 128 == 0)
    launch_gemm<128, 6>(A, lda, B, ldb, C, ldc, M, N, K, bias, ACT_NONE, s, nullptr, 0, C2,
                        nullptr, 0, split_n, ldc2);
  else if (N % 192 == 0 && prefer_256(M, N))
    launch_gemm<256, 4>(A, lda, B, ldb, C, ldc, M, N, K, bias, ACT_NONE, s, nullptr, 0, C2,
                        nullptr, 0, split_n, ldc2);
  else if (N % 192 == 0)
    launch_gemm<192, 4>(A, lda, B, ldb, C, ldc, M, N, K, bias, ACT_NONE, s, nullptr, 0, C2,
                        nullptr, 0, split_n, ldc2);
  else if (N % 256 == 0 || N > 1024)
    launch_gemm<256, 4>(A, lda, B, ldb, C, ldc, M, N, K, bias, ACT_NONE, s, nullptr, 0, C2,
                        nullptr, 0, split_n, ldc2);
  else
    launch_gemm<128, 6>(A, lda, B, ldb, C, ldc, M, N, K, bias, ACT_NONE, s, nullptr, 0, C2,
                        nullptr, 0, split_n, ldc2);
}

void gemm_x3(const Planes& A, int64_t lda, const Planes& B, int64_t ldb, const PlanesOut& C,
             int64_t ldc, int M, int N, int K, const float* bias, int act, cudaStream_t s,
             const Planes* resid, int64_t ldr) {
  // the loads address A and B as stacked planes (one tensor map each)
  const int64_t pa = (int64_t)M * lda, pb = (int64_t)N * ldb;
  if (A.mid != A.hi + pa || A.lo != A.mid + pa || B.mid != B.hi + pb || B.lo != B.mid + pb)
    throw CudaError("gemm_x3: the planes of A and B must be stacked contiguously");
  const bf16* r = resid ? resid->hi : nullptr;
  const int64_t rps = resid ? resid->mid - resid->hi : 0;
  if (resid && resid->lo - resid->mid != rps)
    throw CudaError("gemm_x3: residual planes must be evenly spaced");
  if (M <= 128 && N % 64 == 0 && N >= 128)
    launch_gemm<64, 8, true>(A.hi, lda, B.hi, ldb, C.hi, ldc, M, N, K, bias, act, s, r, ldr, C.mid,
                             C.lo, rps);
  else if (N % 128 == 0 || N > 64)
    launch_gemm<128, 6, true>(A.hi, lda, B.hi, ldb, C.hi, ldc, M, N, K, bias, act, s, r, ldr,
                              C.mid, C.lo, rps);
  else
    launch_gemm<64, 8, true>(A.hi, lda, B.hi, ldb, C.hi, ldc, M, N, K, bias, act, s, r, ldr, C.mid,
                             C.lo, rps);
}

}  // namespace fsvd
