// ffn_tc.cu -- K3 / K4: FlashSVD-FFN on tcgen05.
//
// K3 (FUSED = false) replaces the V1 feature-block stream of ffn_v1
// (ffn.cpp:136-147 -> stream_feature_blocks :84-104):
//     Z[tile] = sum_f act(P[tile] V_up[:, f] + b_up[f]) U_down[f, :]
// K4 (FUSED = true) replaces ffn_v2 (ffn.cpp:158-185) end to end:
//     P = X U_up ; stream as above ; out = Z V_down + b_down
// with nothing but the [T, d_model] output leaving the SM.
//
// One CTA owns 128 token rows.  The rank-width P tile lives in shared memory
// (bf16, K-major SW128 atoms) for the whole stream; Z accumulates in TMEM
// (FR fp32 columns) across every feature block; the d_ff-wide hidden exists
// only as one 128 x 128 block: H in TMEM -> registers (+b_up, GELU) -> bf16
// smem -> A operand of the next MMA.
//
// Operand streaming: every B operand (V_up^T / U_down^T / U_up^T / V_down^T)
// arrives as 16 KB slots ([<=128 rows x 64] bf16, SW128) through a TMA ring
// of 32 KB stages (two slots per stage), so each barrier round trip carries
// >= 8 MMAs.  The producer and the MMA issuer are single threads with
// precomputed descriptors (the tensor pipe is issue-bound otherwise).  X
// chunks of the fused up-projection are staged through the H buffer, which is
// idle in that phase.
//
// Pipelining per feature block f: MMA1(f+1) is issued as soon as the
// epilogue has drained H(f) from TMEM; MMA2(f) consumes the activated block
// one 64-wide K atom at a time, so its first half overlaps the epilogue's
// work on the second.
//
// Warps: 0 and 11 TMA producers (alternating stages), 1 MMA issuer + TMEM
// owner, 2..9 epilogue (two warps per TMEM lane quadrant, alternating
// 32-column chunks), 10 residual producer of the fused post-LN epilogue
// (ln_epi.cuh; V2 with LN2 only).
#include "common.cuh"
#include "kernels.cuh"
#ifdef FSVD_TRACE
namespace fsvd { __device__ long long g_trace_ffn_ln[512]; }
#define LN_TRACE(slot) \
  do { if (blockIdx.x == 0 && (slot) < 512) ::fsvd::g_trace_ffn_ln[(slot)] = clock64(); } while (0)
#endif
#include "ln_epi.cuh"
#include "ptx.cuh"

namespace fsvd {
FSVD_CTA_TIMES(ffn)
}  // namespace fsvd

namespace fsvd {
namespace {

using namespace ptx;

constexpr int kThreads = 384;
constexpr int kEpi = 256;
constexpr int BMr = 128;         // token rows per CTA
constexpr int BF = 128;          // features per block
constexpr int SLOT = BMr * 128;  // one [128 x 64] bf16 SW128 atom / ring slot (16 KB)
constexpr int STAGE = 2 * SLOT;  // two slots per ring stage
// fused LN2 second sweep: gamma | beta (2 x 768 fp32) at the ring's start,
// output staging boxes from here on (the ring is idle once the MMAs are done)
constexpr int kLnStage = 8192;

// WIDE (K3 only, FFN ranks above 384): Z no longer fits TMEM next to H, so
// the rank is cut into slices of FR columns, one CTA per (row tile, slice);
// P is not resident -- MMA1 streams it with V_up as (P atom, V_up atom) slot
// pairs, and each slice recomputes the hidden block.
//
// X3 (fp32 policy, K3 only, on the WIDE structure): P, V_up, U_down and the
// hidden block are three bf16 planes each (kernels.cuh; P / V_up / U_down
// through one stacked tensor map each).  MMA1 streams (P_pl, V_up_pl) for the
// three planes as three consecutive ring stages and issues the six plane
// pairs of order <= 2; the epilogue writes H in three planes; MMA2 takes
// (U_dn_hi, U_dn_mid) and (U_dn_lo) as two stages per (atom, piece).
template <int FR, bool WIDE = false, bool X3 = false>
struct FfnCfg {
  static_assert(FR % 64 == 0 && FR <= 384, "FR must be a multiple of 64, <= 384");
  static_assert(!X3 || WIDE, "the split-plane stream runs on the WIDE structure");
  static constexpr int NATOM = FR / 64;
  static constexpr int PS = (FR % 128 == 0) ? 128 : 64;  // rows per Z / P piece
  static constexpr int NPIECE = FR / PS;
  static constexpr int PATOMS = WIDE ? 0 : NATOM;        // resident P atoms
  static constexpr int HATOMS = X3 ? 6 : 2;              // H tile atoms (X3: 3 planes)
  static constexpr int STAGES_FIT = (227 * 1024 - 2048 - (PATOMS + HATOMS) * SLOT) / STAGE;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int o_p = 0;                  // P / Z tile, NATOM atoms
  static constexpr int o_h = PATOMS * SLOT;      // H tile (2 atoms, X3: + 2 lo) / X double buffer
  static constexpr int o_ring = o_h + HATOMS * SLOT;
  static constexpr int o_bar = o_ring + STAGES * STAGE;
  static constexpr int SMEM = 1024 + o_bar + 512;
  static constexpr int t_z = 0;    // Z / P accumulator (FR cols)
  static constexpr int t_h = 384;  // H (128 cols)
};

struct FfnBars {
  uint64_t full[8], empty[8];
  uint64_t x_full[2], x_empty[2];
  uint64_t p_full, p_acc, p_ready, h_full, h_free, sh_full[2], sh_free[2], z_full, zs_ready;
  uint64_t o_full[2], o_free[2];
  uint64_t res_full[2], res_empty[2];  // residual boxes of the fused LN2 (H region)
  uint64_t box_full[4], box_free[4];   // its output boxes (ln_epi.cuh store_boxes), ring-staged
  uint32_t tmem;
};

// X3 plane pairs of order <= 2: (hi,hi) (hi,mid) (mid,hi) (hi,lo) (lo,hi) (mid,mid)
__device__ __forceinline__ int x3_pa(int g) { return (0x120100 >> (4 * g)) & 15; }
__device__ __forceinline__ int x3_pb(int g) { return (0x102010 >> (4 * g)) & 15; }

// 32 consecutive fp32 columns of this thread's TMEM row.
__device__ __forceinline__ void ld_chunk(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  tmem_ld32(taddr, r);
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// Stores 32 values as bf16 at columns [c0, c0+32) of a K-major tile made of
// [128 x 64] SW128 atoms.
__device__ __forceinline__ void st_chunk_smem(uint32_t tile, uint32_t row, int c0,
                                              const float (&v)[32]) {
  const uint32_t atom = tile + (c0 >> 6) * SLOT;
  const int cc = (c0 & 63) >> 3;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    st_shared_v4(atom + swz_offset(row, cc + c, 128), pack_bf16(v[8 * c + 0], v[8 * c + 1]),
                 pack_bf16(v[8 * c + 2], v[8 * c + 3]), pack_bf16(v[8 * c + 4], v[8 * c + 5]),
                 pack_bf16(v[8 * c + 6], v[8 * c + 7]));
}
// Drains a [128 x FR] fp32 TMEM tile (this thread's row) to bf16 SW128 atoms
// in shared memory, the thread's chunks c = half, half + 2, ... two TMEM loads
// in flight per wait.
template <int FR>
__device__ __forceinline__ void drain_tile(uint32_t taddr, uint32_t tile, uint32_t row,
                                           uint32_t half) {
#pragma unroll
  for (int c = static_cast<int>(half); c < FR / 32; c += 4) {
    uint32_t r0[32], r1[32];
    const bool two = c + 2 < FR / 32;
    tmem_ld32(taddr + c * 32, r0);
    if (two) tmem_ld32(taddr + (c + 2) * 32, r1);
    tmem_ld_wait();
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r0[i]);
    st_chunk_smem(tile, row, c * 32, v);
    if (two) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r1[i]);
      st_chunk_smem(tile, row, (c + 2) * 32, v);
    }
  }
}
__device__ __forceinline__ void st_chunk_global(bf16* dst, const float (&v)[32]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int c = 0; c < 4; ++c)
    d[c] = make_uint4(pack_bf16(v[8 * c + 0], v[8 * c + 1]), pack_bf16(v[8 * c + 2], v[8 * c + 3]),
                      pack_bf16(v[8 * c + 4], v[8 * c + 5]), pack_bf16(v[8 * c + 6], v[8 * c + 7]));
}

#ifdef FSVD_TRACE
__device__ long long g_trace[4096];
}  // namespace
extern "C" __attribute__((visibility("default"))) int fsvd_debug_trace_copy(long long* host, int n) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace, sizeof(long long) * n));
}
extern "C" __attribute__((visibility("default"))) int fsvd_debug_trace_ffn_ln_copy(long long* host, int n) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace_ffn_ln, sizeof(long long) * n));
}
namespace {
#define TRACE(slot) do { if (blockIdx.x == 0) g_trace[(slot)] = clock64(); } while (0)
#else
#define TRACE(slot) do { } while (0)
#endif

template <int FR, bool FUSED, bool WIDE, bool X3 = false>
__global__ void __launch_bounds__(kThreads, 1)
    k_ffn(const __grid_constant__ CUtensorMap tmX,    // X [T, d]        box 128x64 (FUSED)
          const __grid_constant__ CUtensorMap tmP,    // P [T, FR]       box 128x64 (V1)
          const __grid_constant__ CUtensorMap tmUup,  // U_up^T [FR, d]  box PSx64
          const __grid_constant__ CUtensorMap tmVup,  // V_up^T [df, FR] box 128x64
          const __grid_constant__ CUtensorMap tmUdn,  // U_dn^T [FR, df] box PSx64
          const __grid_constant__ CUtensorMap tmVdn,  // V_dn^T [d, FR]  box QSx64
          const __grid_constant__ CUtensorMap tmY,    // out [T, d]      box 128x64 (fused LN)
          const __grid_constant__ CUtensorMap tmR,    // LN residual [T, d] box 128x64 (= X
                                                      // unless pre-LN chaining)
          const float* __restrict__ b_up, const float* __restrict__ b_dn, int act, int T,
          int d_model, int d_ff, bf16* z_out, bf16* out,
          const float* __restrict__ ln_g, const float* __restrict__ ln_b, float ln_eps,
          int split_blocks, float* __restrict__ z_part, const bf16* resid,
          int frk, bf16* sum_out, int64_t z_ps, int rot_mode) {
  static_assert(!(WIDE && FUSED), "wide ranks run the V1 chain");
  using C = FfnCfg<FR, WIDE, X3>;
  CTA_T(0);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays __shared__
  FfnBars* bars = reinterpret_cast<FfnBars*>(smem + C::o_bar);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int m0 = blockIdx.x * BMr;
  // V1 with split_blocks > 0: blockIdx.y streams feature blocks
  // [fb0, fb0 + NB) only and writes an fp32 partial Z (summed by the caller;
  // decode rows use this to spread one row tile's d_ff over many CTAs)
  // blockIdx.y = split * (frk / FR) + slice: the rank slice [zc0, zc0 + FR)
  // of a frk-wide P / Z (frk == FR unless WIDE)
  const int nsl = frk / FR;
  const int zc0 = static_cast<int>(blockIdx.y % nsl) * FR;
  const int split = static_cast<int>(blockIdx.y / nsl);
  const int NK = WIDE ? frk / 64 : C::NATOM;  // K atoms of MMA1
  const int NBall = (d_ff + BF - 1) / BF;
  const int fb0 = split_blocks ? split * split_blocks : 0;
  const int NB = split_blocks ? min(split_blocks, NBall - fb0) : NBall;
  // Loop rotation (FUSED): each tile starts its K-chunk, feature-block and
  // output-piece loops at an offset, so concurrent CTAs read different weight
  // boxes.  rot_mode > 0: 128-row tiles per sequence (FfnTcArgs::seq_tiles),
  // the offset follows the tile's place in its sequence (independent of the
  // batch position); < 0: by CTA index (developer experiment, FSVD_FFN_ROT=1).
  const int rpos = !FUSED || rot_mode == 0 ? 0
                   : rot_mode > 0 ? static_cast<int>(blockIdx.x) % rot_mode
                                  : static_cast<int>(blockIdx.x);
  const int rdiv = rot_mode > 0 ? rot_mode : 1;
  const int rot = rot_mode > 0 ? rpos * NBall / rdiv : rpos % NBall;
  const int rotk = rot_mode > 0 ? rpos * (d_model / 64) / rdiv : rpos;
  auto blk = [&](int f) { return rot ? (f + rot) % NB : f; };
  const int KC = d_model / 64;                        // X K-chunks (FUSED)
  const bool fuse_ln = FUSED && ln_g != nullptr;     // out = LN2(x + ffn(x)) (ln_epi.cuh)
  const int QS = (d_model % 128 == 0 && !fuse_ln) ? 128 : 64;  // output columns per piece
  const int NQ = d_model / QS;
  const int rotq = rot_mode > 0 ? rpos * NQ / rdiv : 0;  // fused-LN output pieces

  if (threadIdx.x == 0) TRACE(0);
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmUup);
    tma_prefetch(&tmVup);
    tma_prefetch(&tmUdn);
    tma_prefetch(&tmVdn);
    if (FUSED) tma_prefetch(&tmX); else tma_prefetch(&tmP);

    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&bars->full[i], 1);
      mbar_init(&bars->empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->x_full[i], 1);
      mbar_init(&bars->x_empty[i], 1);
      mbar_init(&bars->sh_full[i], kEpi);
      mbar_init(&bars->sh_free[i], 1);
      mbar_init(&bars->o_full[i], 1);
      mbar_init(&bars->o_free[i], fuse_ln ? lnepi::acc_drain_arrivals<64>() : kEpi);
      mbar_init(&bars->res_full[i], 1);
      mbar_init(&bars->res_empty[i], lnepi::res_box_readers<64>());
      mbar_init(&bars->box_full[i], lnepi::box_writer_warps<64>());
      mbar_init(&bars->box_free[i], 1);
      mbar_init(&bars->box_full[i + 2], lnepi::box_writer_warps<64>());
      mbar_init(&bars->box_free[i + 2], 1);
    }
    mbar_init(&bars->p_full, 1);
    mbar_init(&bars->p_acc, 1);
    mbar_init(&bars->p_ready, kEpi);
    mbar_init(&bars->h_full, 1);
    mbar_init(&bars->h_free, kEpi);
    mbar_init(&bars->z_full, 1);
    mbar_init(&bars->zs_ready, kEpi);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  pdl_wait();
  CTA_T(1);
  if (threadIdx.x == 0) TRACE(5);
  const uint32_t tmem = bars->tmem;
  uint8_t* ring = smem + C::o_ring;

  if (warp == 0 || warp == 11) {
    // ================================================= TMA producers
    // One thread in each of warps 0 and 11, alternating ring stages: a TMA
    // instruction holds its issuing thread for ~250 cycles whatever the box
    // size (tests/cuda/tma_probe.cu), one issuer cannot feed the MMA.
    if (lane == 0) {
      const uint32_t me = warp == 0 ? 0 : 1;
      uint32_t st = 0, ph = 0, it = 0;
#ifdef FSVD_FFN_EXP
      bool exp_stream = false;  // developer experiment builds only
#endif
      // Streams n slots, two per stage.  slot(i, dst, size_only) returns the
      // byte count of slot i and, unless size_only, issues its TMA.
      auto emit = [&](int n, auto&& slot) {
        for (int i = 0; i < n; i += 2, ++it) {
          if ((it & 1) == me) {
            mbar_wait(&bars->empty[st], ph ^ 1);
#ifdef FSVD_FFN_EXP
            if (FSVD_FFN_EXP == 1 && exp_stream) {  // no refill: MMAs reuse stale stages
              mbar_arrive(&bars->full[st]);
              if (++st == C::STAGES) { st = 0; ph ^= 1; }
              continue;
            }
#endif
            uint8_t* base = ring + st * STAGE;
            uint32_t bytes = slot(i, base, true);
            if (i + 1 < n) bytes += slot(i + 1, base + SLOT, true);
            mbar_arrive_expect_tx(&bars->full[st], bytes);
            slot(i, base, false);
            if (i + 1 < n) slot(i + 1, base + SLOT, false);
          }
          if (++st == C::STAGES) { st = 0; ph ^= 1; }
        }
      };
      auto mma1_slots = [&](int f) {
        if (X3) {  // (P_pl a, V_pl a) for pl = hi, mid, lo: three stages per atom
          emit(6 * NK, [&](int j, uint8_t* dst, bool size_only) -> uint32_t {
            if (!size_only) {
              const int a = j / 6, w = j % 6, pl = w >> 1;
              if (w & 1)
                tma_load_2d(&tmVup, &bars->full[st], dst, a * 64, (fb0 + f) * BF + pl * d_ff);
              else
                tma_load_2d(&tmP, &bars->full[st], dst, a * 64, m0 + pl * T);
            }
            return SLOT;
          });
          return;
        }
        if (WIDE) {  // (P atom a, V_up atom a) per stage
          emit(2 * NK, [&](int j, uint8_t* dst, bool size_only) -> uint32_t {
            if (!size_only) {
              if (j & 1) tma_load_2d(&tmVup, &bars->full[st], dst, (j >> 1) * 64, (fb0 + f) * BF);
              else tma_load_2d(&tmP, &bars->full[st], dst, (j >> 1) * 64, m0);
            }
            return SLOT;
          });
          return;
        }
        emit(C::NATOM, [&](int a, uint8_t* dst, bool size_only) -> uint32_t {
          if (!size_only) tma_load_2d(&tmVup, &bars->full[st], dst, a * 64, (fb0 + blk(f)) * BF);
          return SLOT;
        });
      };
      auto mma2_slots = [&](int f) {  // atom-major: (a0: p0..), (a1: p0..)
        if (X3) {  // per (atom, piece): stages (U_dn_hi, U_dn_mid), (U_dn_lo)
          for (int k = 0; k < 2 * C::NPIECE; ++k) {
            const int a = k / C::NPIECE, p = k % C::NPIECE;
            emit(3, [&](int pl, uint8_t* dst, bool size_only) -> uint32_t {
              if (!size_only)
                tma_load_2d(&tmUdn, &bars->full[st], dst, (fb0 + f) * BF + a * 64,
                            zc0 + p * C::PS + pl * frk);
              return C::PS * 128;
            });
          }
          return;
        }
        emit(2 * C::NPIECE, [&](int j, uint8_t* dst, bool size_only) -> uint32_t {
          const int a = j / C::NPIECE, p = j % C::NPIECE;
          if (!size_only)
            tma_load_2d(&tmUdn, &bars->full[st], dst, (fb0 + blk(f)) * BF + a * 64, zc0 + p * C::PS);
          return C::PS * 128;
        });
      };
      if (FUSED) {
        for (int kc = 0; kc < KC; ++kc) {
          const int xb = kc & 1;
          if (static_cast<uint32_t>(xb) == me) {
            mbar_wait(&bars->x_empty[xb], ((kc >> 1) & 1) ^ 1);
            mbar_arrive_expect_tx(&bars->x_full[xb], SLOT);
            tma_load_2d(&tmX, &bars->x_full[xb], smem + C::o_h + xb * SLOT, ((kc + rotk) % KC) * 64, m0);
          }
          emit(C::NPIECE, [&](int p, uint8_t* dst, bool size_only) -> uint32_t {
            if (!size_only) tma_load_2d(&tmUup, &bars->full[st], dst, ((kc + rotk) % KC) * 64, p * C::PS);
            return C::PS * 128;
          });
        }
      } else if (!WIDE) {
        if (me == 0) mbar_arrive_expect_tx(&bars->p_full, C::NATOM * SLOT);
        for (int a = me; a < C::NATOM; a += 2)
          tma_load_2d(&tmP, &bars->p_full, smem + C::o_p + a * SLOT, a * 64, m0);
      }
      TRACE(2);
      mma1_slots(0);
#ifdef FSVD_FFN_EXP
      exp_stream = true;
#endif
      for (int f = 0; f < NB; ++f) {
        TRACE(2048 + f * 2);
        if (f + 1 < NB) mma1_slots(f + 1);
        TRACE(2048 + f * 2 + 1);
        mma2_slots(f);
      }
#ifdef FSVD_FFN_EXP
      exp_stream = false;
#endif
      if (FUSED) {
        for (int q = 0; q < NQ; ++q)
          emit(C::NATOM, [&](int a, uint8_t* dst, bool size_only) -> uint32_t {
            if (!size_only)
              tma_load_2d(&tmVdn, &bars->full[st], dst, a * 64,
                          (fuse_ln ? lnepi::piece_of(q, NQ, rotq) : q) * QS);
            return QS * 128;
          });
      }
    }
    __syncwarp();
  } else if (warp == 10) {
    // ================================================= residual producer (fused LN2)
    // The H tile is idle once every MMA2 has completed (z_full); the residual
    // (= this tile of X) streams through it as two [128 x 64] boxes.
    if (fuse_ln && lane == 0) {
      mbar_wait_sleep(&bars->z_full, 0, 256);
      lnepi::produce_residual<64>(&tmR, smem + C::o_h, bars->res_full, bars->res_empty, 2,
                                  d_model, m0, rotq);
      // output boxes: 4 staging slots in the weight ring after gamma / beta
      lnepi::store_boxes<64, 4>(&tmY, smem_u32(ring) + kLnStage, bars->box_full, bars->box_free,
                                d_model, m0, rotq);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================================================= MMA issuer
    // Warp-uniform loop (descriptors stay in uniform registers, ~1 issue
    // slot per MMA); one elected lane issues and commits.
    {
      uint32_t st = 0, ph = 0;
      const uint64_t dhi = desc_hi_kmajor(128);
      const uint64_t d_p = desc_at(dhi, smem_u32(smem + C::o_p));
      const uint64_t d_h = desc_at(dhi, smem_u32(smem + C::o_h));
      const uint64_t d_ring = desc_at(dhi, smem_u32(ring));
      auto commit = [&](uint64_t* bar) {
        if (elect_one()) mma_commit(bar);
        __syncwarp();
      };
      // Consumes n slots two per stage: fn(i, slot_desc) issues slot i's MMAs;
      // each stage is released once its MMAs have been issued.
      auto consume = [&](int n, auto&& fn) {
        for (int i = 0; i < n; i += 2) {
          mbar_wait(&bars->full[st], ph);
          tc_fence_after();
          const uint64_t base = d_ring + ((st * STAGE) >> 4);
          fn(i, base);
          if (i + 1 < n) fn(i + 1, base + (SLOT >> 4));
          commit(&bars->empty[st]);
          if (++st == C::STAGES) { st = 0; ph ^= 1; }
        }
      };
      // 4 K-steps of 16 over one 64-wide SW128 atom (start address += 32 B)
      auto mma4 = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, bool acc0) {
        if (elect_one()) {
          mma_bf16_ss(d, a, b, idesc, acc0 ? 1u : 0u);
          mma_bf16_ss(d, a + 2, b + 2, idesc, 1u);
          mma_bf16_ss(d, a + 4, b + 4, idesc, 1u);
          mma_bf16_ss(d, a + 6, b + 6, idesc, 1u);
        }
        __syncwarp();
      };
      constexpr uint32_t kAtom = SLOT >> 4;  // one [128 x 64] atom in descriptor units
      if (FUSED) {
        // P = X U_up into the Z columns of TMEM
        for (int kc = 0; kc < KC; ++kc) {
          const int xb = kc & 1;
          TRACE(3000 + kc * 2);
          mbar_wait(&bars->x_full[xb], (kc >> 1) & 1);
          TRACE(3000 + kc * 2 + 1);
          tc_fence_after();
          consume(C::NPIECE, [&](int p, uint64_t slot) {
            mma4(tmem + C::t_z + p * C::PS, d_h + xb * kAtom, slot, idesc_bf16(128, C::PS),
                 kc != 0);
          });
          commit(&bars->x_empty[xb]);
        }
        commit(&bars->p_acc);
        TRACE(3);
        mbar_wait(&bars->p_ready, 0);
        TRACE(4);
      } else if (!WIDE) {
        mbar_wait(&bars->p_full, 0);
      }
      tc_fence_after();
      auto mma1 = [&](int f) {
        TRACE(64 + f * 8 + 0);
        if (f > 0) {
          mbar_wait(&bars->h_free, (f - 1) & 1);
          tc_fence_after();
        }
        TRACE(64 + f * 8 + 1);
        if (X3) {
          // three stages per atom (plane pl: P at the stage base, V_up one
          // slot on): hold all three, issue the six plane pairs, release
          for (int a = 0; a < NK; ++a) {
            uint32_t sts[3];
            uint64_t sd[3];
            for (int pl = 0; pl < 3; ++pl) {
              sts[pl] = st;
              mbar_wait(&bars->full[st], ph);
              sd[pl] = d_ring + ((st * STAGE) >> 4);
              if (++st == C::STAGES) { st = 0; ph ^= 1; }
            }
            tc_fence_after();
            const uint32_t idh = idesc_bf16(128, BF);
#pragma unroll
            for (int g = 0; g < 6; ++g)
              mma4(tmem + C::t_h, sd[x3_pa(g)], sd[x3_pb(g)] + kAtom, idh, (a | g) != 0);
            for (int pl = 0; pl < 3; ++pl) commit(&bars->empty[sts[pl]]);
          }
        } else if (WIDE) {
          uint64_t pa = 0;
          consume(2 * NK, [&](int j, uint64_t slot) {
            if (j & 1) mma4(tmem + C::t_h, pa, slot, idesc_bf16(128, BF), j > 1);
            else pa = slot;
          });
        } else {
          consume(C::NATOM, [&](int a, uint64_t slot) {
            mma4(tmem + C::t_h, d_p + a * kAtom, slot, idesc_bf16(128, BF), a != 0);
          });
        }
        commit(&bars->h_full);
        TRACE(64 + f * 8 + 2);
      };
      auto mma2 = [&](int f) {
        if (X3) {
          for (int k = 0; k < 2 * C::NPIECE; ++k) {
            const int a = k / C::NPIECE, p = k % C::NPIECE;
            if (p == 0) {
              mbar_wait(&bars->sh_full[a], f & 1);
              tc_fence_after();
            }
            const uint32_t st1 = st;  // (U_hi, U_mid)
            mbar_wait(&bars->full[st], ph);
            const uint64_t s1 = d_ring + ((st * STAGE) >> 4);
            if (++st == C::STAGES) { st = 0; ph ^= 1; }
            const uint32_t st2 = st;  // (U_lo)
            mbar_wait(&bars->full[st], ph);
            const uint64_t s2 = d_ring + ((st * STAGE) >> 4);
            if (++st == C::STAGES) { st = 0; ph ^= 1; }
            tc_fence_after();
            const uint64_t u[3] = {s1, s1 + kAtom, s2};
            const uint32_t idz = idesc_bf16(128, C::PS);
            const uint32_t zt = tmem + C::t_z + p * C::PS;
#pragma unroll
            for (int g = 0; g < 6; ++g)  // H plane x3_pa(g) (atoms 2*pl + a), U plane x3_pb(g)
              mma4(zt, d_h + (2 * x3_pa(g) + a) * kAtom, u[x3_pb(g)], idz, (f | a | g) != 0);
            commit(&bars->empty[st1]);
            commit(&bars->empty[st2]);
            if (p == C::NPIECE - 1) commit(&bars->sh_free[a]);
          }
          return;
        }
        consume(2 * C::NPIECE, [&](int j, uint64_t slot) {
          const int a = j / C::NPIECE, p = j % C::NPIECE;
          if (p == 0) {
            TRACE(64 + f * 8 + 3 + a * 2);
            mbar_wait(&bars->sh_full[a], f & 1);
            tc_fence_after();
            TRACE(64 + f * 8 + 4 + a * 2);
          }
          mma4(tmem + C::t_z + p * C::PS, d_h + a * kAtom, slot, idesc_bf16(128, C::PS),
               (f | a) != 0);
          if (p == C::NPIECE - 1) commit(&bars->sh_free[a]);
        });
      };
      mma1(0);
      for (int f = 0; f < NB; ++f) {
        if (f + 1 < NB) mma1(f + 1);
        mma2(f);
      }
      commit(&bars->z_full);
      if (FUSED) {
        mbar_wait(&bars->zs_ready, 0);
        tc_fence_after();
        for (int q = 0; q < NQ; ++q) {
          if (q >= 2) {
            mbar_wait(&bars->o_free[q & 1], ((q >> 1) - 1) & 1);
            tc_fence_after();
          }
          const uint32_t idq = QS == 128 ? idesc_bf16(128, 128) : idesc_bf16(128, 64);
          consume(C::NATOM, [&](int a, uint64_t slot) {
            mma4(tmem + (q & 1) * QS, d_p + a * kAtom, slot, idq, a != 0);
          });
          commit(&bars->o_full[q & 1]);
        }
      }
    }
  } else {
    // ================================================= epilogue (8 warps)
    const uint32_t quad = warp & 3;
    const uint32_t half = (warp - 2) >> 2;
    const uint32_t row = quad * 32 + lane;
    const uint32_t loff = (quad * 32) << 16;
    const int grow = m0 + static_cast<int>(row);
    const uint32_t s_p = smem_u32(smem + C::o_p), s_h = smem_u32(smem + C::o_h);
    if (FUSED) {
      mbar_wait(&bars->p_acc, 0);
      tc_fence_after();
      drain_tile<FR>(tmem + C::t_z + loff, s_p, row, half);
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->p_ready);
    }
    for (int f = 0; f < NB; ++f) {
      float bb[2][32];  // b_up of this block, fetched while the MMA runs
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int fb = (fb0 + blk(f)) * BF + (half + 2 * i) * 32;
        load_bias<32>(bb[i], b_up + fb, d_ff - fb);
      }
      if (threadIdx.x == 64) TRACE(1024 + f * 8 + 0);
      mbar_wait(&bars->h_full, f & 1);
      tc_fence_after();
      if (threadIdx.x == 64) TRACE(1024 + f * 8 + 1);
      float v[2][32];
#pragma unroll
      for (int i = 0; i < 2; ++i) ld_chunk(tmem + C::t_h + loff + (half + 2 * i) * 32, v[i]);
      tc_fence_before();
      mbar_arrive(&bars->h_free);
#pragma unroll
      for (int i = 0; i < 2; ++i) {  // i = K atom of the H block
        if (X3) bias_act_chunk2_exact<32>(v[i], bb[i], act);
        else bias_act_chunk2<32>(v[i], bb[i], act);
        if (threadIdx.x == 64) TRACE(1024 + f * 8 + 2 + i * 2);
        if (f > 0) mbar_wait(&bars->sh_free[i], (f - 1) & 1);
        if (threadIdx.x == 64) TRACE(1024 + f * 8 + 3 + i * 2);
#ifdef FSVD_FFN_EXP
        if (FSVD_FFN_EXP != 2)
#endif
        st_chunk_smem(s_h, row, (half + 2 * i) * 32, v[i]);
        if (X3) {  // mid and lo planes of the activated block, atoms 2..3 and 4..5
#pragma unroll
          for (int pl = 1; pl < 3; ++pl) {
#pragma unroll
            for (int k = 0; k < 32; ++k) v[i][k] -= bf16_round_f(v[i][k]);
            st_chunk_smem(s_h + 2 * pl * SLOT, row, (half + 2 * i) * 32, v[i]);
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&bars->sh_full[i]);
      }
    }
    mbar_wait(&bars->z_full, 0);
    if (threadIdx.x == 64) TRACE(6);
    tc_fence_after();
    if (!FUSED) {
      for (int c = half; c < FR / 32; c += 2) {
        float v[32];
        ld_chunk(tmem + C::t_z + loff + c * 32, v);
        if (grow >= T) continue;
        if (z_part) {
          float4* d = reinterpret_cast<float4*>(
              z_part + ((int64_t)split * T + grow) * frk + zc0 + c * 32);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            d[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        } else {
          st_chunk_global(z_out + (int64_t)grow * frk + zc0 + c * 32, v);
          if (X3) {
#pragma unroll
            for (int pl = 1; pl < 3; ++pl) {
#pragma unroll
              for (int k = 0; k < 32; ++k) v[k] -= bf16_round_f(v[k]);
              st_chunk_global(z_out + pl * z_ps + (int64_t)grow * frk + zc0 + c * 32, v);
            }
          }
        }
      }
    } else {
      drain_tile<FR>(tmem + C::t_z + loff, s_p, row, half);
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->zs_ready);
      if (threadIdx.x == 64) TRACE(7);
      if (fuse_ln) {
        // residual = the FFN input x, streamed through the idle H tile
        // gamma / beta are staged in the weight ring, idle once all MMAs are done
        lnepi::run<64, 4>(tmem, quad, half, row, d_model, b_dn, smem_u32(smem + C::o_h),
                       bars->res_full, bars->res_empty, 2, ln_g, ln_b, ln_eps, &tmY, m0,
                       reinterpret_cast<float*>(ring), smem_u32(ring) + kLnStage, bars->box_full,
                       bars->box_free, bars->o_full,
                       bars->o_free, 1, 0, sum_out, T, rotq);
      } else {
        for (int q = 0; q < NQ; ++q) {
          mbar_wait(&bars->o_full[q & 1], (q >> 1) & 1);
          tc_fence_after();
          for (int c = half; c < QS / 32; c += 2) {
            float v[32];
            ld_chunk(tmem + (q & 1) * QS + loff + c * 32, v);
            const int n0 = q * QS + c * 32;
            bias_act_chunk<32>(v, b_dn + n0, 32, 3);
            if (grow < T) {
              if (resid) {  // pre-LN layers: out = resid + ffn(x)
                const uint4* rr = reinterpret_cast<const uint4*>(resid + (int64_t)grow * d_model + n0);
#pragma unroll
                for (int q8 = 0; q8 < 4; ++q8) {
                  const uint4 u = rr[q8];
                  const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    v[8 * q8 + 2 * e] += __uint_as_float(w4[e] << 16);
                    v[8 * q8 + 2 * e + 1] += __uint_as_float(w4[e] & 0xffff0000u);
                  }
                }
              }
              st_chunk_global(out + (int64_t)grow * d_model + n0, v);
            }
          }
          tc_fence_before();
          mbar_arrive(&bars->o_free[q & 1]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) TRACE(1);
  if (warp == 1) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
  CTA_T(2);
}

// FR = Z columns per CTA; frk = a.rank_pad (the P / Z width, K of MMA1).
int ffn_rot_mode() {
  static const int m = [] {
    const char* e = getenv("FSVD_FFN_ROT");  // 0 off, 1 by CTA (experiment), 2 by tile in sequence
    return e ? atoi(e) : 2;
  }();
  return m;
}

template <int FR, bool FUSED, bool WIDE = false, bool X3 = false>
void launch_ffn(const FfnTcArgs& a, cudaStream_t s) {
  using C = FfnCfg<FR, WIDE, X3>;
  static bool attr = false;
  if (!attr) {
    FSVD_CUDA_CHECK(cudaFuncSetAttribute(k_ffn<FR, FUSED, WIDE, X3>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  const int frk = a.rank_pad;
  const int boxp = C::PS;
  const int boxd = (a.d_model % 128 == 0) ? 128 : 64;
  const CUtensorMap tup = tmap_bf16(a.up_u_t, frk, a.d_model, a.d_model, boxp, 64, TmaSwizzle::B128);
  // X3: stacked planes (kernels.cuh): V_up^T [3 d_ff, frk], U_dn^T [3 frk, d_ff], P [3T, frk]
  const uint64_t npl = X3 ? 3 : 1;
  const CUtensorMap tvup = tmap_bf16(a.up_v_t, npl * a.d_ff, frk, frk, BF, 64, TmaSwizzle::B128);
  const CUtensorMap tudn = tmap_bf16(a.dn_u_t, npl * frk, a.d_ff, a.d_ff, boxp, 64, TmaSwizzle::B128);
  const CUtensorMap tvdn = tmap_bf16(a.dn_v_t, a.d_model, frk, frk, FUSED && a.ln_g ? 64 : boxd, 64,
                                     TmaSwizzle::B128);
  CUtensorMap tx = tvup, tp = tvup, ty = tvup, tr = tvup;
  if (FUSED && a.ln_g) ty = tmap_bf16(a.out, a.T, a.d_model, a.d_model, 128, 64, TmaSwizzle::B128);
  if (FUSED) {
    tx = tmap_bf16(a.x, a.T, a.d_model, a.d_model, 128, 64, TmaSwizzle::B128);
    tr = a.ln_resid ? tmap_bf16(a.ln_resid, a.T, a.d_model, a.d_model, 128, 64, TmaSwizzle::B128)
                    : tx;
  } else
    tp = tmap_bf16(a.p_in, npl * a.T, frk, frk, 128, 64, TmaSwizzle::B128);
  const int grid = (a.T + BMr - 1) / BMr;
  const int nball = (a.d_ff + BF - 1) / BF;
  const int splits = (!FUSED && a.split_blocks) ? (nball + a.split_blocks - 1) / a.split_blocks : 1;
  launch_pdl(k_ffn<FR, FUSED, WIDE, X3>, dim3(grid, splits * (frk / FR)), dim3(kThreads), C::SMEM,
             s, tx, tp, tup, tvup, tudn, tvdn, ty, tr, a.up_b, a.dn_b, a.act, a.T, a.d_model,
             a.d_ff, a.z_out, a.out, a.ln_g, a.ln_b, a.ln_eps, FUSED ? 0 : a.split_blocks,
             FUSED ? nullptr : a.z_part, FUSED ? a.resid : nullptr, frk,
             FUSED && a.ln_g ? a.sum_out : nullptr, X3 ? (int64_t)a.T * frk : (int64_t)0,
             !FUSED ? 0 : ffn_rot_mode() == 1 ? -1 : ffn_rot_mode() == 0 ? 0 : a.seq_tiles);
  check_launch(FUSED ? "k_ffn_fused" : "k_ffn_stream");
}

template <bool FUSED>
void dispatch_ffn(const FfnTcArgs& a, cudaStream_t s) {
  if (!FUSED && a.planes) {  // split planes (fp32 policy)
    if (a.split_blocks) throw CudaError("ffn (planes): split partials are bf16-only");
    switch (ffn_wide_slice(a.rank_pad)) {
      case 64: launch_ffn<64, false, true, true>(a, s); return;
      case 128: launch_ffn<128, false, true, true>(a, s); return;
      case 192: launch_ffn<192, false, true, true>(a, s); return;
      case 256: launch_ffn<256, false, true, true>(a, s); return;
      case 320: launch_ffn<320, false, true, true>(a, s); return;
      case 384: launch_ffn<384, false, true, true>(a, s); return;
      default: throw CudaError("ffn (planes): unsupported FFN rank padding");
    }
  }
  if (!FUSED && a.rank_pad > 384) {
    static const bool recompute = [] {
      const char* e = getenv("FSVD_FFN_WIDE_RECOMPUTE");
      return e && e[0] == '1';
    }();
    if (!recompute && ffn_wide_cluster_supported(a)) {  // ffn_wide_tc.cu
      ffn_wide_cluster_bf16(a, s);
      return;
    }
    switch (ffn_wide_slice(a.rank_pad)) {
      case 64: launch_ffn<64, false, true>(a, s); return;
      case 128: launch_ffn<128, false, true>(a, s); return;
      case 192: launch_ffn<192, false, true>(a, s); return;
      case 256: launch_ffn<256, false, true>(a, s); return;
      case 320: launch_ffn<320, false, true>(a, s); return;
      case 384: launch_ffn<384, false, true>(a, s); return;
      default: throw CudaError("ffn: unsupported FFN rank padding");
    }
  }
  switch (a.rank_pad) {
    case 64: launch_ffn<64, FUSED>(a, s); break;
    case 128: launch_ffn<128, FUSED>(a, s); break;
    case 192: launch_ffn<192, FUSED>(a, s); break;
    case 256: launch_ffn<256, FUSED>(a, s); break;
    case 320: launch_ffn<320, FUSED>(a, s); break;
    case 384: launch_ffn<384, FUSED>(a, s); break;
    default: throw CudaError("ffn: unsupported FFN rank padding");
  }
}

}  // namespace

// Rank padding: multiples of 64 up to 384 (Z resident in TMEM); above that
// the smallest n * S (S <= 384, a multiple of 64, n slices) covering the rank,
// fewest slices on ties -- e.g. 512 = 2 x 256, 768 = 2 x 384, 1024 = 4 x 256.
int ffn_rank_pad(int fr) {
  const int p64 = (fr + 63) / 64 * 64;
  if (p64 <= 384) return p64;
  const int n0 = (fr + 383) / 384;
  int best = 0;
  for (int n = n0; n <= n0 + 2; ++n) {
    const int sl = ((fr + n - 1) / n + 63) / 64 * 64;
    if (best == 0 || n * sl < best) best = n * sl;
  }
  return best;
}
int ffn_wide_slice(int rank_pad) {
  if (rank_pad <= 384) return rank_pad;
  for (int n = (rank_pad + 383) / 384;; ++n)
    if (rank_pad % n == 0 && (rank_pad / n) % 64 == 0) return rank_pad / n;
}
bool ffn_tc_supported(int d_model, int d_ff, int rank_pad) {
  return d_model % 64 == 0 && d_ff % 8 == 0 && rank_pad % 64 == 0 && rank_pad >= 64 &&
         rank_pad <= kFfnMaxRankPad && ffn_wide_slice(rank_pad) <= 384;
}

void ffn_stream_bf16(const FfnTcArgs& a, cudaStream_t s) { dispatch_ffn<false>(a, s); }
void ffn_fused_bf16(const FfnTcArgs& a, cudaStream_t s) { dispatch_ffn<true>(a, s); }

}  // namespace fsvd
