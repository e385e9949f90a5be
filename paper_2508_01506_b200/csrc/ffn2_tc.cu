// ffn2_tc.cu -- K4 on a CTA pair: FlashSVD-FFN V2 with cta_group::2 MMAs.
//
// Same dataflow as k_ffn<FR, true> (ffn_tc.cu; ffn_v2, ffn.cpp:158-185):
//     P = X U_up ; Z = sum_f act(P V_up[:, f] + b_up[f]) U_down[f, :] ;
//     out = Z V_down + b_down   (optionally LN(x + out), ln_epi.cuh)
// but a cluster of two CTAs on one TPC owns 256 token rows: each CTA keeps
// its own 128 rows of X, P, H and Z (shared memory / TMEM) and streams only
// HALF of every weight slot; the even CTA issues M = 256 MMAs that read A
// from both CTAs and B (the weights) split between them.  Per SM this halves
// the weight bytes pulled from L2 and the B-operand bytes read from shared
// memory -- the single-CTA kernel is shared-memory-bandwidth bound (N = 128
// SS MMAs alone read 128 B/clk, TMA fills and the H tile come on top).
//
// Barrier ownership: the leader (rank 0) owns every barrier the MMA issuer
// waits on (full, x_full, p_ready, h_free, sh_full, zs_ready, o_free); TMA
// bytes of both CTAs complete on the leader's full barriers and the peer's
// epilogue warps arrive remotely.  Barriers the MMA signals (empty, x_empty,
// p_acc, h_full, sh_free, z_full, o_full) exist in both CTAs and receive a
// multicast commit.
//
// Warps: 0 and 11 TMA producers, 1 MMA issuer (leader) + TMEM owner, 2..9
// epilogue, 10 residual producer of the fused LN.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#ifdef FSVD_TRACE
namespace fsvd { __device__ long long g_trace2_ln[512]; }
#define LN_TRACE(slot) \
  do { if (blockIdx.x == 0 && (slot) < 512) ::fsvd::g_trace2_ln[(slot)] = clock64(); } while (0)
#endif
#include "ln_epi.cuh"
#include "ptx.cuh"

namespace fsvd {
namespace {

using namespace ptx;

constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;
constexpr int BMr = 128;            // token rows per CTA (256 per pair)
constexpr int BF = 128;             // features per block
constexpr int ATOM = BMr * 128;     // [128 x 64] bf16 SW128 atom of own rows (16 KB)
constexpr int HSLOT = 64 * 128;     // ring slot: half of a 128-row weight box (8 KB)
constexpr int STAGE = 2 * HSLOT;
// fused LN2 second sweep: gamma | beta at the ring's start, output staging
// boxes from here on (the ring is idle once the MMAs are done)
constexpr int kLnStage = 8192;

template <int FR>
struct Ffn2Cfg {
  static_assert(FR % 128 == 0 && FR <= 384, "pair FFN: FR in {128, 256, 384}");
  static constexpr int NATOM = FR / 64;
  static constexpr int PS = 128;  // Z / P piece width (pair MMA N)
  static constexpr int NPIECE = FR / PS;
  static constexpr int STAGES_FIT = (227 * 1024 - 2048 - (NATOM + 2) * ATOM) / STAGE;
  static constexpr int STAGES = STAGES_FIT > 12 ? 12 : STAGES_FIT;
  static constexpr int o_p = 0;
  static constexpr int o_h = NATOM * ATOM;
  static constexpr int o_ring = o_h + 2 * ATOM;
  static constexpr int o_bar = o_ring + STAGES * STAGE;
  static constexpr int SMEM = 1024 + o_bar + 1024;
  static constexpr int t_z = 0, t_h = 384;
  static_assert(SMEM <= 227 * 1024, "shared-memory budget");
  static_assert(STAGES * STAGE >= kLnStage + 4 * 128 * 128, "LN output staging in the ring");
};

// P phase: X chunks ([128 x 64] of the own rows) stream through x_slots()
// slots -- the two H atoms, then the P tile's atoms, idle until P is drained
// into them after the last P MMA -- so the loads run that far ahead of the
// MMAs instead of two chunks.
constexpr int kXSlotsMax = 8;
template <int FR>
constexpr int x_slots() { return 2 + FR / 64 < kXSlotsMax ? 2 + FR / 64 : kXSlotsMax; }
template <int FR>
__host__ __device__ constexpr int x_slot_off(int xb) {
  return xb < 2 ? Ffn2Cfg<FR>::o_h + xb * ATOM : Ffn2Cfg<FR>::o_p + (xb - 2) * ATOM;
}

struct Ffn2Bars {
  uint64_t full[12], empty[12];
  uint64_t x_full[kXSlotsMax], x_empty[kXSlotsMax];  // X chunks of the P phase (x_slots)
  uint64_t p_acc, p_ready, h_full, h_free, sh_full[2], sh_free[2], z_full, zs_ready;
  uint64_t sh_loc[2];  // this CTA's epilogue warps -> relay (local, no cluster fence)
  uint64_t o_full[2], o_free[2];
  uint64_t res_full[2], res_empty[2];
  uint64_t box_full[4], box_free[4];  // LN output boxes (ln_epi.cuh store_boxes), ring-staged
  uint32_t tmem;
};
static_assert(sizeof(Ffn2Bars) <= 1024, "barrier block");

__device__ __forceinline__ void ld_chunk(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  tmem_ld32(taddr, r);
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void st_chunk_smem(uint32_t tile, uint32_t row, int c0,
                                              const float (&v)[32]) {
  const uint32_t atom = tile + (c0 >> 6) * ATOM;
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
// Epilogue warp -> leader barrier (after the caller's per-thread fences).
__device__ __forceinline__ void warp_arrive_leader(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive_cluster(mapa_shared(smem_u32(bar), 0));
}
// Same, without release ordering (TMEM-drained signals carry no smem data).
__device__ __forceinline__ void warp_arrive_leader_relaxed(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(bar), 0));
}

#ifdef FSVD_TRACE
__device__ long long g_trace2[8192];
}  // namespace
extern "C" __attribute__((visibility("default"))) int fsvd_debug_trace2_copy(long long* host, int n) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace2, sizeof(long long) * n));
}
extern "C" __attribute__((visibility("default"))) int fsvd_debug_trace2_ln_copy(long long* host, int n) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace2_ln, sizeof(long long) * n));
}
namespace {
// cluster 0 only; slot offset 4096 for the peer CTA
#define TRACE2(slot) do { if (blockIdx.x < 2) g_trace2[(slot) + 4096 * blockIdx.x] = clock64(); } while (0)
#else
#define TRACE2(slot) do { } while (0)
#endif

template <int FR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_ffn2(const __grid_constant__ CUtensorMap tmX,    // X [T, d]        box 128 x 64
           const __grid_constant__ CUtensorMap tmUup,  // U_up^T [FR, d]  box 64 x 64
           const __grid_constant__ CUtensorMap tmVup,  // V_up^T [df, FR] box 64 x 64
           const __grid_constant__ CUtensorMap tmUdn,  // U_dn^T [FR, df] box 64 x 64
           const __grid_constant__ CUtensorMap tmVdn,  // V_dn^T [d, FR]  box QS/2 x 64
           const __grid_constant__ CUtensorMap tmY,    // out [T, d]      box 128 x 64 (LN)
           const __grid_constant__ CUtensorMap tmR,    // residual [T, d] box 128 x 64 (LN; X
                                                       //   post-LN, the residual stream pre-LN)
           const float* __restrict__ b_up, const float* __restrict__ b_dn, int act, int T,
           int d_model, int d_ff, bf16* out, const float* __restrict__ ln_g,
           const float* __restrict__ ln_b, float ln_eps, int seq_pairs, bf16* sum_out) {
  if (threadIdx.x == 0) TRACE2(0);
  using C = Ffn2Cfg<FR>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays __shared__
  Ffn2Bars* bars = reinterpret_cast<Ffn2Bars*>(smem + C::o_bar);
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_rank();
  const int m0 = (blockIdx.x >> 1) * (2 * BMr) + static_cast<int>(rank) * BMr;  // own rows
  const int NB = (d_ff + BF - 1) / BF;
  const int KC = d_model / 64;
  const bool fuse_ln = ln_g != nullptr;
  // Z V_down in N = 128 MMA steps (8 KB weight half-slots).  With the fused
  // LN the epilogue consumes each step as two 64-column pieces, one per warp
  // group and accumulator buffer (ln_epi.cuh run_groups); the next step waits
  // for both groups.
  const int QS = 128;
  const int NQ = d_model / QS;
  const int NQ64 = d_model / 64;  // LN pieces
  // loop rotation by the pair tile's place in its sequence (as k_ffn,
  // FfnTcArgs::seq_tiles): both CTAs of the pair use the same offsets
  const int rpos = seq_pairs > 1 ? static_cast<int>(blockIdx.x >> 1) % seq_pairs : 0;
  const int rdiv = seq_pairs > 1 ? seq_pairs : 1;
  const int rot = rpos * NB / rdiv, rotk = rpos * KC / rdiv;
  // in 64-column LN pieces, even so a step's two pieces stay adjacent
  const int rotq = fuse_ln ? 2 * (rpos * NQ / rdiv) : 0;
  auto blk = [&](int f) { const int b = f + rot; return b >= NB ? b - NB : b; };
  auto kch = [&](int kc) { const int k = kc + rotk; return k >= KC ? k - KC : k; };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmUup);
    tma_prefetch(&tmVup);
    tma_prefetch(&tmUdn);
    tma_prefetch(&tmVdn);
    if (fuse_ln) {
      tma_prefetch(&tmY);
      tma_prefetch(&tmR);
    }
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&bars->full[i], 1);
      mbar_init(&bars->empty[i], 1);
    }
    for (int i = 0; i < x_slots<FR>(); ++i) {
      mbar_init(&bars->x_full[i], 1);
      mbar_init(&bars->x_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->sh_full[i], 2);  // one relay arrival per CTA
      mbar_init(&bars->sh_free[i], 1);
      mbar_init(&bars->sh_loc[i], kEpiWarps);
      mbar_init(&bars->o_full[i], 1);
      // LN epilogue: one warp group per piece (ln_epi.cuh run); plain: all 8 warps
      mbar_init(&bars->o_free[i], fuse_ln ? 2 * (kEpiWarps / 2) : 2 * kEpiWarps);
      mbar_init(&bars->res_full[i], 1);
      mbar_init(&bars->res_empty[i], lnepi::res_box_readers<64>());
      mbar_init(&bars->box_full[i], lnepi::box_writer_warps<64>());
      mbar_init(&bars->box_free[i], 1);
      mbar_init(&bars->box_full[i + 2], lnepi::box_writer_warps<64>());
      mbar_init(&bars->box_free[i + 2], 1);
    }
    mbar_init(&bars->p_acc, 1);
    mbar_init(&bars->p_ready, 2 * kEpiWarps);
    mbar_init(&bars->h_full, 1);
    mbar_init(&bars->h_free, 2 * kEpiWarps);
    mbar_init(&bars->z_full, 1);
    mbar_init(&bars->zs_ready, 2 * kEpiWarps);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_pair<512>(&bars->tmem);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) TRACE2(6);
  const uint32_t tmem = bars->tmem;
  uint8_t* ring = smem + C::o_ring;

  if (warp == 0 || warp == 11) {
    // ================================================= TMA producers (both CTAs)
    if (lane == 0) {
      const uint32_t me = warp == 0 ? 0 : 1;
      uint32_t st = 0, ph = 0, it = 0;
      // n half-slots, two per stage; slot(i, dst) issues half-slot i and
      // returns its bytes.  The leader arms the full barrier for both CTAs.
      auto emit = [&](int n, auto&& slot, uint32_t slot_bytes) {
        for (int i = 0; i < n; i += 2, ++it) {
          if ((it & 1) == me) {
            mbar_wait(&bars->empty[st], ph ^ 1);
            const int k = (i + 1 < n) ? 2 : 1;
            if (rank == 0) mbar_arrive_expect_tx(&bars->full[st], 2 * k * slot_bytes);
            uint8_t* base = ring + st * STAGE;
            slot(i, base);
            if (k == 2) slot(i + 1, base + HSLOT);
          }
          if (++st == C::STAGES) { st = 0; ph ^= 1; }
        }
      };
      const int hr = static_cast<int>(rank) * 64;  // this CTA's half of a 128-row weight box
      for (int kc = 0; kc < KC; ++kc) {
        const int xb = kc % x_slots<FR>();
        if (static_cast<uint32_t>(kc & 1) == me) {
          mbar_wait(&bars->x_empty[xb], ((kc / x_slots<FR>()) & 1) ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&bars->x_full[xb], 2 * ATOM);
          tma_load_2d_pair(&tmX, &bars->x_full[xb], smem + x_slot_off<FR>(xb), kch(kc) * 64, m0);
        }
        emit(C::NPIECE, [&](int p, uint8_t* dst) {
          tma_load_2d_pair(&tmUup, &bars->full[st], dst, kch(kc) * 64, p * C::PS + hr);
        }, HSLOT);
      }
      auto mma1_slots = [&](int f) {
        emit(C::NATOM, [&](int a, uint8_t* dst) {
          tma_load_2d_pair(&tmVup, &bars->full[st], dst, a * 64, blk(f) * BF + hr);
        }, HSLOT);
      };
      auto mma2_slots = [&](int f) {  // atom-major: (a0: p0..), (a1: p0..)
        emit(2 * C::NPIECE, [&](int j, uint8_t* dst) {
          const int a = j / C::NPIECE, p = j % C::NPIECE;
          tma_load_2d_pair(&tmUdn, &bars->full[st], dst, blk(f) * BF + a * 64, p * C::PS + hr);
        }, HSLOT);
      };
      mma1_slots(0);
      for (int f = 0; f < NB; ++f) {
        if (me == 0) TRACE2(2048 + f * 2);
        if (f + 1 < NB) mma1_slots(f + 1);
        if (me == 0) TRACE2(2048 + f * 2 + 1);
        mma2_slots(f);
      }
      for (int q = 0; q < NQ; ++q)
        emit(C::NATOM, [&](int a, uint8_t* dst) {
          tma_load_2d_pair(&tmVdn, &bars->full[st], dst, a * 64,
                           lnepi::piece_of(2 * q, NQ64, rotq) * 64 +
                               static_cast<int>(rank) * (QS / 2));
        }, (QS / 2) * 128);
    }
    __syncwarp();
  } else if (warp == 10) {
    // ================================================= relay + residual producer
    // Stream phase: the epilogue warps of this CTA arrive locally on sh_loc;
    // this lane forwards ONE release.cluster arrival per H atom to the
    // leader, so the cluster-scope fence is paid once per atom instead of on
    // every epilogue warp's critical path.
    if (lane == 0) {
      for (int f = 0; f < NB; ++f)
        for (int a = 0; a < 2; ++a) {
          mbar_wait(&bars->sh_loc[a], f & 1);
          TRACE2(3000 + f * 4 + a * 2);
          mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&bars->sh_full[a]), 0));
          TRACE2(3001 + f * 4 + a * 2);
        }
    }
    __syncwarp();
    if (fuse_ln && lane == 0) {
      mbar_wait(&bars->z_full, 0);
      lnepi::produce_residual<64>(&tmR, smem + C::o_h, bars->res_full, bars->res_empty, 2,
                                  d_model, m0, rotq);
      // output boxes: 4 staging slots in the weight ring after gamma / beta
      lnepi::store_boxes<64, 4>(&tmY, smem_u32(ring) + kLnStage, bars->box_full, bars->box_free,
                                d_model, m0, rotq);
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================================================= MMA issuer (leader only)
    if (rank == 0) {
      uint32_t st = 0, ph = 0;
      const uint64_t dhi = desc_hi_kmajor(128);
      const uint64_t d_p = desc_at(dhi, smem_u32(smem + C::o_p));
      const uint64_t d_h = desc_at(dhi, smem_u32(smem + C::o_h));
      const uint64_t d_ring = desc_at(dhi, smem_u32(ring));
      auto commit = [&](uint64_t* bar) {
        if (elect_one()) mma_commit_pair(bar, 0x3);
        __syncwarp();
      };
      auto consume = [&](int n, auto&& fn) {
        for (int i = 0; i < n; i += 2) {
          mbar_wait(&bars->full[st], ph);
          tc_fence_after();
          const uint64_t base = d_ring + ((st * STAGE) >> 4);
          fn(i, base);
          if (i + 1 < n) fn(i + 1, base + (HSLOT >> 4));
          commit(&bars->empty[st]);
          if (++st == C::STAGES) { st = 0; ph ^= 1; }
        }
      };
      auto mma4 = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, bool acc0) {
        if (elect_one()) {
          mma_bf16_ss_pair(d, a, b, idesc, acc0 ? 1u : 0u);
          mma_bf16_ss_pair(d, a + 2, b + 2, idesc, 1u);
          mma_bf16_ss_pair(d, a + 4, b + 4, idesc, 1u);
          mma_bf16_ss_pair(d, a + 6, b + 6, idesc, 1u);
        }
        __syncwarp();
      };
      constexpr uint32_t kAtom = ATOM >> 4;
      constexpr uint32_t id128 = idesc_bf16(2 * BMr, 128);
      // P = X U_up into the Z columns
      const uint64_t d_x0 = desc_at(dhi, smem_u32(smem));
      for (int kc = 0; kc < KC; ++kc) {
        const int xb = kc % x_slots<FR>();
        mbar_wait(&bars->x_full[xb], (kc / x_slots<FR>()) & 1);
        tc_fence_after();
        const uint64_t dx = d_x0 + (x_slot_off<FR>(xb) >> 4);
        consume(C::NPIECE, [&](int p, uint64_t slot) {
          mma4(tmem + C::t_z + p * C::PS, dx, slot, id128, kc != 0);
        });
        commit(&bars->x_empty[xb]);
      }
      commit(&bars->p_acc);
      TRACE2(7);
      mbar_wait(&bars->p_ready, 0);
      tc_fence_after();
      auto mma1 = [&](int f) {
        TRACE2(64 + f * 8 + 0);
        if (f > 0) {
          mbar_wait(&bars->h_free, (f - 1) & 1);
          tc_fence_after();
        }
        TRACE2(64 + f * 8 + 1);
        consume(C::NATOM, [&](int a, uint64_t slot) {
          mma4(tmem + C::t_h, d_p + a * kAtom, slot, id128, a != 0);
        });
        commit(&bars->h_full);
        TRACE2(64 + f * 8 + 2);
      };
      auto mma2 = [&](int f) {
        consume(2 * C::NPIECE, [&](int j, uint64_t slot) {
          const int a = j / C::NPIECE, p = j % C::NPIECE;
          if (p == 0) {
            TRACE2(64 + f * 8 + 3 + a * 2);
            mbar_wait(&bars->sh_full[a], f & 1);
            tc_fence_after();
            TRACE2(64 + f * 8 + 4 + a * 2);
          }
          mma4(tmem + C::t_z + p * C::PS, d_h + a * kAtom, slot, id128, (f | a) != 0);
          if (p == C::NPIECE - 1) commit(&bars->sh_free[a]);
        });
      };
      mma1(0);
      for (int f = 0; f < NB; ++f) {
        if (f + 1 < NB) mma1(f + 1);
        mma2(f);
      }
      commit(&bars->z_full);
      TRACE2(2);
      mbar_wait(&bars->zs_ready, 0);
      tc_fence_after();
      TRACE2(3);
      const uint32_t idq = idesc_bf16(2 * BMr, 128);
      for (int q = 0; q < NQ; ++q) {
        if (fuse_ln) {
          // one 128-column step fills both 64-column LN buffers: both groups
          // must have drained the previous step
          if (q >= 1) {
            mbar_wait(&bars->o_free[0], (q - 1) & 1);
            mbar_wait(&bars->o_free[1], (q - 1) & 1);
            tc_fence_after();
          }
          consume(C::NATOM, [&](int a, uint64_t slot) {
            mma4(tmem, d_p + a * kAtom, slot, idq, a != 0);
          });
          commit(&bars->o_full[0]);
          commit(&bars->o_full[1]);
        } else {
          if (q >= 2) {
            mbar_wait(&bars->o_free[q & 1], ((q >> 1) - 1) & 1);
            tc_fence_after();
          }
          consume(C::NATOM, [&](int a, uint64_t slot) {
            mma4(tmem + (q & 1) * QS, d_p + a * kAtom, slot, idq, a != 0);
          });
          commit(&bars->o_full[q & 1]);
        }
      }
    }
  } else {
    // ================================================= epilogue (8 warps, own rows)
    const uint32_t quad = warp & 3;
    const uint32_t half = (warp - 2) >> 2;
    const uint32_t row = quad * 32 + lane;
    const uint32_t loff = (quad * 32) << 16;
    const int grow = m0 + static_cast<int>(row);
    const uint32_t s_p = smem_u32(smem + C::o_p), s_h = smem_u32(smem + C::o_h);
    mbar_wait(&bars->p_acc, 0);
    tc_fence_after();
    drain_tile<FR>(tmem + C::t_z + loff, s_p, row, half);
    fence_proxy_async_smem();
    tc_fence_before();
    warp_arrive_leader(&bars->p_ready);
    for (int f = 0; f < NB; ++f) {
      float bb[2][32];  // b_up of this block, fetched while the MMA runs
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int fb = blk(f) * BF + (half + 2 * i) * 32;
        load_bias<32>(bb[i], b_up + fb, d_ff - fb);
      }
      if (threadIdx.x == 64) TRACE2(1024 + f * 8 + 0);
      mbar_wait(&bars->h_full, f & 1);
      tc_fence_after();
      if (threadIdx.x == 64) TRACE2(1024 + f * 8 + 1);
      float v[2][32];
#pragma unroll
      for (int i = 0; i < 2; ++i) ld_chunk(tmem + C::t_h + loff + (half + 2 * i) * 32, v[i]);
      tc_fence_before();
      warp_arrive_leader_relaxed(&bars->h_free);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        bias_act_chunk2<32>(v[i], bb[i], act);
        if (threadIdx.x == 64) TRACE2(1024 + f * 8 + 2 + i * 2);
        if (f > 0) mbar_wait(&bars->sh_free[i], (f - 1) & 1);
        if (threadIdx.x == 64) TRACE2(1024 + f * 8 + 3 + i * 2);
        st_chunk_smem(s_h, row, (half + 2 * i) * 32, v[i]);
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->sh_loc[i]);
      }
    }
    mbar_wait(&bars->z_full, 0);
    tc_fence_after();
    drain_tile<FR>(tmem + C::t_z + loff, s_p, row, half);
    fence_proxy_async_smem();
    tc_fence_before();
    warp_arrive_leader(&bars->zs_ready);
    if (fuse_ln) {
      lnepi::run<64, 4>(tmem, quad, half, row, d_model, b_dn, smem_u32(smem + C::o_h),
                     bars->res_full, bars->res_empty, 2, ln_g, ln_b, ln_eps, &tmY, m0,
                     reinterpret_cast<float*>(ring), smem_u32(ring) + kLnStage, bars->box_full,
                     bars->box_free, bars->o_full,
                     bars->o_free, 1,
                     mapa_shared(smem_u32(&bars->o_free[0]), 0), sum_out, T, rotq);
    } else {
      for (int q = 0; q < NQ; ++q) {
        mbar_wait(&bars->o_full[q & 1], (q >> 1) & 1);
        tc_fence_after();
        for (int c = half; c < QS / 32; c += 2) {
          float v[32];
          ld_chunk(tmem + (q & 1) * QS + loff + c * 32, v);
          const int n0 = q * QS + c * 32;
          bias_act_chunk<32>(v, b_dn + n0, 32, 3);
          if (grow < T) st_chunk_global(out + (int64_t)grow * d_model + n0, v);
        }
        tc_fence_before();
        warp_arrive_leader(&bars->o_free[q & 1]);
      }
    }
  }
  if (threadIdx.x == 0 || threadIdx.x == 64) TRACE2(1 + (threadIdx.x == 64 ? 4 : 0));
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_free_pair<512>(tmem);
  }
}

bool ffn_pair_rotation() {
  static const bool on = [] {
    const char* e = getenv("FSVD_FFN_ROT");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int FR>
void launch_ffn2(const FfnTcArgs& a, cudaStream_t s) {
  using C = Ffn2Cfg<FR>;
  static bool attr = false;
  if (!attr) {
    FSVD_CUDA_CHECK(cudaFuncSetAttribute(k_ffn2<FR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::SMEM));
    attr = true;
  }
  const bool ln = a.ln_g != nullptr;
  const CUtensorMap tx = tmap_bf16(a.x, a.T, a.d_model, a.d_model, BMr, 64, TmaSwizzle::B128);
  const CUtensorMap tup = tmap_bf16(a.up_u_t, FR, a.d_model, a.d_model, 64, 64, TmaSwizzle::B128);
  const CUtensorMap tvup = tmap_bf16(a.up_v_t, a.d_ff, FR, FR, 64, 64, TmaSwizzle::B128);
  const CUtensorMap tudn = tmap_bf16(a.dn_u_t, FR, a.d_ff, a.d_ff, 64, 64, TmaSwizzle::B128);
  const CUtensorMap tvdn = tmap_bf16(a.dn_v_t, a.d_model, FR, FR, 64, 64, TmaSwizzle::B128);
  const CUtensorMap ty =
      ln ? tmap_bf16(a.out, a.T, a.d_model, a.d_model, BMr, 64, TmaSwizzle::B128) : tx;
  // pre-LN chains: the LN2 epilogue adds the residual stream (ln_resid), not
  // X, and stores the un-normalised sum to sum_out (the single K4's contract)
  const CUtensorMap tr = ln && a.ln_resid
                             ? tmap_bf16(a.ln_resid, a.T, a.d_model, a.d_model, BMr, 64, TmaSwizzle::B128)
                             : tx;
  const int pairs = (a.T + 2 * BMr - 1) / (2 * BMr);
  launch_pdl(k_ffn2<FR>, dim3(2 * pairs), dim3(kThreads), C::SMEM, s, tx, tup, tvup, tudn, tvdn,
             ty, tr, a.up_b, a.dn_b, a.act, a.T, a.d_model, a.d_ff, a.out, a.ln_g, a.ln_b, a.ln_eps,
             ffn_pair_rotation() && a.seq_tiles % 2 == 0 ? a.seq_tiles / 2 : 0,
             ln ? a.sum_out : nullptr);
  check_launch("k_ffn2");
}

}  // namespace

bool ffn_pair_supported(int d_model, int d_ff, int rank_pad) {
  return d_model % 128 == 0 && d_ff % 128 == 0 && rank_pad % 128 == 0 && rank_pad <= 384;
}

void ffn_fused_pair_bf16(const FfnTcArgs& a, cudaStream_t s) {
  switch (a.rank_pad) {
    case 128: launch_ffn2<128>(a, s); break;
    case 256: launch_ffn2<256>(a, s); break;
    case 384: launch_ffn2<384>(a, s); break;
    default: throw CudaError("ffn_fused_pair_bf16: unsupported FFN rank padding");
  }
}

}  // namespace fsvd
