// ffn_wide_tc.cu -- K3 for FFN ranks above 384 on a cluster of n CTAs.
//
// Same contraction as k_ffn<FR, false> (ffn_tc.cu; stream_feature_blocks,
// ffn.cpp:84-104):
//     Z[tile] = sum_f act(P[tile] V_up[:, f] + b_up[f]) U_down[f, :]
// for ranks whose Z (fr fp32 columns) does not fit TMEM next to the hidden
// block.  The rank is cut into n slices of FR <= 384 columns and the n CTAs
// of a cluster (one per slice) share one 128-row tile: CTA j computes only
// the hidden blocks f = j (mod n) -- P V_up with P streamed through the ring
// next to V_up, bias, activation -- writes each activated block to its own
// shared memory and pushes it to the n - 1 peers with bulk shared::cluster
// copies; every CTA accumulates its Z slice over all blocks.  No hidden block
// is computed twice (the cluster-free WIDE variant of k_ffn recomputes
// P V_up in every slice).
//
// H buffers: two slots (block f uses slot f & 1) of two 64-wide K atoms.
//   sh_loc[s][a]   own block written by the local epilogue (kEpi arrivals)
//   hs_full[s][a]  peer block landed (armed by the MMA issuer, 16 KB of tx)
//   hs_free[f & 3] block f consumed by the MMAs of all n CTAs (multicast
//                  commits).  Four barriers, not one per slot: the producer of
//                  block f waits for block f - 2, and with n > 2 its epilogue
//                  may reach that wait two completions of a per-slot barrier
//                  late (parity aliasing); block f + 2 -- the next completion
//                  of hs_free[(f - 2) & 3] -- cannot be consumed before the
//                  waiter writes block f.
// Warps: 0 and 11 TMA producers, 1 MMA issuer + TMEM owner, 2..9 epilogue,
// 10 relay (bulk copies of the own blocks to the peers).
#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace fsvd {
namespace {

using namespace ptx;

constexpr int kThreads = 384;
constexpr int kEpi = 256;
constexpr int BMr = 128;         // token rows per cluster
constexpr int BF = 128;          // features per block
constexpr int SLOT = BMr * 128;  // one [128 x 64] bf16 SW128 atom / ring slot (16 KB)
constexpr int STAGE = 2 * SLOT;

template <int FR>
struct WideCfg {
  static_assert(FR % 64 == 0 && FR <= 384, "slice width: a multiple of 64, <= 384");
  static constexpr int PS = (FR % 128 == 0) ? 128 : 64;  // Z columns per MMA2 piece
  static constexpr int NPIECE = FR / PS;
  static constexpr int o_h = 0;  // H: 2 slots x 2 atoms
  static constexpr int o_ring = 4 * SLOT;
  static constexpr int STAGES_FIT = (227 * 1024 - 2048 - 4 * SLOT) / STAGE;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int o_bar = o_ring + STAGES * STAGE;
  static constexpr int SMEM = 1024 + o_bar + 512;
  static constexpr int t_z = 0;    // Z slice (FR cols)
  static constexpr int t_h = 384;  // hidden block accumulator (128 cols)
};

struct WideBars {
  uint64_t full[8], empty[8];
  uint64_t h_full, h_free;
  uint64_t sh_loc[2][2], hs_full[2][2], hs_free[4];
  uint64_t z_full;
  uint32_t tmem;
};

__device__ __forceinline__ void ld_chunk(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  tmem_ld32(taddr, r);
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// 32 values as bf16 at columns [c0, c0+32) of a K-major tile of SW128 atoms.
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
__device__ __forceinline__ void st_chunk_global(bf16* dst, const float (&v)[32]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int c = 0; c < 4; ++c)
    d[c] = make_uint4(pack_bf16(v[8 * c + 0], v[8 * c + 1]), pack_bf16(v[8 * c + 2], v[8 * c + 3]),
                      pack_bf16(v[8 * c + 4], v[8 * c + 5]), pack_bf16(v[8 * c + 6], v[8 * c + 7]));
}

template <int FR>
__global__ void __launch_bounds__(kThreads, 1)
    k_ffn_wide(const __grid_constant__ CUtensorMap tmP,    // P [T, frk]        box 128x64
               const __grid_constant__ CUtensorMap tmVup,  // V_up^T [df, frk]  box 128x64
               const __grid_constant__ CUtensorMap tmUdn,  // U_dn^T [frk, df]  box PSx64
               const float* __restrict__ b_up, int act, int T, int d_ff, int frk,
               bf16* __restrict__ z_out) {
  using C = WideCfg<FR>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays __shared__
  WideBars* bars = reinterpret_cast<WideBars*>(smem + C::o_bar);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int rank = static_cast<int>(cluster_rank()), ns = static_cast<int>(cluster_nctarank());
  const int m0 = blockIdx.x * BMr;
  const int zc0 = rank * FR;
  const int NK = frk / 64;                // K atoms of P V_up
  const int NB = (d_ff + BF - 1) / BF;    // hidden blocks
  uint8_t* hbuf = smem + C::o_h;          // slot s, atom a at (2 s + a) * SLOT
  uint8_t* ring = smem + C::o_ring;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmP);
    tma_prefetch(&tmVup);
    tma_prefetch(&tmUdn);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&bars->full[i], 1);
      mbar_init(&bars->empty[i], 1);
    }
    mbar_init(&bars->h_full, 1);
    mbar_init(&bars->h_free, kEpi);
    for (int s = 0; s < 2; ++s) {
      for (int a = 0; a < 2; ++a) {
        mbar_init(&bars->sh_loc[s][a], kEpi);
        mbar_init(&bars->hs_full[s][a], 1);
      }
    }
    for (int i = 0; i < 4; ++i) mbar_init(&bars->hs_free[i], ns);
    mbar_init(&bars->z_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  cluster_sync_all();  // every CTA's barriers exist before the first remote arrival
  // No early pdl_trigger: the grid runs in several waves of clusters, and
  // dependents launched early would take SMs one at a time as CTAs retire,
  // so a later cluster might never find n free SMs together.
  pdl_wait();
  const uint32_t tmem = bars->tmem;

  if (warp == 0 || warp == 11) {
    // ================================================= TMA producers
    if (lane == 0) {
      const uint32_t me = warp == 0 ? 0 : 1;
      uint32_t st = 0, ph = 0, it = 0;
      auto emit = [&](int n, auto&& slot) {
        for (int i = 0; i < n; i += 2, ++it) {
          if ((it & 1) == me) {
            mbar_wait(&bars->empty[st], ph ^ 1);
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
      auto mma1_slots = [&](int f) {  // (P atom a, V_up atom a) per stage
        emit(2 * NK, [&](int j, uint8_t* dst, bool size_only) -> uint32_t {
          if (!size_only) {
            if (j & 1) tma_load_2d(&tmVup, &bars->full[st], dst, (j >> 1) * 64, f * BF);
            else tma_load_2d(&tmP, &bars->full[st], dst, (j >> 1) * 64, m0);
          }
          return SLOT;
        });
      };
      auto mma2_slots = [&](int f) {  // atom-major: (a0: p0..), (a1: p0..)
        emit(2 * C::NPIECE, [&](int j, uint8_t* dst, bool size_only) -> uint32_t {
          const int a = j / C::NPIECE, p = j % C::NPIECE;
          if (!size_only)
            tma_load_2d(&tmUdn, &bars->full[st], dst, f * BF + a * 64, zc0 + p * C::PS);
          return C::PS * 128;
        });
      };
      if (rank < NB) mma1_slots(rank);
      for (int f = 0; f < NB; ++f) {
        if (f % ns == rank && f + ns < NB) mma1_slots(f + ns);
        mma2_slots(f);
      }
    }
    __syncwarp();
  } else if (warp == 10) {
    // ================================================= relay: own blocks -> peers
    if (lane == 0 && ns > 1) {
      uint32_t phs = 0;  // bit s: parity of slot s
      for (int f = rank; f < NB; f += ns) {
        const int s = f & 1;
        for (int a = 0; a < 2; ++a) {
          mbar_wait(&bars->sh_loc[s][a], (phs >> s) & 1);
          uint8_t* src = hbuf + (2 * s + a) * SLOT;
          for (int q = 1; q < ns; ++q) {
            const uint32_t peer = static_cast<uint32_t>((rank + q) % ns);
            bulk_copy_to_peer(mapa_shared(smem_u32(src), peer), src, SLOT,
                              mapa_shared(smem_u32(&bars->hs_full[s][a]), peer));
          }
        }
        phs ^= 1u << s;
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ================================================= MMA issuer
    uint32_t st = 0, ph = 0;
    const uint64_t dhi = desc_hi_kmajor(128);
    const uint64_t d_h = desc_at(dhi, smem_u32(hbuf));
    const uint64_t d_ring = desc_at(dhi, smem_u32(ring));
    const uint16_t mask = static_cast<uint16_t>((1u << ns) - 1);
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) mma_commit(bar);
      __syncwarp();
    };
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
    auto mma4 = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, bool acc0) {
      if (elect_one()) {
        mma_bf16_ss(d, a, b, idesc, acc0 ? 1u : 0u);
        mma_bf16_ss(d, a + 2, b + 2, idesc, 1u);
        mma_bf16_ss(d, a + 4, b + 4, idesc, 1u);
        mma_bf16_ss(d, a + 6, b + 6, idesc, 1u);
      }
      __syncwarp();
    };
    constexpr uint32_t kAtom = SLOT >> 4;
    int kown = 0;
    auto mma1 = [&]() {
      if (kown > 0) {
        mbar_wait(&bars->h_free, (kown - 1) & 1);
        tc_fence_after();
      }
      uint64_t pa = 0;
      consume(2 * NK, [&](int j, uint64_t slot) {
        if (j & 1) mma4(tmem + C::t_h, pa, slot, idesc_bf16(128, BF), j > 1);
        else pa = slot;
      });
      commit(&bars->h_full);
      ++kown;
    };
    uint32_t ph_loc = 0, ph_rem = 0;  // bit s: parity of slot s
    auto mma2 = [&](int f) {
      const int s = f & 1;
      const bool mine = f % ns == rank;
      consume(2 * C::NPIECE, [&](int j, uint64_t slot) {
        const int a = j / C::NPIECE, p = j % C::NPIECE;
        if (p == 0) {
          if (mine) {
            mbar_wait(&bars->sh_loc[s][a], (ph_loc >> s) & 1);
          } else {
            if (elect_one()) mbar_arrive_expect_tx(&bars->hs_full[s][a], SLOT);
            __syncwarp();
            mbar_wait(&bars->hs_full[s][a], (ph_rem >> s) & 1);
          }
          tc_fence_after();
        }
        mma4(tmem + C::t_z + p * C::PS, d_h + (2 * s + a) * kAtom, slot,
             idesc_bf16(128, C::PS), (f | a) != 0);
      });
      if (mine) ph_loc ^= 1u << s;
      else ph_rem ^= 1u << s;
      if (elect_one()) mma_commit_multicast(&bars->hs_free[f & 3], mask);
      __syncwarp();
    };
    if (rank < NB) mma1();
    for (int f = 0; f < NB; ++f) {
      if (f % ns == rank && f + ns < NB) mma1();
      mma2(f);
    }
    commit(&bars->z_full);
  } else {
    // ================================================= epilogue (8 warps)
    const uint32_t quad = warp & 3;
    const uint32_t half = (warp - 2) >> 2;
    const uint32_t row = quad * 32 + lane;
    const uint32_t loff = (quad * 32) << 16;
    const int grow = m0 + static_cast<int>(row);
    int k = 0;
    for (int f = rank; f < NB; f += ns, ++k) {
      float bb[2][32];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int fb = f * BF + (static_cast<int>(half) + 2 * i) * 32;
        load_bias<32>(bb[i], b_up + fb, d_ff - fb);
      }
      mbar_wait(&bars->h_full, k & 1);
      tc_fence_after();
      float v[2][32];
#pragma unroll
      for (int i = 0; i < 2; ++i) ld_chunk(tmem + C::t_h + loff + (half + 2 * i) * 32, v[i]);
      tc_fence_before();
      mbar_arrive(&bars->h_free);
      const int s = f & 1;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        bias_act_chunk2<32>(v[i], bb[i], act);
        if (i == 0 && f >= 2) mbar_wait(&bars->hs_free[(f - 2) & 3], ((f - 2) >> 2) & 1);
        st_chunk_smem(smem_u32(hbuf + 2 * s * SLOT), row, (half + 2 * i) * 32, v[i]);
        fence_proxy_async_smem();
        mbar_arrive(&bars->sh_loc[s][i]);
      }
    }
    mbar_wait(&bars->z_full, 0);
    tc_fence_after();
    for (int c = half; c < FR / 32; c += 2) {
      float v[32];
      ld_chunk(tmem + C::t_z + loff + c * 32, v);
      if (grow < T) st_chunk_global(z_out + (int64_t)grow * frk + zc0 + c * 32, v);
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // peers' copies and multicast arrivals have landed
  if (warp == 1) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

template <int FR>
void launch_wide(const FfnTcArgs& a, int ns, cudaStream_t s) {
  using C = WideCfg<FR>;
  static bool attr = false;
  if (!attr) {
    FSVD_CUDA_CHECK(cudaFuncSetAttribute(k_ffn_wide<FR>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  const int frk = a.rank_pad;
  const CUtensorMap tp = tmap_bf16(a.p_in, a.T, frk, frk, 128, 64, TmaSwizzle::B128);
  const CUtensorMap tvup = tmap_bf16(a.up_v_t, a.d_ff, frk, frk, BF, 64, TmaSwizzle::B128);
  const CUtensorMap tudn = tmap_bf16(a.dn_u_t, frk, a.d_ff, a.d_ff, C::PS, 64, TmaSwizzle::B128);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((a.T + BMr - 1) / BMr, ns);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = static_cast<unsigned>(ns);
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  FSVD_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_ffn_wide<FR>, tp, tvup, tudn, a.up_b, a.act, a.T,
                                     a.d_ff, frk, a.z_out));
  check_launch("k_ffn_wide");
}

}  // namespace

bool ffn_wide_cluster_supported(const FfnTcArgs& a) {
  const int sl = ffn_wide_slice(a.rank_pad);
  const int ns = a.rank_pad / sl;
  return a.rank_pad > 384 && a.split_blocks == 0 && ns >= 2 && ns <= 8 && sl <= 384;
}

void ffn_wide_cluster_bf16(const FfnTcArgs& a, cudaStream_t s) {
  const int sl = ffn_wide_slice(a.rank_pad);
  const int ns = a.rank_pad / sl;
  switch (sl) {
    case 64: launch_wide<64>(a, ns, s); break;
    case 128: launch_wide<128>(a, ns, s); break;
    case 192: launch_wide<192>(a, ns, s); break;
    case 256: launch_wide<256>(a, ns, s); break;
    case 320: launch_wide<320>(a, ns, s); break;
    case 384: launch_wide<384>(a, ns, s); break;
    default: throw CudaError("ffn: unsupported wide-rank slice");
  }
}

}  // namespace fsvd
