// attn_tc.cu -- K2: FlashSVD attention on tcgen05, rank-space streaming.
//
// Replaces flash_svd_attention's per-head stream (attention.cpp:249-267 and
// online_softmax_head :92-137).  The reference rebuilds head-width Q, K, V
// tiles from the rank-r activations P = X U and the factor slices V (bias
// preloaded, :254-264) and runs an online softmax over key tiles.  Here the
// same algebra runs with the factors folded on chip:
//
//   Q   = (P_q Vq + b_q) * scale*log2e          tcgen05, M=128 N=64  K=r
//   Qt  = Q Vk^T                                tcgen05, M=128 N=r   K=64
//   S_j = Qt P_k,j^T  (= Q K_j^T - Q b_k 1^T)   tcgen05, M=128 N=128 K=r
//   online softmax over j (exp2), P_j -> smem bf16
//   O  <- O * alpha_j  (rank-width TMEM rescale by the softmax threads)
//   O += P_j P_v,j                              tcgen05, M=128 N=r   K=128
//   ctx = (O / l) Vv + b_v                      tcgen05, M=128 N=64  K=r
//
// The K bias only adds the per-row constant Q.b_k to every score, which the
// softmax cancels; the V bias passes through because softmax rows sum to one.
// So no head-width K or V tile is ever formed, P_k / P_v tiles stream straight
// from HBM by TMA, and dense Q/K/V never exist in HBM.
//
// CTA = one (batch, head) and TWO 128-row query tiles.  Warps 0-3 and 4-7 are
// two softmax groups (thread = query row, TMEM lane quadrant warp%4), one per
// query tile, so every SM sub-partition runs two softmax warps whose exp2
// streams interleave on the MUFU pipe; each K/V tile is loaded once for both
// query tiles.  Warp 8 is the TMA producer, warp 9 the MMA issuer and TMEM
// owner.  Per group, TMEM holds S (128 cols), the rank-width O accumulator
// (r cols) and the Q / output accumulator (64 cols).
#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace fsvd {
namespace {

using namespace ptx;

constexpr int kThreads = 320;
constexpr int QT = 128;  // query rows per group
constexpr int KT = 128;  // keys per tile
constexpr int DH = 64;   // head dim
constexpr int kTma = 8, kMma = 9;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__host__ __device__ constexpr int up1k(int x) { return (x + 1023) / 1024 * 1024; }

template <int RP>
struct AttnCfg {
  static constexpr int STAGES = RP >= 64 ? 2 : 3;
  static constexpr int RB = RP * 2;            // bytes per rank-width row
  static constexpr int PQ = QT * RB;           // one P_q tile
  static constexpr int VQ = DH * RB, VK = RP * DH * 2, VV = DH * RB;
  static constexpr int SQT = QT * RB;
  static constexpr int KV = KT * RB;           // one of P_k / P_v
  static constexpr int SP = QT * KT * 2;       // probabilities (also holds Q bf16)
  static constexpr int o_pq = 0;               // 2 tiles
  static constexpr int o_vq = o_pq + 2 * up1k(PQ);
  static constexpr int o_vk = o_vq + up1k(VQ);
  static constexpr int o_vv = o_vk + up1k(VK);
  static constexpr int o_qt = o_vv + up1k(VV);  // 2 tiles
  static constexpr int o_kv = o_qt + 2 * up1k(SQT);
  static constexpr int KV_STAGE = 2 * up1k(KV);
  static constexpr int o_p = o_kv + STAGES * KV_STAGE;  // 2 tiles
  static constexpr int o_bar = o_p + 2 * SP;
  static constexpr int SMEM = 1024 + o_bar + 512;
  // TMEM columns, relative to group base g*256
  static constexpr int t_s = 0;
  static constexpr int t_o = 128;           // PV result (also Qt accumulator in the prologue)
  static constexpr int t_q = 128 + RP;      // Q accumulator / final output (64 cols)
  static_assert(t_q + 64 <= 256, "TMEM budget per group");
  static_assert(SMEM <= 232448, "shared memory budget");
};

struct Bars {
  uint64_t pro;
  uint64_t kv_full[3], kv_empty[3];
  uint64_t q_done[2], qs[2], qt_done[2], qts[2];
  uint64_t s_full[2], s_free[2], p_full[2], o_full[2], o_free[2], ofin[2], out_done[2];
  uint32_t tmem;
};

template <int RP>
__device__ __forceinline__ void ld_rank(uint32_t taddr, float (&o)[RP]) {
  if constexpr (RP == 16) {
    uint32_t r[16];
    tmem_ld16(taddr, r);
    tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i] = __uint_as_float(r[i]);
  } else {
#pragma unroll
    for (int c = 0; c < RP; c += 32) {
      uint32_t r[32];
      tmem_ld32(taddr + c, r);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) o[c + i] = __uint_as_float(r[i]);
    }
  }
}

// Writes N floats of one row as bf16 into a K-major swizzled tile whose rows
// are N*2 bytes long (N in {16, 32, 64}).
template <int N>
__device__ __forceinline__ void store_row_bf16(uint32_t tile, uint32_t row, const float* v) {
  constexpr uint32_t RB = N * 2;
#pragma unroll
  for (int c = 0; c < N / 8; ++c)
    st_shared_v4(tile + swz_offset(row, c, RB), pack_bf16(v[8 * c + 0], v[8 * c + 1]),
                 pack_bf16(v[8 * c + 2], v[8 * c + 3]), pack_bf16(v[8 * c + 4], v[8 * c + 5]),
                 pack_bf16(v[8 * c + 6], v[8 * c + 7]));
}

template <int RP>
__global__ void __launch_bounds__(kThreads, 1)
    k_attn_rankspace(const __grid_constant__ CUtensorMap tmP,
                     const __grid_constant__ CUtensorMap tmVq,
                     const __grid_constant__ CUtensorMap tmVk,
                     const __grid_constant__ CUtensorMap tmVv, const float* __restrict__ bq,
                     const float* __restrict__ bv, float q_scale, bf16* __restrict__ ctx,
                     int64_t ldc, int seq, int heads, int groups) {
  using C = AttnCfg<RP>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  Bars* bars = reinterpret_cast<Bars*>(smem + C::o_bar);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int h = blockIdx.y, b = blockIdx.z;
  const int g_of_h = h / (heads / groups);
  const int row0 = b * seq;                       // first token row of this sequence
  const int qbase = blockIdx.x * 2 * QT;          // first query of group 0
  const int ng = (qbase + QT < seq) ? 2 : 1;      // active query groups
  const int nj = (seq + KT - 1) / KT;

  if (warp == kTma && lane == 0) {
    tma_prefetch(&tmP);
    tma_prefetch(&tmVq);
    tma_prefetch(&tmVk);
    tma_prefetch(&tmVv);
    mbar_init(&bars->pro, 1);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&bars->q_done[g], 1);
      mbar_init(&bars->qs[g], 128);
      mbar_init(&bars->qt_done[g], 1);
      mbar_init(&bars->qts[g], 128);
      mbar_init(&bars->s_full[g], 1);
      mbar_init(&bars->s_free[g], 128);
      mbar_init(&bars->p_full[g], 128);
      mbar_init(&bars->o_full[g], 1);
      mbar_init(&bars->o_free[g], 128);
      mbar_init(&bars->ofin[g], 128);
      mbar_init(&bars->out_done[g], 1);
    }
    fence_barrier_init();
  }
  if (warp == kMma) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem;
  const uint32_t s_pq = smem_u32(smem + C::o_pq), s_vq = smem_u32(smem + C::o_vq);
  const uint32_t s_vk = smem_u32(smem + C::o_vk), s_vv = smem_u32(smem + C::o_vv);
  const uint32_t s_qt = smem_u32(smem + C::o_qt), s_kv = smem_u32(smem + C::o_kv);
  const uint32_t s_p = smem_u32(smem + C::o_p);

  if (warp == kTma) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars->pro, ng * C::PQ + C::VQ + C::VK + C::VV);
      for (int g = 0; g < ng; ++g)
        tma_load_2d(&tmP, &bars->pro, smem + C::o_pq + g * up1k(C::PQ), g_of_h * RP,
                    row0 + qbase + g * QT);
      tma_load_2d(&tmVq, &bars->pro, smem + C::o_vq, 0, h * DH);
      tma_load_2d(&tmVk, &bars->pro, smem + C::o_vk, 0, h * RP);
      tma_load_2d(&tmVv, &bars->pro, smem + C::o_vv, 0, h * DH);
    }
    __syncwarp();
    uint32_t st = 0, ph = 0;
    for (int j = 0; j < nj; ++j) {
      mbar_wait(&bars->kv_empty[st], ph ^ 1);
      if (lane == 0) {
        uint8_t* kv = smem + C::o_kv + st * C::KV_STAGE;
        mbar_arrive_expect_tx(&bars->kv_full[st], 2 * C::KV);
        tma_load_2d(&tmP, &bars->kv_full[st], kv, (groups + g_of_h) * RP, row0 + j * KT);
        tma_load_2d(&tmP, &bars->kv_full[st], kv + up1k(C::KV), (2 * groups + g_of_h) * RP,
                    row0 + j * KT);
      }
      __syncwarp();
      if (++st == C::STAGES) { st = 0; ph ^= 1; }
    }
  } else if (warp == kMma) {
    // ------------------------------------------------ MMA issuer
    mbar_wait(&bars->pro, 0);
    tc_fence_after();
    if (lane == 0) {
      for (int g = 0; g < ng; ++g) {  // Q = P_q Vq  (M=128, N=64, K=RP)
#pragma unroll
        for (int k = 0; k < RP / 16; ++k)
          mma_bf16_ss(tmem + g * 256 + C::t_q,
                      desc_kmajor(s_pq + g * up1k(C::PQ) + k * 32, C::RB),
                      desc_kmajor(s_vq + k * 32, C::RB), idesc_bf16(128, DH), k != 0);
        mma_commit(&bars->q_done[g]);
      }
    }
    __syncwarp();
    for (int g = 0; g < ng; ++g) {  // Qt = Q Vk^T (M=128, N=RP, K=64); Q bf16 sits in the P tile
      mbar_wait(&bars->qs[g], 0);
      tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < DH / 16; ++k)
          mma_bf16_ss(tmem + g * 256 + C::t_o, desc_kmajor(s_p + g * C::SP + k * 32, 128),
                      desc_kmajor(s_vk + k * 32, 128), idesc_bf16(128, RP), k != 0);
        mma_commit(&bars->qt_done[g]);
      }
      __syncwarp();
    }
    for (int g = 0; g < ng; ++g) mbar_wait(&bars->qts[g], 0);
    tc_fence_after();

    auto issue_s = [&](int g, int j) {
      const uint32_t st = j % C::STAGES;
      if (g == 0) mbar_wait(&bars->kv_full[st], (j / C::STAGES) & 1);
      if (j > 0) mbar_wait(&bars->s_free[g], (j - 1) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t pk = s_kv + st * C::KV_STAGE;
#pragma unroll
        for (int k = 0; k < RP / 16; ++k)
          mma_bf16_ss(tmem + g * 256 + C::t_s,
                      desc_kmajor(s_qt + g * up1k(C::SQT) + k * 32, C::RB),
                      desc_kmajor(pk + k * 32, C::RB), idesc_bf16(128, KT), k != 0);
        mma_commit(&bars->s_full[g]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int g, int j) {
      const uint32_t st = j % C::STAGES;
      mbar_wait(&bars->p_full[g], j & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t pv = s_kv + st * C::KV_STAGE + up1k(C::KV);
        const uint32_t pa = s_p + g * C::SP;
#pragma unroll
        for (int k = 0; k < KT / 16; ++k)
          mma_bf16_ss(tmem + g * 256 + C::t_o,
                      desc_kmajor(pa + (k >> 2) * (QT * 128) + (k & 3) * 32, 128),
                      desc_mnmajor(pv + k * 16 * C::RB, C::RB), idesc_bf16(128, RP, 0, 1),
                      (j | k) != 0);
        mma_commit(&bars->o_full[g]);
      }
      __syncwarp();
    };
    for (int g = 0; g < ng; ++g) issue_s(g, 0);
    for (int j = 0; j < nj; ++j) {
      if (j + 1 < nj)
        for (int g = 0; g < ng; ++g) issue_s(g, j + 1);
      for (int g = 0; g < ng; ++g) issue_pv(g, j);
      if (lane == 0) mma_commit(&bars->kv_empty[j % C::STAGES]);
      __syncwarp();
    }
    for (int g = 0; g < ng; ++g) {  // ctx = O Vv (M=128, N=64, K=RP), O staged in the Qt tile
      mbar_wait(&bars->ofin[g], 0);
      tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < RP / 16; ++k)
          mma_bf16_ss(tmem + g * 256 + C::t_q,
                      desc_kmajor(s_qt + g * up1k(C::SQT) + k * 32, C::RB),
                      desc_kmajor(s_vv + k * 32, C::RB), idesc_bf16(128, DH), k != 0);
        mma_commit(&bars->out_done[g]);
      }
      __syncwarp();
    }
  } else if (warp < 8) {
    // ------------------------------------------------ softmax / epilogue groups
    const int g = warp >> 2;
    if (g < ng) {
      const uint32_t quad = warp & 3;
      const uint32_t row = quad * 32 + lane;  // query row within the group's tile
      const uint32_t tg = tmem + g * 256 + ((quad * 32) << 16);
      const uint32_t my_p = s_p + g * C::SP;
      const uint32_t my_qt = s_qt + g * up1k(C::SQT);

      // Q epilogue: bias, softmax scale (log2 domain), bf16 -> smem (P tile slot)
      mbar_wait(&bars->q_done[g], 0);
      tc_fence_after();
      {
        float qv[DH];
#pragma unroll
        for (int c = 0; c < DH; c += 32) {
          uint32_t r[32];
          tmem_ld32(tg + C::t_q + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i)
            qv[c + i] = (__uint_as_float(r[i]) + __ldg(bq + h * DH + c + i)) * q_scale;
        }
        store_row_bf16<DH>(my_p, row, qv);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->qs[g]);
      // Qt epilogue
      mbar_wait(&bars->qt_done[g], 0);
      tc_fence_after();
      {
        float t[RP];
        ld_rank<RP>(tg + C::t_o, t);
        store_row_bf16<RP>(my_qt, row, t);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->qts[g]);

      float m_run = -INFINITY, l_run = 0.0f;

      // O lives in TMEM and accumulates across key tiles (PV MMAs accumulate);
      // before PV_j the running O is rescaled by alpha_j here (correction).
      auto rescale_o = [&](float alpha) {
#pragma unroll
        for (int c = 0; c < RP; c += 16) {
          uint32_t r[16];
          tmem_ld16(tg + C::t_o + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
          tmem_st16(tg + C::t_o + c, r);
        }
        tmem_st_wait();
      };

      for (int j = 0; j < nj; ++j) {
        mbar_wait(&bars->s_full[g], j & 1);
        tc_fence_after();
        float s[KT];
#pragma unroll
        for (int c = 0; c < KT; c += 32) {
          uint32_t r[32];
          tmem_ld32(tg + C::t_s + c, r);
#pragma unroll
          for (int i = 0; i < 32; ++i) s[c + i] = __uint_as_float(r[i]);
        }
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&bars->s_free[g]);
        const int valid = seq - j * KT;  // keys of this tile inside the sequence
        float tmax = -INFINITY;
        if (valid >= KT) {
#pragma unroll
          for (int i = 0; i < KT; ++i) tmax = fmaxf(tmax, s[i]);
        } else {
#pragma unroll
          for (int i = 0; i < KT; ++i) s[i] = (i < valid) ? s[i] : -INFINITY;
#pragma unroll
          for (int i = 0; i < KT; ++i) tmax = fmaxf(tmax, s[i]);
        }
        const float m_new = fmaxf(m_run, tmax);
        const float alpha = ex2(m_run - m_new);
        m_run = m_new;
        // single-buffered probability tile and O accumulator: PV_{j-1} must be done
        if (j >= 1) {
          mbar_wait(&bars->o_full[g], (j - 1) & 1);
          tc_fence_after();
          // tcgen05.ld/st are warp-collective: the branch must be warp-uniform
          if (__any_sync(0xffffffffu, alpha != 1.0f)) rescale_o(alpha);
        }
        float part = 0.0f;
#pragma unroll
        for (int c = 0; c < KT / 8; ++c) {
          float p[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) p[i] = ex2(s[8 * c + i] - m_new);
          part += ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
          st_shared_v4(my_p + (c >> 3) * (QT * 128) + swz_offset(row, c & 7, 128),
                       pack_bf16(p[0], p[1]), pack_bf16(p[2], p[3]), pack_bf16(p[4], p[5]),
                       pack_bf16(p[6], p[7]));
        }
        l_run = fmaf(l_run, alpha, part);
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&bars->p_full[g]);
      }
      mbar_wait(&bars->o_full[g], (nj - 1) & 1);
      tc_fence_after();
      {
        float o[RP];
        ld_rank<RP>(tg + C::t_o, o);
        const float inv = 1.0f / l_run;
#pragma unroll
        for (int i = 0; i < RP; ++i) o[i] *= inv;
        store_row_bf16<RP>(my_qt, row, o);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->ofin[g]);
      // ctx epilogue: + b_v, bf16, direct row store
      mbar_wait(&bars->out_done[g], 0);
      tc_fence_after();
      const int qrow = qbase + g * QT + static_cast<int>(row);
#pragma unroll
      for (int c = 0; c < DH; c += 32) {
        uint32_t r[32];
        tmem_ld32(tg + C::t_q + c, r);
        tmem_ld_wait();
        if (qrow < seq) {
          uint4* dst = reinterpret_cast<uint4*>(ctx + (int64_t)(row0 + qrow) * ldc + h * DH + c);
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            float f[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
              f[i] = __uint_as_float(r[8 * v + i]) + __ldg(bv + h * DH + c + 8 * v + i);
            dst[v] = make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]),
                                pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMma) {
    tc_fence_after();
    tmem_free<512>(tmem);
  }
}

template <int RP>
void launch_attn(const AttnTcArgs& a, cudaStream_t s) {
  using C = AttnCfg<RP>;
  static bool attr = false;
  if (!attr) {
    FSVD_CUDA_CHECK(cudaFuncSetAttribute(k_attn_rankspace<RP>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  const int T = a.batch * a.seq;
  const TmaSwizzle sw = swizzle_for_row_bytes(C::RB);
  const CUtensorMap tp = tmap_bf16(a.P, T, 3 * a.groups * RP, a.ldp, 128, RP, sw);
  const CUtensorMap tq = tmap_bf16(a.vq_t, (uint64_t)a.heads * DH, RP, RP, DH, RP, sw);
  const CUtensorMap tk = tmap_bf16(a.vk, (uint64_t)a.heads * RP, DH, DH, RP, DH, TmaSwizzle::B128);
  const CUtensorMap tv = tmap_bf16(a.vv_t, (uint64_t)a.heads * DH, RP, RP, DH, RP, sw);
  dim3 grid((a.seq + 2 * QT - 1) / (2 * QT), a.heads, a.batch);
  k_attn_rankspace<RP><<<grid, kThreads, C::SMEM, s>>>(tp, tq, tk, tv, a.bq, a.bv, a.q_scale,
                                                       a.ctx, a.ldc, a.seq, a.heads, a.groups);
  check_launch("k_attn_rankspace");
}

}  // namespace

bool attn_rankspace_supported(int head_dim, int rank_pad) {
  return head_dim == DH && (rank_pad == 16 || rank_pad == 32 || rank_pad == 64);
}

void attn_rankspace_bf16(const AttnTcArgs& a, cudaStream_t s) {
  switch (a.rank_pad) {
    case 16: launch_attn<16>(a, s); break;
    case 32: launch_attn<32>(a, s); break;
    case 64: launch_attn<64>(a, s); break;
    default: throw CudaError("attn_rankspace_bf16: unsupported rank padding");
  }
}

}  // namespace fsvd
