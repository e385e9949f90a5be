// attn_tc.cu -- K2: FlashSVD attention on tcgen05, rank-space streaming.
//
// Replaces flash_svd_attention's per-head stream (attention.cpp:249-267 and
// online_softmax_head :92-137).  Per CTA = one (batch b, head h, 128-row query
// tile).  The reference rebuilds head-width Q, K, V tiles from the rank-r
// activations P = X U and the factor slices V (bias preloaded, :254-264) and
// runs an online softmax over key tiles.  Here the same algebra runs with the
// factors folded on chip:
//
//   Q   = (P_q Vq + b_q) * scale*log2e          tcgen05, M=128 N=64  K=r
//   Qt  = Q Vk^T                                tcgen05, M=128 N=r   K=64
//   S_j = Qt P_k,j^T  (= Q K_j^T - Q b_k 1^T)   tcgen05, M=128 N=128 K=r
//   online softmax over j (exp2), P_j -> smem bf16
//   O_j = P_j P_v,j                             tcgen05, M=128 N=r   K=128
//   o   = o * alpha_j + O_j                     registers (rank width)
//   ctx = (o / l) Vv + b_v                      tcgen05, M=128 N=64  K=r
//
// The K bias only adds the per-row constant Q.b_k to every score, which the
// softmax cancels; the V bias passes through because softmax rows sum to one.
// So no head-width K or V tile is ever formed and P_k / P_v tiles stream
// straight from HBM by TMA.  Dense Q/K/V never exist in HBM.
//
// Warp roles: 0 TMA producer, 1 MMA issuer (one lane) + TMEM owner,
// 2..5 softmax / epilogue (thread = query row, TMEM lane quadrant warp%4).
#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace fsvd {
namespace {

using namespace ptx;

constexpr int kThreads = 192;
constexpr int QT = 128;  // query rows per CTA
constexpr int KT = 128;  // keys per tile
constexpr int DH = 64;   // head dim

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int RP>
struct AttnCfg {
  static constexpr int STAGES = RP >= 64 ? 2 : 3;
  static constexpr int RB = RP * 2;  // bytes per rank-width row
  static constexpr int PQ = QT * RB;
  static constexpr int VQ = DH * RB;
  static constexpr int VK = RP * DH * 2;
  static constexpr int VV = DH * RB;
  static constexpr int SQ = QT * DH * 2;
  static constexpr int SQT = QT * RB;
  static constexpr int KV = KT * RB;  // one of P_k / P_v
  static constexpr int SP = QT * KT * 2;
  // offsets (all multiples of 1024)
  static constexpr int o_pq = 0;
  static constexpr int o_vq = o_pq + ((PQ + 1023) / 1024) * 1024;
  static constexpr int o_vk = o_vq + ((VQ + 1023) / 1024) * 1024;
  static constexpr int o_vv = o_vk + ((VK + 1023) / 1024) * 1024;
  static constexpr int o_q = o_vv + ((VV + 1023) / 1024) * 1024;
  static constexpr int o_qt = o_q + SQ;
  static constexpr int o_kv = o_qt + ((SQT + 1023) / 1024) * 1024;
  static constexpr int KV_STAGE = 2 * ((KV + 1023) / 1024) * 1024;
  static constexpr int o_p = o_kv + STAGES * KV_STAGE;
  static constexpr int o_bar = o_p + 2 * SP;
  static constexpr int SMEM = 1024 + o_bar + 512;
  // TMEM columns
  static constexpr int t_s = 0;            // 2 x 128
  static constexpr int t_o = 256;          // 2 x RP
  static constexpr int t_q = 256 + 2 * RP; // 64 (also final output)
  static constexpr int t_qt = t_q + 64;    // RP
};

struct Bars {
  uint64_t pro, q, qs, qt, qts, ofin, out;
  uint64_t kv_full[3], kv_empty[3];
  uint64_t s_full[2], s_free[2], p_full[2], o_full[2], o_free[2];
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

// Writes `n` floats of one row as bf16 into a K-major swizzled tile whose rows
// are row_bytes long (n * 2 == row_bytes).
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
  const int qtile = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int g = h / (heads / groups);
  const int row0 = b * seq;               // first token row of this sequence
  const int q0 = qtile * QT;              // first query (within the sequence)
  const int nj = (seq + KT - 1) / KT;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmP);
    tma_prefetch(&tmVq);
    tma_prefetch(&tmVk);
    tma_prefetch(&tmVv);
    mbar_init(&bars->pro, 1);
    mbar_init(&bars->q, 1);
    mbar_init(&bars->qs, 128);
    mbar_init(&bars->qt, 1);
    mbar_init(&bars->qts, 128);
    mbar_init(&bars->ofin, 128);
    mbar_init(&bars->out, 1);
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->s_free[i], 128);
      mbar_init(&bars->p_full[i], 128);
      mbar_init(&bars->o_full[i], 1);
      mbar_init(&bars->o_free[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars->pro, C::PQ + C::VQ + C::VK + C::VV);
      tma_load_2d(&tmP, &bars->pro, smem + C::o_pq, (0 * groups + g) * RP, row0 + q0);
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
        tma_load_2d(&tmP, &bars->kv_full[st], kv, (1 * groups + g) * RP, row0 + j * KT);
        tma_load_2d(&tmP, &bars->kv_full[st], kv + C::KV_STAGE / 2, (2 * groups + g) * RP,
                    row0 + j * KT);
      }
      __syncwarp();
      if (++st == C::STAGES) { st = 0; ph ^= 1; }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    const uint32_t s_pq = smem_u32(smem + C::o_pq), s_vq = smem_u32(smem + C::o_vq);
    const uint32_t s_vk = smem_u32(smem + C::o_vk), s_vv = smem_u32(smem + C::o_vv);
    const uint32_t s_q = smem_u32(smem + C::o_q), s_qt = smem_u32(smem + C::o_qt);
    const uint32_t s_kv = smem_u32(smem + C::o_kv), s_p = smem_u32(smem + C::o_p);
    // Q = P_q Vq  (M=128, N=64, K=RP)
    mbar_wait(&bars->pro, 0);
    tc_fence_after();
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < RP / 16; ++k)
        mma_bf16_ss(tmem + C::t_q, desc_kmajor(s_pq + k * 32, C::RB),
                    desc_kmajor(s_vq + k * 32, C::RB), idesc_bf16(128, DH), k != 0);
      mma_commit(&bars->q);
    }
    __syncwarp();
    // Qt = Q Vk^T (M=128, N=RP, K=64)
    mbar_wait(&bars->qs, 0);
    tc_fence_after();
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < DH / 16; ++k)
        mma_bf16_ss(tmem + C::t_qt, desc_kmajor(s_q + k * 32, 128),
                    desc_kmajor(s_vk + k * 32, 128), idesc_bf16(128, RP), k != 0);
      mma_commit(&bars->qt);
    }
    __syncwarp();
    mbar_wait(&bars->qts, 0);
    tc_fence_after();

    auto issue_s = [&](int j) {
      const uint32_t st = j % C::STAGES, ph = (j / C::STAGES) & 1;
      mbar_wait(&bars->kv_full[st], ph);
      mbar_wait(&bars->s_free[j & 1], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t pk = s_kv + st * C::KV_STAGE;
#pragma unroll
        for (int k = 0; k < RP / 16; ++k)
          mma_bf16_ss(tmem + C::t_s + (j & 1) * 128, desc_kmajor(s_qt + k * 32, C::RB),
                      desc_kmajor(pk + k * 32, C::RB), idesc_bf16(128, KT), k != 0);
        mma_commit(&bars->s_full[j & 1]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int j) {
      const uint32_t st = j % C::STAGES;
      mbar_wait(&bars->p_full[j & 1], (j >> 1) & 1);
      mbar_wait(&bars->o_free[j & 1], ((j >> 1) & 1) ^ 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t pv = s_kv + st * C::KV_STAGE + C::KV_STAGE / 2;
        const uint32_t pa = s_p + (j & 1) * C::SP;
#pragma unroll
        for (int k = 0; k < KT / 16; ++k)
          mma_bf16_ss(tmem + C::t_o + (j & 1) * RP,
                      desc_kmajor(pa + (k >> 2) * (QT * 128) + (k & 3) * 32, 128),
                      desc_mnmajor(pv + k * 16 * C::RB, C::RB), idesc_bf16(128, RP, 0, 1),
                      k != 0);
        mma_commit(&bars->o_full[j & 1]);
        mma_commit(&bars->kv_empty[st]);
      }
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < nj; ++j) {
      if (j + 1 < nj) issue_s(j + 1);
      issue_pv(j);
    }
    // ctx = O Vv (M=128, N=64, K=RP), O staged in the Qt tile
    mbar_wait(&bars->ofin, 0);
    tc_fence_after();
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < RP / 16; ++k)
        mma_bf16_ss(tmem + C::t_q, desc_kmajor(s_qt + k * 32, C::RB),
                    desc_kmajor(s_vv + k * 32, C::RB), idesc_bf16(128, DH), k != 0);
      mma_commit(&bars->out);
    }
    __syncwarp();
  } else {
    // ------------------------------------------------ softmax / epilogue
    const uint32_t quad = warp & 3;
    const uint32_t row = quad * 32 + lane;  // query row within the tile
    const uint32_t lane_off = (quad * 32) << 16;
    const uint32_t s_q = smem_u32(smem + C::o_q), s_qt = smem_u32(smem + C::o_qt);
    const uint32_t s_p = smem_u32(smem + C::o_p);

    // Q epilogue: bias, softmax scale (log2 domain), bf16 -> smem
    mbar_wait(&bars->q, 0);
    tc_fence_after();
    {
      float qv[DH];
#pragma unroll
      for (int c = 0; c < DH; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + C::t_q + lane_off + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i)
          qv[c + i] = (__uint_as_float(r[i]) + __ldg(bq + h * DH + c + i)) * q_scale;
      }
      store_row_bf16<DH>(s_q, row, qv);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    mbar_arrive(&bars->qs);
    // Qt epilogue
    mbar_wait(&bars->qt, 0);
    tc_fence_after();
    {
      float t[RP];
      ld_rank<RP>(tmem + C::t_qt + lane_off, t);
      store_row_bf16<RP>(s_qt, row, t);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    mbar_arrive(&bars->qts);

    float o[RP];
#pragma unroll
    for (int i = 0; i < RP; ++i) o[i] = 0.0f;
    float m_run = -INFINITY, l_run = 0.0f;
    float alpha_hist[2] = {0.0f, 0.0f};

    auto consume_o = [&](int t, float alpha) {
      mbar_wait(&bars->o_full[t & 1], (t >> 1) & 1);
      tc_fence_after();
      float ot[RP];
      ld_rank<RP>(tmem + C::t_o + (t & 1) * RP + lane_off, ot);
      tc_fence_before();
      mbar_arrive(&bars->o_free[t & 1]);
#pragma unroll
      for (int i = 0; i < RP; ++i) o[i] = o[i] * alpha + ot[i];
    };

    for (int j = 0; j < nj; ++j) {
      mbar_wait(&bars->s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      float s[KT];
#pragma unroll
      for (int c = 0; c < KT; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + C::t_s + (j & 1) * 128 + lane_off + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c + i] = __uint_as_float(r[i]);
      }
      tc_fence_before();
      mbar_arrive(&bars->s_free[j & 1]);
      const int valid = seq - j * KT;  // keys of this tile inside the sequence
      float tmax = -INFINITY;
#pragma unroll
      for (int i = 0; i < KT; ++i)
        if (i < valid) tmax = fmaxf(tmax, s[i]);
      const float m_new = fmaxf(m_run, tmax);
      const float alpha = ex2(m_run - m_new);
      float part = 0.0f;
#pragma unroll
      for (int i = 0; i < KT; ++i) {
        const float p = (i < valid) ? ex2(s[i] - m_new) : 0.0f;
        s[i] = p;
        part += p;
      }
      l_run = l_run * alpha + part;
      m_run = m_new;
      // P buffer (j&1) was read by PV_{j-2}: consume that result first.
      if (j >= 2) consume_o(j - 2, alpha_hist[j & 1]);
      alpha_hist[j & 1] = alpha;
      const uint32_t pb = s_p + (j & 1) * C::SP;
#pragma unroll
      for (int a = 0; a < 2; ++a) store_row_bf16<64>(pb + a * (QT * 128), row, s + a * 64);
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->p_full[j & 1]);
    }
    if (nj >= 2) consume_o(nj - 2, alpha_hist[nj & 1]);
    consume_o(nj - 1, alpha_hist[(nj - 1) & 1]);
    const float inv = 1.0f / l_run;
#pragma unroll
    for (int i = 0; i < RP; ++i) o[i] *= inv;
    store_row_bf16<RP>(s_qt, row, o);
    fence_proxy_async_smem();
    tc_fence_before();
    mbar_arrive(&bars->ofin);
    // ctx epilogue: + b_v, bf16, direct row store
    mbar_wait(&bars->out, 0);
    tc_fence_after();
    const int qrow = q0 + static_cast<int>(row);
#pragma unroll
    for (int c = 0; c < DH; c += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + C::t_q + lane_off + c, r);
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
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
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
  dim3 grid((a.seq + QT - 1) / QT, a.heads, a.batch);
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
