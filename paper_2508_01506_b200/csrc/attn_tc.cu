// attn_tc.cu -- K2: FlashSVD attention on tcgen05, rank-space streaming.
//
// Replaces flash_svd_attention's per-head stream (attention.cpp:249-267 and
// online_softmax_head :92-137).  The reference rebuilds head-width Q, K, V
// tiles from the rank-r activations P = X U and the factor slices V (bias
// preloaded, :254-264) before scoring.  The same algebra is evaluated here
// with the factors folded:
//
//   S  = Q K^T           with Q = (X U_q V_q + b_q) s, K = X U_k V_k + b_k
//      = Qt P_k^T + (row constant)      Qt = Q V_k^T  (rank width, per head)
//   O  = softmax(S) V    = (softmax(S) P_v) V_v + b_v
//
// Qt is linear in X, so the projection GEMM produces it directly from the
// folded weight U_q V_q V_k^T s (runtime.cu); the row constant Q.b_k cancels
// in the softmax; and (softmax(S) P_v) V_v + b_v is folded into the output
// projection.  This kernel is therefore a pure rank-space flash loop:
//
//   S_j = Qt P_k,j^T              tcgen05, M=128 N=128 K=r   (TMEM)
//   online softmax (exp2, scores are pre-scaled by log2 e)
//   O  <- O * alpha_j             rank-width TMEM rescale
//   O += P_j P_v,j                tcgen05, M=128 N=r   K=128 (TMEM)
//   out = O / l                   [T, H * r] bf16, rank space
//
// It is also the dense-attention kernel of the materializing baselines: with
// r = head_dim and Q/K/V as its three inputs it computes softmax(Q K^T) V.
//
// P never touches shared memory: the softmax warps tcgen05.st the bf16
// probabilities into TMEM and the PV MMA reads its A operand from there (the
// kernel is shared-memory-bandwidth bound otherwise: P would cost a 32 KB
// st.shared plus a 32 KB MMA read per key tile).
//
// CTA = one (batch, head, 128-row query tile); 10 warps: 0-7 softmax (two
// threads per query row, 64 keys each; TMEM lane quadrant warp%4), 8 TMA
// producer, 9 MMA issuer and TMEM owner.  ~92 KB smem and 256 TMEM columns,
// so two CTAs share an SM (16 softmax warps per SM to hide MUFU / TMEM
// latency; the softmax is issue- and latency-bound, not exp-bound).
//
// Output (bf16 RP <= 32): each quadrant pair stages its 32 rows of O / l in
// shared memory and one thread TMA-stores them as a [32 x RP] box of a
// [batch, seq, H*RP] map (rows past the sequence are clipped); the store of
// item e is issued during item e+1 and drained two items later.  Against
// per-thread row stores this is -0.8% on the 12-layer step; keeping Bars in
// the shared window (LDS / STS instead of generic loads) and the spill
// reduction that came with it another -1.3% (`tools/ab.sh`).
#include "common.cuh"
#include "kernels.cuh"
#include "ptx.cuh"

namespace fsvd {
FSVD_CTA_TIMES(attn)
}  // namespace fsvd

namespace fsvd {
namespace {

using namespace ptx;

constexpr int QT = 128;  // query rows per CTA
constexpr int KT = 128;  // keys per tile
constexpr float kRescaleSlack = 8.0f;  // log2 headroom before the running max moves
constexpr int kThreads = 320;
constexpr int kSoftmax = 256;  // warps 0-7: two per TMEM lane quadrant, 64 keys each
constexpr int kTma = 8, kMma = 9;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (x <= 0): x = n + f with n = round(x) taken from the
// mantissa of x + 1.5*2^23, f in [-0.5, 0.5]; 2^f by a degree-3 polynomial
// (relative error 2.1e-4, far below the bf16 rounding of P), 2^n added to
// the exponent field.  A share of the probabilities takes this path so the
// softmax is not bound by the 16/clk/SM MUFU rate alone (EMU_EVERY: one
// pair of probabilities in EMU_EVERY takes the polynomial).
#ifndef EMU_EVERY
#define EMU_EVERY 3
#endif
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  x.x = fmaxf(x.x, -125.0f);
  x.y = fmaxf(x.y, -125.0f);
  const float2 magic = make_float2(12582912.0f, 12582912.0f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 f = __fadd2_rn(x, __fadd2_rn(magic, make_float2(-t.x, -t.y)));
  float2 p = __ffma2_rn(f, make_float2(0.054848f, 0.054848f), make_float2(0.24180661f, 0.24180661f));
  p = __ffma2_rn(p, f, make_float2(0.6932482f, 0.6932482f));
  p = __ffma2_rn(p, f, make_float2(0.9999887f, 0.9999887f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

__host__ __device__ constexpr int up1k(int x) { return (x + 1023) / 1024 * 1024; }

#ifdef FSVD_TRACE
__device__ long long g_trace_at[2048];
}  // namespace
extern "C" __attribute__((visibility("default"))) int fsvd_debug_trace_attn_copy(long long* host, int n) {
  return static_cast<int>(cudaMemcpyFromSymbol(host, g_trace_at, sizeof(long long) * n));
}
namespace {
// CTA 0 (first work item) and its SM clock
#define ATRACE(slot) do { if (blockIdx.x == 0) g_trace_at[(slot)] = clock64(); } while (0)
#else
#define ATRACE(slot) do { } while (0)
#endif

// X3 (fp32 policy, split planes -- kernels.cuh): Qt, P_k, P_v arrive as three
// bf16 planes each (one stacked tensor map, plane p at row offset p*plane_rows);
// S and O accumulate the six plane pairs of order <= 2, the probabilities are
// computed in fp32 (MUFU ex2 only) and stored to TMEM as three planes, and the
// output leaves as three planes (out_ps elements apart).  One CTA per SM.
__device__ __forceinline__ int x3_pa(int g) { return (0x120100 >> (4 * g)) & 15; }
__device__ __forceinline__ int x3_pb(int g) { return (0x102010 >> (4 * g)) & 15; }

template <int RP, bool X3 = false>
struct AttnCfg {
  static constexpr int STAGES = X3 ? (RP >= 64 ? 1 : RP >= 32 ? 2 : 3) : (RP >= 64 ? 2 : 3);
  static constexpr int RB = RP * 2;       // bytes per rank-width row
  static constexpr int TILE = QT * RB;    // one Qt / P_k / P_v tile (one plane)
  static constexpr int NPL = X3 ? 3 : 1;  // planes per operand
  static constexpr int Q_SLOT = NPL * up1k(TILE);
  static constexpr int o_q = 0;           // two Qt slots (next item prefetched)
  static constexpr int o_kv = o_q + 2 * Q_SLOT;
  // KV stage: the K planes, then the V planes
  static constexpr int KV_STAGE = 2 * NPL * up1k(TILE);
  static constexpr int kv_v = NPL * up1k(TILE);
  static constexpr int o_bar = o_kv + STAGES * KV_STAGE;
  // output staging (two items, swizzled like the output tensor map) for the
  // TMA-store epilogue; the fp32-policy planes and RP = 64 store directly
  static constexpr bool TMA_OUT = !X3 && RP <= 32;
  static constexpr int OUT_TILE = QT * RB;
  static constexpr int o_stage = up1k(o_bar + 4608);
  static constexpr int SMEM = 1024 + (TMA_OUT ? o_stage + 2 * OUT_TILE : o_bar + 4608);
  // TMEM columns: S (fp32, 128 keys), O (fp32, RP; two buffers when they fit
  // so an item's output is written while the next item runs), P (bf16 pairs),
  // X3: the P planes at t_p + 64 * plane
  static constexpr int t_s = 0, t_o = 128, t_p = 192;
  static constexpr int NOB = RP <= 32 ? 2 : 1;
  static constexpr int TMEM_COLS = X3 ? 512 : 256;
  static constexpr int CTAS = X3 ? 1 : 2;
  static_assert(CTAS * SMEM <= 228 * 1024, "CTAs per SM");
  static_assert(!TMA_OUT || NOB == 2, "the staged epilogue runs during the next item");
};

struct Bars {
  uint64_t q_full[2], q_empty[2];
  uint64_t kv_full[3], kv_empty[3];
  uint64_t s_full, s_free, p_full, o_full, o_free[2];
  uint64_t item_full[4], item_empty[4];  // dynamic schedule: item ids, producer -> MMA / softmax
  int item_ring[4];
  uint32_t tmem;
  float xmax[2][2][QT];  // [tile parity][half][row]: per-half row maxima
  float xsum[2][2][QT];  // [item parity][half][row]: per-half row sums of an item
};
static_assert(sizeof(Bars) <= 4608, "Bars outgrew its shared-memory reservation");

// Work item w -> (query tile, head, batch).  Encoder: query tile fastest, so
// consecutive items share (batch, head) and K/V stay hot in L2.  Causal: the
// query tile is the SLOWEST index and runs from the last (most key tiles)
// down, so the stride-gridDim walk hands every CTA a mix of long and short
// items instead of a fixed query-tile position (largest work first).
struct Item {
  int qt, h, b;
};
__device__ __forceinline__ Item item_of(int w, int nqt, int heads, int batch, int causal) {
  Item it;
  if (causal) {
    const int hb = heads * batch, rem = w % hb;
    it.qt = nqt - 1 - w / hb;
    it.h = rem % heads;
    it.b = rem / heads;
  } else {
    it.qt = w % nqt;
    it.h = (w / nqt) % heads;
    it.b = w / (nqt * heads);
  }
  return it;
}

// Persistent: each CTA walks work items (batch, head, 128-query tile) with
// stride gridDim.x; consecutive items share (batch, head) so K/V stay hot in
// L2.  Q of the next item and its first K/V tiles are prefetched while the
// current item finishes, and TMEM / barriers are set up once per CTA.
template <int RP, bool X3 = false, bool TMAO = false>
__global__ void __launch_bounds__(kThreads) __maxnreg__(X3 ? 168 : 96)  // X3: one CTA per SM
    k_attn_rankspace(const __grid_constant__ CUtensorMap tmQKV,
                     const __grid_constant__ CUtensorMap tmKV,
                     const __grid_constant__ CUtensorMap tmO, int* sched, bf16* out,
                     int64_t ldo, int batch, int seq, int heads, int groups, int q_off, int k_off,
                     int v_off, int causal, int plane_rows, int64_t out_ps) {
  using C = AttnCfg<RP, X3>;
  constexpr bool staged = C::TMA_OUT && TMAO;
  CTA_T(0);
  extern __shared__ uint8_t smem_raw[];
  // 1 KB aligned by pointer arithmetic on the __shared__ array, so the
  // compiler keeps the shared address space (LDS / STS, not generic LD / ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Bars* bars = reinterpret_cast<Bars*>(smem + C::o_bar);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int nqt = (seq + QT - 1) / QT;
  const int items = nqt * heads * batch;
  const int nj = (seq + KT - 1) / KT;
  const int hpg = heads / groups;

  if (warp == kTma && lane == 0) {
    tma_prefetch(&tmQKV);
    tma_prefetch(&tmKV);
    if (staged) tma_prefetch(&tmO);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->q_full[i], 1);
      mbar_init(&bars->q_empty[i], 1);
    }
    for (int i = 0; i < C::STAGES; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->s_free, kSoftmax);
    mbar_init(&bars->p_full, kSoftmax);
    mbar_init(&bars->o_full, 1);
    mbar_init(&bars->o_free[0], kSoftmax);
    mbar_init(&bars->o_free[1], kSoftmax);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&bars->item_full[i], 1);
      mbar_init(&bars->item_empty[i], 1 + kSoftmax);
    }
    fence_barrier_init();
  }
  if (threadIdx.x == 0) ATRACE(0);
  if (warp == kMma) tmem_alloc<C::TMEM_COLS>(&bars->tmem);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  pdl_wait();
  CTA_T(1);
  const uint32_t tmem = bars->tmem;
  const uint32_t s_q = smem_u32(smem + C::o_q), s_kv = smem_u32(smem + C::o_kv);
  // Work items: the first is blockIdx.x; then, with a schedule counter
  // (sched[0]), the TMA thread takes the next free one (gridDim.x +
  // atomicAdd) as it starts loading it and publishes the id through a
  // four-slot ring (-1: done), so a CTA that runs ahead -- or shares its SM
  // with a slower one -- takes more items; without one, stride gridDim.x.
  const bool dyn = sched != nullptr;
  const int G = static_cast<int>(gridDim.x);
  auto ring_get = [&](int k) -> int {
    mbar_wait(&bars->item_full[k & 3], (k >> 2) & 1);
    return reinterpret_cast<volatile int*>(bars->item_ring)[k & 3];
  };

  if (warp == kTma) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t st = 0, ph = 0;
      int w = blockIdx.x;
      for (int it = 0;; ++it) {
        if (it > 0) w = dyn ? G + atomicAdd(sched, 1) : w + G;
        if (dyn) {
          mbar_wait(&bars->item_empty[it & 3], ((it >> 2) & 1) ^ 1);
          reinterpret_cast<volatile int*>(bars->item_ring)[it & 3] = w < items ? w : -1;
          mbar_arrive(&bars->item_full[it & 3]);
        }
        if (w >= items) break;
        const Item iw = item_of(w, nqt, heads, batch, causal);
        const int qt = iw.qt, h = iw.h, b = iw.b;
        const int g = h / hpg, row0 = b * seq;
        const int qs = it & 1;
        mbar_wait(&bars->q_empty[qs], ((it >> 1) & 1) ^ 1);
        if (it < 100) ATRACE(500 + it);
        mbar_arrive_expect_tx(&bars->q_full[qs], C::NPL * C::TILE);
        for (int pl = 0; pl < C::NPL; ++pl)
          tma_load_2d(&tmQKV, &bars->q_full[qs], smem + C::o_q + qs * C::Q_SLOT + pl * up1k(C::TILE),
                      q_off + h * RP, row0 + qt * QT + pl * plane_rows);
        const int nji = causal ? min(nj, qt + 1) : nj;  // key tiles of this item
        for (int j = 0; j < nji; ++j) {
          mbar_wait(&bars->kv_empty[st], ph ^ 1);
          uint8_t* kv = smem + C::o_kv + st * C::KV_STAGE;
          mbar_arrive_expect_tx(&bars->kv_full[st], 2 * C::NPL * C::TILE);
          for (int pl = 0; pl < C::NPL; ++pl) {
            tma_load_2d(&tmKV, &bars->kv_full[st], kv + pl * up1k(C::TILE), k_off + g * RP,
                        row0 + j * KT + pl * plane_rows);
            tma_load_2d(&tmKV, &bars->kv_full[st], kv + C::kv_v + pl * up1k(C::TILE),
                        v_off + g * RP, row0 + j * KT + pl * plane_rows);
          }
          if (++st == C::STAGES) { st = 0; ph ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == kMma) {
    // ------------------------------------------------ MMA issuer (warp-uniform)
    const uint64_t dk0 = desc_kmajor(s_kv, C::RB);
    const uint64_t dv0 = desc_mnmajor(s_kv + C::kv_v, C::RB);
    constexpr uint32_t kPlOff = up1k(C::TILE) >> 4;  // one plane, descriptor units
    int gt = 0;  // key tiles issued so far by this CTA (all items)
    int it = 0;
    // S for global tile index t of the item whose Qt is in slot qs
    auto issue_s = [&](int t, int qs) {
      const uint32_t st = t % C::STAGES;
      mbar_wait(&bars->kv_full[st], (t / C::STAGES) & 1);
      if (t > 0) mbar_wait(&bars->s_free, (t - 1) & 1);
      tc_fence_after();
      const uint64_t dq = desc_kmajor(s_q + qs * C::Q_SLOT, C::RB);
      const uint64_t dk = dk0 + ((st * C::KV_STAGE) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < RP / 16; ++k)
          mma_bf16_ss(tmem + C::t_s, dq + 2 * k, dk + 2 * k, idesc_bf16(128, KT), k != 0);
        if (X3) {  // the other five plane pairs of order <= 2
#pragma unroll
          for (int g = 1; g < 6; ++g)
#pragma unroll
            for (int k = 0; k < RP / 16; ++k)
              mma_bf16_ss(tmem + C::t_s, dq + x3_pa(g) * kPlOff + 2 * k,
                          dk + x3_pb(g) * kPlOff + 2 * k, idesc_bf16(128, KT), 1u);
        }
        mma_commit(&bars->s_full);
      }
      __syncwarp();
    };
    // S of an item's first tile is issued while the previous item's last
    // tile is still in the softmax (right after its S was read out), so the
    // softmax warps find it ready when they move on.
    int w = dyn ? ring_get(0) : static_cast<int>(blockIdx.x);
    if (w >= 0 && w < items) {
      mbar_wait(&bars->q_full[0], 0);
      if (lane == 0) ATRACE(1);
      issue_s(0, 0);
    }
    for (; w >= 0 && w < items; ++it) {
      if (dyn && lane == 0) mbar_arrive(&bars->item_empty[it & 3]);  // id read
      int w_next = -2;  // not fetched yet
      auto fetch_next = [&] {
        if (w_next == -2) w_next = dyn ? ring_get(it + 1) : (w + G < items ? w + G : -1);
      };
      const int qs = it & 1;
      const int nji = causal ? min(nj, item_of(w, nqt, heads, batch, causal).qt + 1) : nj;
      if (lane == 0 && it < 100) ATRACE(400 + it);
      // the next S (this item's next tile, or the next item's first): issued
      // ahead of this tile's PV when the K/V ring has a second stage; with a
      // single stage its K/V can only arrive once this PV has released the
      // stage, so it follows the PV
      auto next_s = [&](int j, int t) {
        if (j + 1 < nji) {
          issue_s(t + 1, qs);
        } else {
          if (elect_one()) mma_commit(&bars->q_empty[qs]);  // after this item's last S
          __syncwarp();
          fetch_next();  // (the producer has loaded this item's last tile: no wait on us)
          if (w_next >= 0 && w_next < items) {
            mbar_wait(&bars->q_full[qs ^ 1], ((it + 1) >> 1) & 1);
            issue_s(t + 1, qs ^ 1);
          }
        }
      };
      for (int j = 0; j < nji; ++j) {
        const int t = gt + j;
        if (C::STAGES > 1) next_s(j, t);
        mbar_wait(&bars->p_full, t & 1);
        // this item's O buffer must have been read out by the softmax warps
        if (j == 0 && it >= C::NOB) mbar_wait(&bars->o_free[it % C::NOB], ((it / C::NOB) - 1) & 1);
        tc_fence_after();
        const uint32_t st = t % C::STAGES;
        const uint64_t dv = dv0 + ((st * C::KV_STAGE) >> 4);
        const uint32_t t_o = tmem + C::t_o + (it % C::NOB) * RP;
        if (elect_one()) {
          // O += P V: P (A operand) straight from TMEM, 8 columns per K = 16 step
#pragma unroll
          for (int k = 0; k < KT / 16; ++k)
            mma_bf16_ts(t_o, tmem + C::t_p + k * 8, dv + ((k * 16 * C::RB) >> 4),
                        idesc_bf16(128, RP, 0, 1), (j | k) != 0);
          if (X3) {  // the other five plane pairs: P plane x3_pa(g) (TMEM), V plane x3_pb(g)
            constexpr uint32_t kPl = up1k(C::TILE) >> 4;
#pragma unroll
            for (int g = 1; g < 6; ++g)
#pragma unroll
              for (int k = 0; k < KT / 16; ++k)
                mma_bf16_ts(t_o, tmem + C::t_p + 64 * x3_pa(g) + k * 8,
                            dv + x3_pb(g) * kPl + ((k * 16 * C::RB) >> 4),
                            idesc_bf16(128, RP, 0, 1), 1u);
          }
          mma_commit(&bars->o_full);
          mma_commit(&bars->kv_empty[st]);
        }
        __syncwarp();
        if (C::STAGES == 1) next_s(j, t);
      }
      gt += nji;
      fetch_next();
      w = w_next;
    }
  } else {
    // ------------------------------------------------ softmax (8 warps)
    // Two threads per query row (warps w and w+4 share TMEM lane quadrant
    // w%4); each owns 64 of the tile's 128 keys, and the pair exchanges its
    // row maxima through shared memory (named barrier per quadrant).
    const uint32_t quad = warp & 3, half = warp >> 2;
    const uint32_t row = quad * 32 + lane;
    const uint32_t tq = tmem + ((quad * 32) << 16);
    constexpr int KH = KT / 2;  // keys per thread
    // O columns owned by this thread for rescale / output (16-column granules)
    constexpr int CH = RP >= 32 ? RP / 2 : RP;
    const bool owns_o = RP >= 32 || half == 0;
    const int oc0 = RP >= 32 ? static_cast<int>(half) * CH : 0;

    auto rescale_o = [&](uint32_t t_o, float alpha) {
#pragma unroll
      for (int c = 0; c < CH; c += 16) {
        uint32_t r[16];
        tmem_ld16(tq + t_o + oc0 + c, r);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
        tmem_st16(tq + t_o + oc0 + c, r);
      }
      tmem_st_wait();
    };
    // O / l of a finished item -> out (rank space); releases its O buffer.
    // The partner half's l is in xsum[item parity], written before a named
    // barrier both halves have passed since.
    // TMA-store form: each lane-quadrant pair (warps q, q+4) stages its 32
    // rows in shared memory (item parity buffer) and one thread stores them as
    // a [32 x RP] box of the [batch, seq, H*RP] output map, so the scattered
    // row stores leave the softmax warps' path.
    auto store_thread = [&] { return threadIdx.x < 128 && (threadIdx.x & 31) == 0; };
    auto epilogue = [&](int it_e, int b_e, int q0_e, int h_e, float l_e) {
      const int ob = it_e % C::NOB;
      const float lt = l_e + bars->xsum[it_e & 1][half ^ 1][row];
      const float inv = X3 ? 1.0f / lt : __fdividef(1.0f, lt);
      const int row0_e = b_e * seq;
      const int qrow = q0_e + static_cast<int>(row);
      if constexpr (staged) {
        const uint32_t stg = smem_u32(smem + C::o_stage) + quad * (32 * C::RB) + (it_e & 1) * C::OUT_TILE;
#pragma unroll
        for (int c = 0; c < CH; c += 16) {
          if (!owns_o) break;
          uint32_t r[16];
          tmem_ld16(tq + C::t_o + ob * RP + oc0 + c, r);
          tmem_ld_wait();
#pragma unroll
          for (int v = 0; v < 2; ++v)
            st_shared_v4(stg + swz_offset(lane, (oc0 + c) / 8 + v, C::RB),
                         pack_bf16(__uint_as_float(r[8 * v + 0]) * inv, __uint_as_float(r[8 * v + 1]) * inv),
                         pack_bf16(__uint_as_float(r[8 * v + 2]) * inv, __uint_as_float(r[8 * v + 3]) * inv),
                         pack_bf16(__uint_as_float(r[8 * v + 4]) * inv, __uint_as_float(r[8 * v + 5]) * inv),
                         pack_bf16(__uint_as_float(r[8 * v + 6]) * inv, __uint_as_float(r[8 * v + 7]) * inv));
        }
        tc_fence_before();
        mbar_arrive(&bars->o_free[ob]);
        fence_proxy_async_smem();
        named_bar_sync(1 + quad, 64);
        if (store_thread()) {
          tma_store_3d(&tmO, stg, h_e * RP, q0_e + static_cast<int>(quad) * 32, b_e);
          tma_store_commit();
        }
        return;
      }
#pragma unroll
      for (int c = 0; c < CH; c += 16) {
        if (!owns_o) break;
        uint32_t r[16];
        tmem_ld16(tq + C::t_o + ob * RP + oc0 + c, r);
        tmem_ld_wait();
        if (qrow < seq) {
          const int64_t off = (int64_t)(row0_e + qrow) * ldo + h_e * RP + oc0 + c;
          float o[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __uint_as_float(r[i]) * inv;
#pragma unroll
          for (int pl = 0; pl < C::NPL; ++pl) {
            if (pl > 0) {
#pragma unroll
              for (int i = 0; i < 16; ++i) o[i] -= bf16_round_f(o[i]);
            }
            uint4* dst = reinterpret_cast<uint4*>(out + pl * out_ps + off);
#pragma unroll
            for (int v = 0; v < 2; ++v)
              dst[v] = make_uint4(pack_bf16(o[8 * v + 0], o[8 * v + 1]),
                                  pack_bf16(o[8 * v + 2], o[8 * v + 3]),
                                  pack_bf16(o[8 * v + 4], o[8 * v + 5]),
                                  pack_bf16(o[8 * v + 6], o[8 * v + 7]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&bars->o_free[ob]);
    };

    int gt = 0;
    int it = 0;
    // the previous item, whose output is written during this item's first tile
    int pv_b = 0, pv_q0 = 0, pv_h = 0;
    float pv_l = 0.0f;
    for (int w = dyn ? ring_get(0) : static_cast<int>(blockIdx.x); w >= 0 && w < items;
         w = dyn ? ring_get(it + 1) : w + G, ++it) {
      if (dyn) mbar_arrive(&bars->item_empty[it & 3]);  // id read
      const Item iw = item_of(w, nqt, heads, batch, causal);
      const int qt = iw.qt, h = iw.h, b = iw.b;
      const int q0 = qt * QT;
      const int nji = causal ? min(nj, qt + 1) : nj;
      const uint32_t t_o = C::t_o + (it % C::NOB) * RP;
      if (threadIdx.x == 0 && it < 100) ATRACE(300 + it);
      float m_run = -INFINITY, l_run = 0.0f;
      for (int j = 0; j < nji; ++j) {
        const int t = gt + j;
        if (threadIdx.x == 0 && it == 0) ATRACE(112 + j);
        mbar_wait(&bars->s_full, t & 1);
        if (threadIdx.x == 0 && it == 0) ATRACE(144 + j);
        if (threadIdx.x == 0 && it < 100 && j <= 1) ATRACE(1100 + it * 8 + (j ? 5 : 0));
        tc_fence_after();
        float s[KH];
#pragma unroll
        for (int c = 0; c < KH; c += 32) {
          uint32_t r[32];
          tmem_ld32(tq + C::t_s + half * KH + c, r);
#pragma unroll
          for (int i = 0; i < 32; ++i) s[c + i] = __uint_as_float(r[i]);
        }
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&bars->s_free);
        // keys of this thread's half that are in the sequence (and, causal,
        // not after the query: key index <= query index)
        int valid = seq - j * KT - static_cast<int>(half) * KH;
        if (causal && j == qt)
          valid = min(valid, static_cast<int>(row) - static_cast<int>(half) * KH + 1);
        if (valid < KH) {
#pragma unroll
          for (int i = 0; i < KH; ++i) s[i] = (i < valid) ? s[i] : -INFINITY;
        }
        float mx[8];  // 8 independent max chains
#pragma unroll
        for (int i = 0; i < 8; ++i) mx[i] = s[i];
#pragma unroll
        for (int i = 8; i < KH; ++i) mx[i & 7] = fmaxf(mx[i & 7], s[i]);
        float tmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                           fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
        bars->xmax[t & 1][half][row] = tmax;
        // the staging buffer the coming epilogue writes: its store (two items
        // back) has been read out before anyone passes this barrier
        if (staged && j == 0 && store_thread()) tma_store_wait_read<1>();
        named_bar_sync(1 + quad, 64);
        tmax = fmaxf(tmax, bars->xmax[t & 1][half ^ 1][row]);
        if (threadIdx.x == 0 && it < 100 && j <= 1) ATRACE(1100 + it * 8 + (j ? 7 : 1));
        // Lazy rescaling: keep the running max unless the tile's max exceeds
        // it by more than kRescaleSlack (log2 units), so p <= 2^slack and the
        // O / l rescale (and its TMEM round trip) is skipped for most tiles.
        // O / l is the same quotient for any reference max.
        const float m_new = tmax > m_run + kRescaleSlack ? tmax : m_run;
        const float alpha = ex2(m_run - m_new);
        m_run = m_new;
        uint32_t pk[KH / 2];
        uint32_t pk2[KH / 2], pk3[KH / 2];  // X3: P_mid, P_lo (dead otherwise)
        float2 sum2 = make_float2(0.0f, 0.0f);
        const float2 nm = make_float2(-m_new, -m_new);
#pragma unroll
        for (int c = 0; c < KH / 2; ++c) {
          const float2 d = __fadd2_rn(make_float2(s[2 * c], s[2 * c + 1]), nm);
          // one pair in EMU_EVERY on the FMA pipe, the rest on MUFU (X3: all MUFU)
          const float2 p = (!X3 && c % EMU_EVERY == EMU_EVERY - 1)
                               ? ex2_poly2(d)
                               : make_float2(ex2(d.x), ex2(d.y));
          sum2 = __fadd2_rn(sum2, p);
          pk[c] = pack_bf16(p.x, p.y);
          if (X3) {
            const float2 r = make_float2(p.x - bf16_round_f(p.x), p.y - bf16_round_f(p.y));
            pk2[c] = pack_bf16(r.x, r.y);
            pk3[c] = pack_bf16(r.x - bf16_round_f(r.x), r.y - bf16_round_f(r.y));
          }
        }
        l_run = fmaf(l_run, alpha, sum2.x + sum2.y);
        // single-buffered probability tile: the previous PV (this item's, or
        // the previous item's last one) must be done before P is rewritten
        const bool prev_pv = j >= 1 || (C::NOB == 2 && it > 0);
        if (prev_pv) {
          mbar_wait(&bars->o_full, (t - 1) & 1);
          tc_fence_after();
          if (j >= 1 && owns_o && __any_sync(0xffffffffu, alpha != 1.0f)) rescale_o(t_o, alpha);
        }
        if (threadIdx.x == 0 && it < 100 && j == 0) ATRACE(1100 + it * 8 + 2);
        // this half's 64 keys -> TMEM columns [t_p + 32*half, +32) of this row
        tmem_st32(tq + C::t_p + half * 32, pk);
        if (X3) {
          tmem_st32(tq + C::t_p + 64 + half * 32, pk2);
          tmem_st32(tq + C::t_p + 128 + half * 32, pk3);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bars->p_full);
        if (threadIdx.x == 0 && it < 100 && j == 0) ATRACE(1100 + it * 8 + 3);
        if (C::NOB == 2 && j == 0 && it > 0) epilogue(it - 1, pv_b, pv_q0, pv_h, pv_l);
        if (threadIdx.x == 0 && it < 100 && j == 0) ATRACE(1100 + it * 8 + 4);
        if (threadIdx.x == 0 && it < 100) ATRACE(600 + it * 4 + min(j, 3));
      }
      gt += nji;
      if (threadIdx.x == 0 && it < 100) ATRACE(1100 + it * 8 + 6);
      bars->xsum[it & 1][half][row] = l_run;
      if (C::NOB == 1) {
        mbar_wait(&bars->o_full, (gt - 1) & 1);
        tc_fence_after();
        named_bar_sync(1 + quad, 64);
        epilogue(it, b, q0, h, l_run);
      }
      pv_b = b;
      pv_q0 = q0;
      pv_h = h;
      pv_l = l_run;
      if (threadIdx.x == 0 && it == 0) ATRACE(2);
    }
    if (C::NOB == 2 && it > 0) {  // the last item's output
      mbar_wait(&bars->o_full, (gt - 1) & 1);
      tc_fence_after();
      if (staged && store_thread()) tma_store_wait_read<1>();
      named_bar_sync(1 + quad, 64);
      epilogue(it - 1, pv_b, pv_q0, pv_h, pv_l);
    }
    if (staged && store_thread()) tma_store_wait<0>();
  }
  if (threadIdx.x == 0) ATRACE(3);
  tc_fence_before();
  __syncthreads();
  if (warp == kMma) {
    tc_fence_after();
    tmem_free<C::TMEM_COLS>(tmem);
  }
  // the last CTA out returns the schedule counters to zero for the next
  // launch on this stream (every CTA has taken its last item by now)
  if (dyn && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(sched + 1, 1) == G - 1) {
      atomicExch(sched, 0);
      atomicExch(sched + 1, 0);
    }
  }
  CTA_T(2);
}

// developer A/B switch: FSVD_ATTN_TMA_OUT=0 writes the output with per-thread stores
bool attn_tma_out_enabled() {
  static const bool on = [] {
    const char* e = getenv("FSVD_ATTN_TMA_OUT");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int RP, bool X3, bool TMAO>
void launch_attn_k(const AttnTcArgs& a, cudaStream_t s, const CUtensorMap& tm, const CUtensorMap& tkv,
                   const CUtensorMap& to, int T) {
  using C = AttnCfg<RP, X3>;
  static bool attr = false;
  if (!attr) {
    FSVD_CUDA_CHECK(cudaFuncSetAttribute(k_attn_rankspace<RP, X3, TMAO>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  const int items = ((a.seq + QT - 1) / QT) * a.heads * a.batch;
  const int grid = items < C::CTAS * num_sms() ? items : C::CTAS * num_sms();
  // causal items are pre-ordered longest first for the stride walk: static
  int* sched = a.causal || grid >= items || !sched_enabled("FSVD_ATTN_DYN") ? nullptr : sched_counter(s);
  launch_pdl(k_attn_rankspace<RP, X3, TMAO>, dim3(grid), dim3(kThreads), C::SMEM, s, tm, tkv, to,
             sched, a.out, a.ldo, a.batch, a.seq, a.heads, a.groups, a.q_off, a.k_off, a.v_off,
             a.causal ? 1 : 0, X3 ? T : 0, X3 ? a.out_ps : (int64_t)0);
  check_launch("k_attn_rankspace");
}

template <int RP, bool X3 = false>
void launch_attn(const AttnTcArgs& a, cudaStream_t s) {
  using C = AttnCfg<RP, X3>;
  const int T = a.batch * a.seq;
  // X3: the three planes of qkv stacked ([3T, qkv_cols], plane p at row p*T)
  const CUtensorMap tm = tmap_bf16(a.qkv, (uint64_t)C::NPL * T, a.qkv_cols, a.ldq, 128, RP,
                                   swizzle_for_row_bytes(C::RB));
  // K / V from a separate region (k_off / v_off relative to it) when given
  const CUtensorMap tkv = a.kv == nullptr ? tm
                                          : tmap_bf16(a.kv, (uint64_t)C::NPL * T, a.kv_cols, a.ldkv,
                                                      128, RP, swizzle_for_row_bytes(C::RB));
  // output as [batch, seq, H*RP] boxes of [32 x RP] (TMA store epilogue) when
  // the layout allows a tensor map (16-byte aligned base and row stride)
  const bool tma_out = C::TMA_OUT && reinterpret_cast<uintptr_t>(a.out) % 16 == 0 &&
                       a.ldo % 8 == 0 && attn_tma_out_enabled();
  const CUtensorMap to = tma_out ? make_tmap_3d(a.out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                                (uint64_t)a.heads * RP, a.seq, a.batch, a.ldo,
                                                (uint64_t)a.seq * a.ldo, RP, 32,
                                                swizzle_for_row_bytes(C::RB))
                                 : tm;
  if (tma_out)
    launch_attn_k<RP, X3, C::TMA_OUT>(a, s, tm, tkv, to, T);
  else
    launch_attn_k<RP, X3, false>(a, s, tm, tkv, to, T);
}

}  // namespace

bool attn_rankspace_supported(int rank_pad) {
  return rank_pad == 16 || rank_pad == 32 || rank_pad == 64;
}

void attn_rankspace_bf16(const AttnTcArgs& a, cudaStream_t s) {
  if (a.planes) {  // split planes (fp32 policy)
    switch (a.rank_pad) {
      case 16: launch_attn<16, true>(a, s); return;
      case 32: launch_attn<32, true>(a, s); return;
      case 64: launch_attn<64, true>(a, s); return;
      default: throw CudaError("attn_rankspace (planes): unsupported rank padding");
    }
  }
  switch (a.rank_pad) {
    case 16: launch_attn<16>(a, s); break;
    case 32: launch_attn<32>(a, s); break;
    case 64: launch_attn<64>(a, s); break;
    default: throw CudaError("attn_rankspace_bf16: unsupported rank padding");
  }
}

}  // namespace fsvd
