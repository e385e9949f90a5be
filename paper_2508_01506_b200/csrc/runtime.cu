// runtime.cu -- factor packs, activation buffer planner and the device
// encoder schedule.
//
// Layer schedule (post-LN, encoder.cpp:241-247), bf16 tensor-core path:
//   K1  P      = X Wqkv^T                      [T, 3*G*rp]   (attention.cpp:239-247)
//   K2  ctx    = FlashSVD attention(P)         [T, d]        (attention.cpp:249-267)
//   K1  Pout   = ctx Uo^T ; K1 branch = Pout Vo^T + b_o      (attention.cpp:381-389)
//   K5  resid  = LN1(x + branch)                              (encoder.cpp:38-50)
//   FFN V1: K1 P = resid Uup^T ; K3 Z = stream(P) ; K1 out = Z Vdn^T + b  (ffn.cpp:118-156)
//   FFN V2: K4 out = fused(resid)                             (ffn.cpp:158-185)
//   K5  y      = LN2(resid + ffn_out)
// Buffers: two [T, d] scratch activations (ctx/branch/resid/ffn_out rotate
// through them in place) plus one transient region sized by RANK, aliased by
// every sublayer: max(3*G*rp, prp, 2*frp) elements per token.  The layer runs
// in place (x may equal out), so a whole model needs no ping-pong pair.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>

#include "common.cuh"
#include "runtime.hpp"

namespace fsvd {

uint16_t f32_to_bf16_bits(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}

Pack::~Pack() {
  if (mem) cudaFree(mem);
}

namespace {


size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Builder {
  std::vector<uint8_t> buf;
  int es;
  std::vector<std::pair<const void**, size_t>> fix;
  std::vector<std::pair<const float**, size_t>> fixf;

  size_t raw(const void* p, size_t bytes) {
    const size_t off = align256(buf.size());
    buf.resize(off + bytes);
    if (bytes) std::memcpy(buf.data() + off, p, bytes);
    return off;
  }
  void store(const void** dst, const std::vector<float>& v) {
    size_t off;
    if (es == 4) {
      off = raw(v.data(), v.size() * 4);
    } else {
      std::vector<uint16_t> h(v.size());
      for (size_t i = 0; i < v.size(); ++i) h[i] = f32_to_bf16_bits(v[i]);
      off = raw(h.data(), h.size() * 2);
    }
    fix.push_back({dst, off});
  }
  // split planes (fp32 policy, kernels.cuh): hi = bf16(v), mid = bf16(v - hi),
  // lo = bf16(v - hi - mid), stored contiguously; *hi -> the hi plane,
  // *mid -> the mid plane (the plane stride is mid - hi)
  void store_planes(const void** hi, const void** mid, const std::vector<float>& v) {
    const size_t n = v.size();
    std::vector<uint16_t> h(3 * n);
    auto widen = [](uint16_t b) {
      uint32_t u = static_cast<uint32_t>(b) << 16;
      float f;
      std::memcpy(&f, &u, 4);
      return f;
    };
    for (size_t i = 0; i < n; ++i) {
      float r = v[i];
      for (int pl = 0; pl < 3; ++pl) {
        h[pl * n + i] = f32_to_bf16_bits(r);
        r -= widen(h[pl * n + i]);
      }
    }
    const size_t off = raw(h.data(), h.size() * 2);
    fix.push_back({hi, off});
    fix.push_back({mid, off + n * 2});
  }
  // tensor-core weight layout: bf16 (bf16 policy) or split planes (x3)
  bool x3 = false;
  void tc(const void** dst, const void** dst_lo, const std::vector<float>& v) {
    if (x3) store_planes(dst, dst_lo, v);
    else store(dst, v);
  }
  void store_f32(const float** dst, const float* p, size_t n) { fixf.push_back({dst, raw(p, n * 4)}); }
  void store_f32(const float** dst, const std::vector<float>& v) { store_f32(dst, v.data(), v.size()); }
};

int pad_to(int x, int m) { return (x + m - 1) / m * m; }

// n values followed by zeros up to length m
std::vector<float> padded(const float* v, int n, int m) {
  std::vector<float> out(static_cast<size_t>(m), 0.0f);
  std::copy(v, v + n, out.begin());
  return out;
}

// W^T[n][k] = sum_j U[k][j] V[j][n] (fp32 accumulate, j ascending) for the
// dense twin (encoder.cpp:295-331 reconstructs W = U V the same way).
std::vector<float> reconstruct_t(const float* u, const float* v, int K, int R, int N, int ldv,
                                 int voff) {
  std::vector<float> wt(static_cast<size_t>(N) * K);
  auto work = [&](int n_begin, int n_end) {
    for (int n = n_begin; n < n_end; ++n)
      for (int k = 0; k < K; ++k) {
        float acc = 0.0f;
        for (int j = 0; j < R; ++j) acc += u[(size_t)k * R + j] * v[(size_t)j * ldv + voff + n];
        wt[(size_t)n * K + k] = acc;
      }
  };
  const int nt = 8;
  std::vector<std::thread> ts;
  for (int t = 0; t < nt; ++t) ts.emplace_back(work, N * t / nt, N * (t + 1) / nt);
  for (auto& t : ts) t.join();
  return wt;
}

}  // namespace

namespace {
// Dense-mode weights (see Pack): from q.dense_w, or rebuilt from the factors
// exactly as dense_equivalent does (encoder.cpp:295-331: W = U V per group,
// reconstruct_t's fp32 j-ascending sums).
void build_dense(const PackRequest& q, Pack& p, Builder& b) {
  // d: the callers' model dimension; D: the padded layout (see build_pack)
  const int d = p.dr, D = p.d, H = static_cast<int>(q.heads), dh = d / H;
  const int dhp = dh <= 16 ? 16 : dh <= 32 ? 32 : 64, hp = H * dhp;
  const double sc = 1.4426950408889634 / std::sqrt(static_cast<double>(dh));
  const fsvd_dense_layer* w = q.dense_w;
  const int df = w ? static_cast<int>(w->d_ff) : static_cast<int>(q.ffn->up.out_dim);
  const int dfp = pad_to(df, 8);
  p.dhp = dhp;
  p.ddf = dfp;
  p.H = H;
  p.dh = dh;
  p.dact = q.ffn ? static_cast<int>(q.ffn->activation) : q.dense_act;
  // W^T of the three projections, [n][k] = W[k][n]
  std::vector<float> wt[3];
  std::vector<float> bias(3 * (size_t)d);
  if (w) {
    const float* ws[3] = {w->wq, w->wk, w->wv};
    const float* bs[3] = {w->bq, w->bk, w->bv};
    for (int m = 0; m < 3; ++m) {
      wt[m].resize((size_t)d * d);
      for (int k = 0; k < d; ++k)
        for (int n = 0; n < d; ++n) wt[m][(size_t)n * d + k] = ws[m][(size_t)k * d + n];
      std::copy(bs[m], bs[m] + d, bias.begin() + (size_t)m * d);
    }
  } else {
    const fsvd_attn_desc& a = *q.attn;
    const int G = static_cast<int>(a.groups), r = static_cast<int>(a.rank), gd = d / G;
    for (int m = 0; m < 3; ++m) {
      wt[m].resize((size_t)d * d);
      for (int g = 0; g < G; ++g) {
        std::vector<float> part = reconstruct_t(a.u + (size_t)(m * G + g) * d * r,
                                                a.v + (size_t)(m * G + g) * r * gd, d, r, gd, gd, 0);
        std::copy(part.begin(), part.end(), wt[m].begin() + (size_t)g * gd * d);
      }
    }
    std::copy(a.bias, a.bias + 3 * (size_t)d, bias.begin());
  }
  std::vector<float> qkv((size_t)3 * hp * D, 0.0f), bq((size_t)3 * hp, 0.0f);
  for (int m = 0; m < 3; ++m)
    for (int h = 0; h < H; ++h)
      for (int c = 0; c < dh; ++c) {
        const float f = m == 0 ? static_cast<float>(sc) : 1.0f;
        const size_t row = (size_t)m * hp + (size_t)h * dhp + c, src = (size_t)h * dh + c;
        for (int k = 0; k < d; ++k) qkv[row * D + k] = wt[m][src * d + k] * f;
        bq[row] = bias[(size_t)m * d + src] * f;
      }
  b.tc(&p.dqkv_t, &p.dqkv_lo, qkv);
  b.store_f32(&p.dqkv_b, bq);
  // output projection W_o^T [D][H dhp], padded rows and head columns zero
  std::vector<float> wo_t = w ? std::vector<float>((size_t)d * d)
                              : reconstruct_t(q.out_proj->u, q.out_proj->v, d,
                                              static_cast<int>(q.out_proj->rank), d, d, 0);
  if (w)
    for (int k = 0; k < d; ++k)
      for (int n = 0; n < d; ++n) wo_t[(size_t)n * d + k] = w->wo[(size_t)k * d + n];
  std::vector<float> wop((size_t)D * hp, 0.0f);
  for (int n = 0; n < d; ++n)
    for (int h = 0; h < H; ++h)
      for (int c = 0; c < dh; ++c)
        wop[(size_t)n * hp + (size_t)h * dhp + c] = wo_t[(size_t)n * d + h * dh + c];
  b.tc(&p.do_t, &p.do_lo, wop);
  b.store_f32(&p.dbo, padded(w ? w->bo : q.out_proj->bias, d, D));
  // FFN: W_in^T [dfp][D], W_out^T [D][dfp]
  std::vector<float> win((size_t)dfp * D, 0.0f), wout((size_t)D * dfp, 0.0f);
  if (w) {
    for (int k = 0; k < d; ++k)
      for (int n = 0; n < df; ++n) win[(size_t)n * D + k] = w->w_in[(size_t)k * df + n];
    for (int k = 0; k < df; ++k)
      for (int n = 0; n < d; ++n) wout[(size_t)n * dfp + k] = w->w_out[(size_t)k * d + n];
  } else {
    const fsvd_ffn_desc& f = *q.ffn;
    const int fr = static_cast<int>(f.up.rank);
    const std::vector<float> a = reconstruct_t(f.up.u, f.up.v, d, fr, df, df, 0);    // [df][d]
    const std::vector<float> c = reconstruct_t(f.down.u, f.down.v, df, fr, d, d, 0);  // [d][df]
    for (int n = 0; n < df; ++n)
      for (int k = 0; k < d; ++k) win[(size_t)n * D + k] = a[(size_t)n * d + k];
    for (int n = 0; n < d; ++n)
      for (int k = 0; k < df; ++k) wout[(size_t)n * dfp + k] = c[(size_t)n * df + k];
  }
  b.tc(&p.din_t, &p.din_lo, win);
  b.tc(&p.dout_t, &p.dout_lo, wout);
  b.store_f32(&p.dbin, padded(w ? w->b_in : q.ffn->up.bias, df, dfp));
  b.store_f32(&p.dbout, padded(w ? w->b_out : q.ffn->down.bias, d, D));
}
}  // namespace

Pack* build_pack(const PackRequest& q, fsvd_dtype dtype) {
  auto P = std::make_unique<Pack>();
  Pack& p = *P;
  p.dtype = dtype;
  p.es = dtype == FSVD_BF16 ? 2 : 4;  // split-plane packs: 6 (set below)
  Builder b;
  b.es = p.es;
  const bool bf = dtype == FSVD_BF16;
  // d: the model dimension of the caller's arrays; D: the model dimension of
  // the device layouts -- d rounded up to 64 with zero rows / columns when the
  // whole pack runs on the tensor cores, so every shape the reference accepts
  // fits the kernels' tiling (K3/K4 need d % 64, TMA 16-byte row pitches).
  // LayerNorm statistics use d (runtime ln); the host API pads and unpads.
  const int d = static_cast<int>(q.d_model);
  bool attn_ok = true, out_ok = true, ffn_ok = true, dense_ok = true;
  if (q.attn) {
    const int r = static_cast<int>(q.attn->rank);
    const int rp = r <= 16 ? 16 : r <= 32 ? 32 : r <= 64 ? 64 : 0;
    attn_ok = rp != 0 && attn_rankspace_supported(rp);
  }
  if (q.ffn) ffn_ok = ffn_rank_pad(static_cast<int>(q.ffn->up.rank)) <= kFfnMaxRankPad;
  // Dense-mode weights: any head width <= 64 (padded to 16 / 32 / 64)
  if (q.dense) {
    const int df = q.dense_w ? static_cast<int>(q.dense_w->d_ff)
                             : (q.ffn ? static_cast<int>(q.ffn->up.out_dim) : 0);
    dense_ok = q.heads > 0 && d % q.heads == 0 && d / static_cast<int>(q.heads) <= 64 && df > 0 &&
               (q.dense_w != nullptr || (q.attn && q.out_proj && q.ffn));
  }
  const bool all_ok = attn_ok && out_ok && ffn_ok && dense_ok;
  const int D = all_ok ? pad_to(d, 64) : d;
  if (!all_ok) {  // bf16 per component on the unpadded layout (CUDA cores otherwise)
    attn_ok = attn_ok && d % 8 == 0;
    out_ok = d % 8 == 0;
    if (q.ffn) {
      const int df = static_cast<int>(q.ffn->up.out_dim);
      ffn_ok = ffn_ok && d % 8 == 0 && df % 8 == 0 &&
               ffn_tc_supported(d, df, ffn_rank_pad(static_cast<int>(q.ffn->up.rank)));
    }
  }
  p.d = D;
  p.dr = d;
  p.x3 = !bf && all_ok;
  b.x3 = p.x3;
  if (p.x3) p.es = 2 * kPlanes;  // three bf16 planes per stored value

  if (q.attn) {
    const fsvd_attn_desc& a = *q.attn;
    p.has_attn = true;
    p.H = static_cast<int>(q.heads);
    p.G = static_cast<int>(a.groups);
    p.r = static_cast<int>(a.rank);
    p.dh = d / p.H;
    p.gd = d / p.G;
    const int G = p.G, r = p.r, H = p.H, dh = p.dh, gd = p.gd, hpg = H / G;
    p.rp = r <= 16 ? 16 : r <= 32 ? 32 : r <= 64 ? 64 : 0;
    p.attn_tc = bf && attn_ok;
    if (p.attn_tc || p.x3) {
      // Folded rank-space projection (attn_tc.cu): rows [0, H*rp) hold
      // Qt_h = s * U_q,g (V_q,h V_k,h^T), rows [H*rp, (H+G)*rp) U_k,g, then U_v,g.
      const int rp = p.rp;
      const double sc = 1.4426950408889634 / std::sqrt(static_cast<double>(dh));
      p.qkv_cols = (H + 2 * G) * rp;
      std::vector<float> w((size_t)p.qkv_cols * D, 0.0f), bp((size_t)p.qkv_cols, 0.0f);
      std::vector<double> mh((size_t)r * r);
      for (int h = 0; h < H; ++h) {
        const int g = h / hpg, hc = (h % hpg) * dh;
        const float* vq = a.v + (size_t)(0 * G + g) * r * gd;
        const float* vk = a.v + (size_t)(1 * G + g) * r * gd;
        const float* uq = a.u + (size_t)(0 * G + g) * d * r;
        for (int j = 0; j < r; ++j)
          for (int i = 0; i < r; ++i) {
            double acc = 0.0;
            for (int c = 0; c < dh; ++c) acc += (double)vq[(size_t)j * gd + hc + c] * vk[(size_t)i * gd + hc + c];
            mh[(size_t)j * r + i] = acc * sc;
          }
        for (int i = 0; i < r; ++i) {
          float* row = &w[((size_t)h * rp + i) * D];
          for (int k = 0; k < d; ++k) {
            double acc = 0.0;
            for (int j = 0; j < r; ++j) acc += (double)uq[(size_t)k * r + j] * mh[(size_t)j * r + i];
            row[k] = static_cast<float>(acc);
          }
          double bb = 0.0;
          for (int c = 0; c < dh; ++c) bb += (double)a.bias[h * dh + c] * vk[(size_t)i * gd + hc + c];
          bp[(size_t)h * rp + i] = static_cast<float>(bb * sc);
        }
      }
      for (int m = 1; m < 3; ++m)
        for (int g = 0; g < G; ++g)
          for (int j = 0; j < r; ++j)
            for (int k = 0; k < d; ++k)
              w[((size_t)(H + (m - 1) * G + g) * rp + j) * D + k] =
                  a.u[((size_t)(m * G + g) * d + k) * r + j];
      b.tc(&p.wproj_t, &p.wproj_lo, w);
      b.store_f32(&p.bproj, bp);
      // block-diagonal V_v: ctx[:, h*dh + c] = sum_j O_h[:, j] V_v,g[j, hc + c] (+ b_v)
      std::vector<float> vc((size_t)D * H * rp, 0.0f);
      for (int h = 0; h < H; ++h) {
        const int g = h / hpg, hc = (h % hpg) * dh;
        for (int c = 0; c < dh; ++c)
          for (int j = 0; j < r; ++j)
            vc[((size_t)h * dh + c) * H * rp + (size_t)h * rp + j] =
                a.v[((size_t)(2 * G + g) * r + j) * gd + hc + c];
      }
      b.tc(&p.wvc_t, &p.wvc_lo, vc);
      b.store_f32(&p.bv, padded(a.bias + 2 * d, d, D));
    } else {
      std::vector<float> w((size_t)d * 3 * G * r);
      for (int m = 0; m < 3; ++m)
        for (int g = 0; g < G; ++g)
          for (int k = 0; k < d; ++k)
            for (int j = 0; j < r; ++j)
              w[(size_t)k * 3 * G * r + (size_t)(m * G + g) * r + j] =
                  a.u[((size_t)(m * G + g) * d + k) * r + j];
      b.store(&p.wqkv, w);
      b.store(&p.attn_v, std::vector<float>(a.v, a.v + (size_t)3 * G * r * gd));
    }
    b.store_f32(&p.attn_b, a.bias, 3 * (size_t)d);
    if (q.dense && (p.attn_tc || p.x3) && (dh == 16 || dh == 32 || dh == 64) && D == d) {
      // NaiveLowRank (attention.cpp:271-292): P = X [U_q|U_k|U_v], then the
      // block-diagonal V rebuilds dense Q|K|V [T, 3d] (Q scaled by s)
      const float sc = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(dh)));
      const int rp = p.rp;
      std::vector<float> wn((size_t)3 * G * rp * d, 0.0f);
      for (int m = 0; m < 3; ++m)
        for (int g = 0; g < G; ++g)
          for (int j = 0; j < r; ++j)
            for (int k = 0; k < d; ++k)
              wn[((size_t)(m * G + g) * rp + j) * d + k] = a.u[((size_t)(m * G + g) * d + k) * r + j];
      b.tc(&p.wpn_t, &p.wpn_lo, wn);
      std::vector<float> bd((size_t)3 * d * 3 * G * rp, 0.0f);
      for (int m = 0; m < 3; ++m)
        for (int g = 0; g < G; ++g)
          for (int c = 0; c < gd; ++c)
            for (int j = 0; j < r; ++j)
              bd[((size_t)m * d + g * gd + c) * (3 * G * rp) + (m * G + g) * rp + j] =
                  a.v[((size_t)(m * G + g) * r + j) * gd + c] * (m == 0 ? sc : 1.0f);
      b.tc(&p.dvbd_t, &p.dvbd_lo, bd);
      std::vector<float> bq(a.bias, a.bias + 3 * (size_t)d);
      for (int i = 0; i < d; ++i) bq[i] *= sc;
      b.store_f32(&p.nqkv_b, bq);
    }
  }
  if (q.out_proj) {
    const fsvd_linear_desc& o = *q.out_proj;
    p.has_out = true;
    p.pr = static_cast<int>(o.rank);
    p.prp = pad_to(p.pr, 16);
    p.out_tc = bf && out_ok;
    if (p.out_tc || p.x3) {
      const int pr = p.pr, prp = p.prp;
      std::vector<float> ut((size_t)prp * D, 0.0f), vt((size_t)D * prp, 0.0f);
      for (int k = 0; k < d; ++k)
        for (int j = 0; j < pr; ++j) ut[(size_t)j * D + k] = o.u[(size_t)k * pr + j];
      for (int j = 0; j < pr; ++j)
        for (int n = 0; n < d; ++n) vt[(size_t)n * prp + j] = o.v[(size_t)j * d + n];
      b.tc(&p.uo_t, &p.uo_t_lo, ut);
      b.tc(&p.vo_t, &p.vo_t_lo, vt);
      if (q.attn && (p.attn_tc || p.x3)) {
        // W_o = U_o V_o; stored transposed: wo_t[n][m] = W_o[m][n]
        std::vector<float> wo_t = reconstruct_t(o.u, o.v, d, pr, d, d, 0);
        if (q.attn && (p.attn_tc || p.x3)) {
          // folded rank-space out-projection: W_ov[(h, j)][n] = sum_c V_v,h[j, c] W_o[h dh + c][n]
          const fsvd_attn_desc& a = *q.attn;
          const int H = p.H, G = p.G, r = p.r, rp = p.rp, dh = p.dh, gd = p.gd, hpg = H / G;
          std::vector<float> wov((size_t)D * H * rp, 0.0f), bov(D, 0.0f);
          for (int n = 0; n < d; ++n) {
            const float* won = &wo_t[(size_t)n * d];
            for (int h = 0; h < H; ++h) {
              const int g = h / hpg, hc = (h % hpg) * dh;
              for (int j = 0; j < r; ++j) {
                const float* vv = a.v + ((size_t)(2 * G + g) * r + j) * gd + hc;
                double acc = 0.0;
                for (int c = 0; c < dh; ++c) acc += (double)vv[c] * won[h * dh + c];
                wov[(size_t)n * H * rp + (size_t)h * rp + j] = static_cast<float>(acc);
              }
            }
            double bb = o.bias[n];
            for (int m = 0; m < d; ++m) bb += (double)a.bias[2 * d + m] * won[m];
            bov[n] = static_cast<float>(bb);
          }
          b.tc(&p.wov_t, &p.wov_lo, wov);
          b.store_f32(&p.bov, bov);
        }
      }
    } else {
      b.store(&p.uo, std::vector<float>(o.u, o.u + (size_t)d * o.rank));
      b.store(&p.vo, std::vector<float>(o.v, o.v + (size_t)o.rank * d));
    }
    b.store_f32(&p.bo, padded(o.bias, d, (p.out_tc || p.x3) ? D : d));
  }
  if (q.ffn) {
    const fsvd_ffn_desc& f = *q.ffn;
    p.has_ffn = true;
    p.fr = static_cast<int>(f.up.rank);
    p.df = static_cast<int>(f.up.out_dim);
    p.act = static_cast<int>(f.activation);
    p.frp = ffn_rank_pad(p.fr);
    const int fr = p.fr, frp = p.frp, df = p.df;
    p.ffn_tc = bf && ffn_ok;
    p.ffn_wide = p.ffn_tc && frp > 384;
    if (p.ffn_tc || p.x3) {
      const int dfp = all_ok ? pad_to(df, 8) : df;  // padded d_ff rows / columns are zero
      p.df = dfp;
      std::vector<float> uu((size_t)frp * D, 0.0f), vu((size_t)dfp * frp, 0.0f),
          ud((size_t)frp * dfp, 0.0f), vd((size_t)D * frp, 0.0f);
      for (int k = 0; k < d; ++k)
        for (int j = 0; j < fr; ++j) uu[(size_t)j * D + k] = f.up.u[(size_t)k * fr + j];
      for (int j = 0; j < fr; ++j)
        for (int c = 0; c < df; ++c) vu[(size_t)c * frp + j] = f.up.v[(size_t)j * df + c];
      for (int c = 0; c < df; ++c)
        for (int j = 0; j < fr; ++j) ud[(size_t)j * dfp + c] = f.down.u[(size_t)c * fr + j];
      for (int j = 0; j < fr; ++j)
        for (int n = 0; n < d; ++n) vd[(size_t)n * frp + j] = f.down.v[(size_t)j * d + n];
      b.tc(&p.uup_t, &p.uup_t_lo, uu);
      b.tc(&p.vup_t, &p.vup_t_lo, vu);
      b.tc(&p.udn_t, &p.udn_t_lo, ud);
      b.tc(&p.vdn_t, &p.vdn_t_lo, vd);
    } else {
      b.store(&p.uup, std::vector<float>(f.up.u, f.up.u + (size_t)d * fr));
      b.store(&p.vup, std::vector<float>(f.up.v, f.up.v + (size_t)fr * df));
      b.store(&p.udn, std::vector<float>(f.down.u, f.down.u + (size_t)df * fr));
      b.store(&p.vdn, std::vector<float>(f.down.v, f.down.v + (size_t)fr * d));
    }
    b.store_f32(&p.bup, padded(f.up.bias, df, p.df));
    b.store_f32(&p.bdn, padded(f.down.bias, d, (p.ffn_tc || p.x3) ? D : d));
  }
  if (q.dense && all_ok) build_dense(q, p, b);
  if (q.ln1g) {
    p.has_ln = true;
    b.store_f32(&p.ln1g, padded(q.ln1g, d, D));
    b.store_f32(&p.ln1b, padded(q.ln1b, d, D));
    b.store_f32(&p.ln2g, padded(q.ln2g, d, D));
    b.store_f32(&p.ln2b, padded(q.ln2b, d, D));
    p.eps1 = q.eps1;
    p.eps2 = q.eps2;
  }
  p.dense = q.dense && all_ok;
  p.bytes = align256(b.buf.size());
  if (p.bytes) {
    FSVD_CUDA_CHECK(cudaMalloc(&p.mem, p.bytes));
    FSVD_CUDA_CHECK(cudaMemcpy(p.mem, b.buf.data(), b.buf.size(), cudaMemcpyHostToDevice));
  }
  auto* base = static_cast<uint8_t*>(p.mem);
  for (auto& f : b.fix) *f.first = base + f.second;
  for (auto& f : b.fixf) *f.first = reinterpret_cast<const float*>(base + f.second);
  return P.release();
}

// ---------------------------------------------------------------- validation
// EncoderLayer::validate (encoder.cpp:156-221) on the flat descriptor: the
// factorized attention (attn.u set, with out_proj), the factorized FFN
// (ffn.up.u set) and the dense weights (L.dense) are each optional, but each
// sublayer needs one representation.
void validate_layer(const fsvd_layer_desc& L) {
  const size_t d = L.attn.d_model;
  if (d == 0) fail(Kind::Shape, "layer norm parameters are empty");
  if (!L.ln1_gamma || !L.ln1_beta || !L.ln2_gamma || !L.ln2_beta)
    fail(Kind::Shape, "layer norm parameters are missing");
  if (L.heads == 0 || d % L.heads != 0) fail(Kind::Config, "heads must divide d_model");
  const bool af = L.attn.u != nullptr, ff = L.ffn.up.u != nullptr, dn = L.dense != nullptr;
  if (!dn && !af) fail(Kind::Config, "layer has no attention weights");
  if (!dn && !ff) fail(Kind::Config, "layer has no FFN weights");
  if (L.out_proj.u && !af) fail(Kind::Config, "output projection factors without attention factors");
  if (af) {
    const fsvd_attn_desc& s = L.attn;
    if (s.groups == 0 || d % s.groups != 0) fail(Kind::Config, "groups must divide d_model");
    if (L.heads % s.groups != 0) fail(Kind::Config, "groups must divide heads");
    if (s.rank == 0 || !s.v || !s.bias) fail(Kind::Shape, "attention factor U: missing");
    const fsvd_linear_desc& o = L.out_proj;
    if (!o.u) fail(Kind::Config, "factorized attention needs an output projection");
    if (o.in_dim != d) fail(Kind::Shape, "out_proj U: expected shape (d, r)");
    if (o.out_dim != d || !o.v) fail(Kind::Shape, "out_proj V: expected shape (r, d)");
    if (!o.bias) fail(Kind::Shape, "out_proj bias: expected a length-d vector");
    if (o.rank == 0) fail(Kind::Shape, "factor rank must be positive");
  }
  if (dn) {
    const fsvd_dense_layer& w = *L.dense;
    if (w.d_model != d) fail(Kind::Shape, "attention weight: expected shape (d, d)");
    for (const float* m : {w.wq, w.wk, w.wv, w.wo})
      if (!m) fail(Kind::Shape, "attention weight: expected shape (d, d)");
    for (const float* b : {w.bq, w.bk, w.bv, w.bo})
      if (!b) fail(Kind::Shape, "attention bias: expected a length-d vector");
  }
  const size_t df = ff ? L.ffn.up.out_dim : (dn ? L.dense->d_ff : 0);
  if (ff) {
    const fsvd_ffn_desc& f = L.ffn;
    if (f.up.rank != f.down.rank) fail(Kind::Config, "FFN up/down factor ranks differ");
    if (f.up.in_dim != d) fail(Kind::Shape, "ffn up U: expected shape (d, r)");
    if (f.down.out_dim != d || !f.down.v) fail(Kind::Shape, "ffn down V: expected shape (r, d)");
    if (f.up.out_dim != f.down.in_dim || f.up.out_dim == 0)
      fail(Kind::Shape, "ffn up V / down U: d_ff mismatch");
    if (!f.up.v || !f.up.bias || !f.down.u || !f.down.bias)
      fail(Kind::Shape, "ffn factor arrays are missing");
    if (f.up.rank == 0) fail(Kind::Shape, "factor rank must be positive");
  }
  if (dn) {
    const fsvd_dense_layer& w = *L.dense;
    if (w.d_ff != df || df == 0 || !w.w_in) fail(Kind::Shape, "ffn input weight: expected shape (d, d_ff)");
    if (!w.b_in) fail(Kind::Shape, "ffn input bias: expected a length-d_ff vector");
    if (!w.w_out) fail(Kind::Shape, "ffn output weight: expected shape (d_ff, d)");
    if (!w.b_out) fail(Kind::Shape, "ffn output bias: expected a length-d vector");
  }
  if (static_cast<int>(L.ffn.activation) < 0 || static_cast<int>(L.ffn.activation) > 3)
    fail(Kind::Config, "unknown activation");
}

// encoder.cpp:27-35 (check_mode_weights)
void check_mode_weights(const fsvd_layer_desc& L, int mode, bool dense_twin_ok) {
  const bool factors = L.attn.u && L.out_proj.u && L.ffn.up.u;
  if (mode == FSVD_MODE_DENSE) {
    if (!L.dense && !(dense_twin_ok && factors))
      fail(Kind::Config, "dense mode needs dense weights on both sublayers");
  } else if (!factors) {
    static const char* names[4] = {"dense", "naive_lowrank", "flash_v1", "flash_v2"};
    fail(Kind::Config, std::string(names[mode & 3]) + " mode needs factorized weights on both sublayers");
  }
}

// ---------------------------------------------------------------- planner
size_t op_transient_elems(const Pack& p, int op, int mode) {
  if (op == 0 || (op == 3 && (mode == FSVD_MODE_DENSE || mode == FSVD_MODE_NAIVE_LOWRANK))) {
    // materializing baselines: Q|K|V [3 H dhp] (+ naive P [3 G rp]) + context [H dhp]
    const size_t hp = (size_t)p.H * p.dhp;
    if (mode == FSVD_MODE_DENSE) return 4 * hp;
    if (mode == FSVD_MODE_NAIVE_LOWRANK) return 3 * (size_t)p.G * p.rp + 4 * hp;
    return (p.attn_tc || p.x3) ? (size_t)p.qkv_cols + (size_t)p.H * p.rp
                               : 3 * (size_t)p.G * p.r;
  }
  if (op == 1) {
    if (mode == FSVD_MODE_DENSE) return 0;
    return (p.out_tc || p.x3) ? p.prp : p.pr;
  }
  if (op == 3) {  // attention inside a layer (rank-space output goes to scratch)
    if (p.attn_tc && p.out_tc && (mode == FSVD_MODE_FLASH_V1 || mode == FSVD_MODE_FLASH_V2))
      return p.qkv_cols;
    return op_transient_elems(p, 0, mode);  // split planes: O after the projection
  }
  const size_t fr = (p.ffn_tc || p.x3) ? p.frp : p.fr;
  switch (mode) {
    case FSVD_MODE_DENSE: return p.ddf;
    case FSVD_MODE_NAIVE_LOWRANK: return 2 * fr + p.df;
    case FSVD_MODE_FLASH_V1: return 2 * fr;
    default: return (p.ffn_wide || p.x3) ? 2 * fr : 0;  // wide ranks / planes: V2 runs the V1 chain
  }
}

namespace {
// 128-row tiles per sequence for the kernels' loop rotation (ln_epi.cuh
// piece_of, FfnTcArgs::seq_tiles); 0 when tiles straddle sequences.
int seq_tiles_of(size_t M) { return M % 128 == 0 ? static_cast<int>(M / 128) : 0; }
// Fused post-LN tensor-core schedule (layer_fwd): rank-space attention output
// A [T, H*rp], LN1 output B [T, d], transient QKV / FFN-V1 region; A holds a
// [T, d] FFN output instead when the FFN cannot take its LN fused.
bool fused_ln_disabled() {
  static const bool off = [] {
    const char* e = getenv("FSVD_UNFUSED_LN");  // developer switch: K5 LayerNorms
    return e && e[0] == '1';
  }();
  return off;
}
bool fused_post_ln(const Pack& p, int mode) {
  const bool flash = mode == FSVD_MODE_FLASH_V1 || mode == FSVD_MODE_FLASH_V2;
  return flash && p.attn_tc && p.out_tc && p.d == p.dr && gemm_ln_supported(p.d, p.H * p.rp) &&
         !fused_ln_disabled();
}
bool ffn_ln_fusable(const Pack& p, int mode) {
  return p.ffn_tc && p.d == p.dr && gemm_ln_supported(p.d, p.frp) &&
         (mode == FSVD_MODE_FLASH_V1 || mode == FSVD_MODE_FLASH_V2);
}
struct WsLayout {
  size_t a, b, t;  // bytes of the A / B / transient regions (256-aligned)
  size_t total() const { return a + b + t + 256; }
  int chunks = 0;  // > 0: the compact fused post-LN layout (qkv_chunks)
  bool unfused_compact = false;  // the compact post-LN layout with K5 LayerNorms
};
// Compact fused post-LN layout (both LayerNorms fused, full attention): the
// LN1 output goes straight into the layer's output buffer (K6 runs in place
// over the residual when out == x, the FFN kernel in place over out: every
// CTA reads its 128 rows before it writes them); region A [T, H*rp] holds Qt
// from the projection and then, in the same cells, K2's rank-space output;
// the [P_k | P_v] columns -- dead once K2 has read them -- go to a transient
// of one chunk of sequences: K1 and K2 run chunk by chunk (qkv_chunks()).
// The FFN V1 chain's P | Z reuse A and the transient.
int qkv_chunks(size_t B) {
  static const int env = [] {
    // memory / speed knob: 1 (default) holds [P_k | P_v] for the whole batch;
    // n > 1 runs K1 + K2 over n chunks of sequences (transient / n, at the
    // cost of n - 1 more kernel ramps per layer: ~5% at cfg2 for n = 2)
    const char* e = getenv("FSVD_QKV_CHUNKS");
    return e ? atoi(e) : 1;
  }();
  const int c = env < 1 ? 1 : env;
  return static_cast<int>(std::min<size_t>(B, static_cast<size_t>(c)));
}
// Post-LN tensor-core layers whose LayerNorms cannot ride in the GEMM
// epilogues (d > 768: the parked row exceeds TMEM): A [T, d] holds the
// attention branch and then the FFN branch; the transient holds [Qt | P_k |
// P_v] with K2's output written over Qt, then the FFN chain's P | Z; both
// LayerNorms (K5) write the layer's output buffer.
bool compact_unfused_post_ln(const Pack& p, int mode) {
  const bool flash = mode == FSVD_MODE_FLASH_V1 || mode == FSVD_MODE_FLASH_V2;
  return flash && p.attn_tc && p.out_tc && p.ffn_tc && p.dtype == FSVD_BF16 && !p.x3 &&
         !fused_post_ln(p, mode);
}
bool compact_post_ln(const Pack& p, int mode) {
  return fused_post_ln(p, mode) && ffn_ln_fusable(p, mode) && (p.H * p.rp) % 64 == 0 &&
         p.dtype == FSVD_BF16;
}
WsLayout ws_layout(const Pack& p, size_t B, size_t M, int mode, bool pre_ln, bool compact) {
  const size_t T = B * M;
  if (!pre_ln && compact && compact_post_ln(p, mode)) {
    const int c = qkv_chunks(B);
    const size_t cb = (B + c - 1) / c;  // sequences per chunk
    const size_t hr = static_cast<size_t>(p.H * p.rp), kvw = 2 * static_cast<size_t>(p.G * p.rp);
    const size_t a = align256(T * hr * p.es);
    size_t t = align256(cb * M * kvw * p.es);
    if (mode == FSVD_MODE_FLASH_V1 || p.ffn_wide) {  // P | Z of the V1 chain over A + transient
      const size_t pz = align256(2 * T * p.frp * p.es);
      if (pz > a + t) t = pz - a;
    }
    WsLayout w{a, 0, t};
    w.chunks = c;
    return w;
  }
  if (!pre_ln && compact && compact_unfused_post_ln(p, mode)) {
    const size_t tcols = std::max<size_t>(p.qkv_cols, op_transient_elems(p, 2, mode));
    WsLayout w{align256(T * p.d * p.es), 0, align256(T * tcols * p.es)};
    w.unfused_compact = true;
    return w;
  }
  if (!pre_ln && fused_post_ln(p, mode)) {
    const bool ffn_fused = ffn_ln_fusable(p, mode);
    const size_t a_cols = ffn_fused ? static_cast<size_t>(p.H * p.rp) : p.d;
    size_t t_cols = p.qkv_cols;
    if (mode == FSVD_MODE_FLASH_V1 || p.ffn_wide)
      t_cols = std::max(t_cols, 2 * static_cast<size_t>(p.frp));
    if (!ffn_fused) t_cols = std::max(t_cols, op_transient_elems(p, 2, mode));
    return {align256(T * a_cols * p.es), align256(T * p.d * p.es), align256(T * t_cols * p.es)};
  }
  size_t tr = 0;
  for (int op : {1, 2, 3}) tr = std::max(tr, op_transient_elems(p, op, mode));
  // B also holds the rank-space attention output [T, H*rp] on the pre-LN
  // tensor-core path (H*rp can exceed d when the rank padding exceeds dh)
  const size_t b_cols = std::max<size_t>(p.d, p.attn_tc ? static_cast<size_t>(p.H * p.rp) : 0);
  return {align256(T * p.d * p.es), align256(T * b_cols * p.es), align256(T * tr * p.es)};
}
}  // namespace

size_t layer_workspace_bytes(const Pack& p, size_t B, size_t M, int mode, bool pre_ln) {
  return ws_layout(p, B, M, mode, pre_ln, true).total();
}
size_t layer_workspace_bytes(const Pack& p, size_t B, size_t M, int mode) {
  return std::max(layer_workspace_bytes(p, B, M, mode, false),
                  layer_workspace_bytes(p, B, M, mode, true));
}
size_t prefill_workspace_bytes(const Pack& p, size_t B, size_t M, bool pre_ln) {
  return ws_layout(p, B, M, FSVD_MODE_FLASH_V2, pre_ln, false).total();
}

// ---------------------------------------------------------------- schedule
namespace {

template <typename T>
T* as(void* p) {
  return static_cast<T*>(p);
}
template <typename T>
const T* as(const void* p) {
  return static_cast<const T*>(p);
}

// split planes of a [rows, cols] activation buffer: hi plane, then lo plane
// split planes of a [rows, cols] activation buffer (n = rows x pitch): hi,
// mid, lo planes one after another
Planes pl(const void* p, size_t n) {
  const bf16* h = static_cast<const bf16*>(p);
  return {h, h + n, h + 2 * n};
}
PlanesOut plo(void* p, size_t n) {
  bf16* h = static_cast<bf16*>(p);
  return {h, h + n, h + 2 * n};
}
// a weight's planes: stored contiguously (Builder::store_planes), `mid` its
// second plane, so the plane stride is mid - hi
Planes wpl(const void* hi, const void* mid) {
  const bf16* h = static_cast<const bf16*>(hi);
  const bf16* m = static_cast<const bf16*>(mid);
  return {h, m, m + (m - h)};
}

void ln(const Pack& p, const void* a, const void* b, const float* g, const float* be, float eps,
        void* y, int rows, cudaStream_t s) {
  // statistics over the callers' d (p.dr); rows stored with the layout pitch p.d
  if (p.x3) {
    const size_t n = static_cast<size_t>(rows) * p.d;
    const Planes bp = b ? pl(b, n) : Planes{nullptr, nullptr, nullptr};
    ln_planes(pl(a, n), b ? &bp : nullptr, g, be, eps, plo(y, n), rows, p.dr, s, p.d);
    return;
  }
  if (p.dtype == FSVD_BF16)
    resid_layernorm_bf16(as<bf16>(a), as<bf16>(b), g, be, eps, as<bf16>(y), rows, p.dr, s, p.d);
  else
    resid_layernorm_f32(as<float>(a), as<float>(b), g, be, eps, as<float>(y), rows, p.dr, s, p.d);
}
void add(const Pack& p, const void* a, const void* b, void* y, int64_t n, cudaStream_t s) {
  if (p.x3) {
    add_planes(pl(a, n), pl(b, n), plo(y, n), n, s);
    return;
  }
  if (p.dtype == FSVD_BF16) add_bf16(as<bf16>(a), as<bf16>(b), as<bf16>(y), n, s);
  else add_f32(as<float>(a), as<float>(b), as<float>(y), n, s);
}

template <typename T>
void simt_attention_t(const Pack& p, size_t B, size_t M, const void* x, void* ctx, void* trans,
                      cudaStream_t s) {
  const int T_ = static_cast<int>(B * M), n = 3 * p.G * p.r;
  simt_gemm<T>(as<T>(x), p.d, as<T>(p.wqkv), n, as<T>(trans), n, T_, n, p.d, nullptr, ACT_NONE, s);
  AttnSimtArgs a{trans, p.attn_v, p.attn_b, (int)B, (int)M, p.H, p.G, p.r, p.d, ctx};
  simt_attention<T>(a, s);
}

void tc_attention(size_t B, size_t M, const bf16* qkv, int qkv_cols, int q_off, int k_off,
                  int v_off, int heads, int groups, int rp, void* out, int64_t ldo,
                  cudaStream_t s, bool causal = false) {
  AttnTcArgs a;
  a.qkv = qkv;
  a.ldq = qkv_cols;
  a.qkv_cols = qkv_cols;
  a.q_off = q_off;
  a.k_off = k_off;
  a.v_off = v_off;
  a.batch = (int)B;
  a.seq = (int)M;
  a.heads = heads;
  a.groups = groups;
  a.rank_pad = rp;
  a.out = as<bf16>(out);
  a.ldo = ldo;
  a.causal = causal;
  attn_rankspace_bf16(a, s);
}

// Tensor-core flash attention up to the rank-space output O [T, H*rp]:
// K1 projection into [Qt | P_k | P_v], then K2.
void tc_attention_rank(const Pack& p, size_t B, size_t M, const void* x, void* o_rank,
                       void* trans, cudaStream_t s, const AttnMode& am = AttnMode{}) {
  const int T = static_cast<int>(B * M), n = p.qkv_cols;
  bf16* qkv = as<bf16>(trans);
  gemm_bf16(as<bf16>(x), p.d, as<bf16>(p.wproj_t), p.d, qkv, n, T, n, p.d, p.bproj, ACT_NONE, s);
  const int hr = p.H * p.rp, kv_w = 2 * p.G * p.rp;
  if (am.kind == AttnMode::Full) {
    tc_attention(B, M, qkv, n, 0, hr, (p.H + p.G) * p.rp, p.H, p.G, p.rp, o_rank, hr, s);
    return;
  }
  // decoder rows: the new tokens' [P_k | P_v] columns go to the rank-space
  // cache (prefill: one strided copy; decode: appended by k_attn_decode)
  if (am.kind == AttnMode::Prefill)
    kv_store_bf16(qkv, n, hr, kv_w, static_cast<int>(B), static_cast<int>(M), as<bf16>(am.cache),
                  static_cast<int>(am.max_seq), static_cast<int>(am.pos), am.pos_dev, s);
  if (am.kind == AttnMode::Prefill) {
    tc_attention(B, M, qkv, n, 0, hr, (p.H + p.G) * p.rp, p.H, p.G, p.rp, o_rank, hr, s, true);
    return;
  }
  DecodeArgs a;
  a.qkv = qkv;
  a.ldq = n;
  a.q_off = 0;
  a.cache = as<bf16>(am.cache);
  a.max_seq = static_cast<int>(am.max_seq);
  a.batch = static_cast<int>(B);
  a.heads = p.H;
  a.groups = p.G;
  a.rank_pad = p.rp;
  a.len = static_cast<int>(am.pos_dev ? am.max_seq : am.pos + 1);
  a.splits = decode_splits(a.batch, a.heads, a.len);
  a.pos_dev = am.pos_dev;
  // split partials live right after the projection rows
  a.part = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(qkv + (size_t)T * n) + 255) & ~uintptr_t(255));
  a.out = as<bf16>(o_rank);
  a.ldo = hr;
  attn_decode_bf16(a, s);
}

// Split-plane (fp32 policy) attention up to the rank-space output O planes
// [T, H*rp] at o_rank (hi) / o_rank + T*H*rp (lo): K1 (X3) projection into
// [Qt | P_k | P_v] planes at the start of `trans`, then K2 (X3).
void x3_attention_rank(const Pack& p, size_t B, size_t M, const void* x, bf16* o_rank,
                       void* trans, cudaStream_t s) {
  const int T = static_cast<int>(B * M), n = p.qkv_cols, hr = p.H * p.rp;
  const size_t tn = static_cast<size_t>(T) * n;
  bf16* qkv = as<bf16>(trans);
  gemm_x3(pl(x, (size_t)T * p.d), p.d, wpl(p.wproj_t, p.wproj_lo), p.d, plo(qkv, tn), n, T, n,
          p.d, p.bproj, ACT_NONE, s);
  AttnTcArgs a;
  a.qkv = qkv;
  a.planes = true;
  a.ldq = n;
  a.qkv_cols = n;
  a.q_off = 0;
  a.k_off = hr;
  a.v_off = (p.H + p.G) * p.rp;
  a.batch = static_cast<int>(B);
  a.seq = static_cast<int>(M);
  a.heads = p.H;
  a.groups = p.G;
  a.rank_pad = p.rp;
  a.out = o_rank;
  a.out_ps = (int64_t)T * hr;
  a.ldo = hr;
  attn_rankspace_bf16(a, s);
}

// Materializing baselines: dense Q|K|V [T, 3d] (dense twin or rebuilt from
// the factors) then the same attention kernel with r = head_dim.
// C[M,N] = A[M,K] W^T (+ bias) (act) in the pack's storage: bf16, or split
// planes (plane stride = rows x leading dimension) on the fp32 policy.
void mm(const Pack& p, const void* A, int64_t lda, const void* W, const void* W_lo, int64_t ldw,
        void* Cm, int64_t ldc, int M, int N, int K, const float* bias, int act, cudaStream_t s) {
  if (p.x3)
    gemm_x3(pl(A, (size_t)M * lda), lda, wpl(W, W_lo), ldw, plo(Cm, (size_t)M * ldc), ldc, M, N,
            K, bias, act, s);
  else
    gemm_bf16(as<bf16>(A), lda, as<bf16>(W), ldw, as<bf16>(Cm), ldc, M, N, K, bias, act, s);
}

// Materializing baselines: Dense (encoder.cpp:99-105: dense_attention on the
// layer's dense weights) and NaiveLowRank (attention.cpp:271-292: Q|K|V
// rebuilt from the factors) -- dense Q|K|V [T, 3*H*dhp] at the start of
// `trans`, then the attention kernel with r = head width (dhp, zero-padded).
// Returns the context [T, H*dhp] (head width when dhp == dh), placed in
// `trans` after Q|K|V (and the naive P).
bf16* tc_attention_dense(const Pack& p, int mode, size_t B, size_t M, const void* x, void* trans,
                         cudaStream_t s) {
  if (!p.dense) fail(Kind::Config, "dense / naive_lowrank modes need a pack built with dense=1 "
                                   "(head width <= 64, d_model and d_ff multiples of 8)");
  if (mode == FSVD_MODE_NAIVE_LOWRANK && !p.wpn_t)
    fail(Kind::Config, "naive_lowrank mode on the tensor cores needs a head width of 16, 32 or 64");
  const int T = static_cast<int>(B * M), d = p.d, hp = p.H * p.dhp, n3 = 3 * hp;
  const size_t ew = p.x3 ? kPlanes : 1;  // bf16 elements per stored value
  bf16* qkv = as<bf16>(trans);
  bf16* o = qkv + ew * (size_t)T * n3;
  if (mode == FSVD_MODE_DENSE) {
    mm(p, x, d, p.dqkv_t, p.dqkv_lo, d, qkv, n3, T, n3, d, p.dqkv_b, ACT_NONE, s);
  } else {
    const int n = 3 * p.G * p.rp;
    bf16* P = o;
    o = P + ew * (size_t)T * n;
    mm(p, x, d, p.wpn_t, p.wpn_lo, d, P, n, T, n, d, nullptr, ACT_NONE, s);
    mm(p, P, n, p.dvbd_t, p.dvbd_lo, n, qkv, n3, T, n3, n, p.nqkv_b, ACT_NONE, s);
  }
  AttnTcArgs a;
  a.qkv = qkv;
  a.ldq = n3;
  a.qkv_cols = n3;
  a.q_off = 0;
  a.k_off = hp;
  a.v_off = 2 * hp;
  a.batch = static_cast<int>(B);
  a.seq = static_cast<int>(M);
  a.heads = p.H;
  a.groups = p.H;
  a.rank_pad = p.dhp;
  a.out = o;
  a.ldo = hp;
  if (p.x3) {
    a.planes = true;
    a.out_ps = (int64_t)T * hp;
  }
  attn_rankspace_bf16(a, s);
  return o;
}

}  // namespace

void attention_fwd(const Pack& p, int mode, size_t B, size_t M, const void* x, void* ctx,
                   void* trans, cudaStream_t s) {
  const int T = static_cast<int>(B * M);
  if (mode == FSVD_MODE_DENSE || mode == FSVD_MODE_NAIVE_LOWRANK)
    fail(Kind::Config, "the materializing attention baselines run inside a layer (run_layer)");
  if (p.attn_tc) {
    // rank-space output after the projection buffer, then back to head width
    const int hr = p.H * p.rp;
    bf16* o_rank = as<bf16>(trans) + (size_t)T * p.qkv_cols;
    tc_attention_rank(p, B, M, x, o_rank, trans, s);
    gemm_bf16(o_rank, hr, as<bf16>(p.wvc_t), hr, as<bf16>(ctx), p.d, T, p.d, hr, p.bv, ACT_NONE, s);
  } else if (p.x3) {
    const int hr = p.H * p.rp;
    bf16* o_rank = as<bf16>(trans) + kPlanes * (size_t)T * p.qkv_cols;
    x3_attention_rank(p, B, M, x, o_rank, trans, s);
    gemm_x3(pl(o_rank, (size_t)T * hr), hr, wpl(p.wvc_t, p.wvc_lo), hr,
            plo(ctx, (size_t)T * p.d), p.d, T, p.d, hr, p.bv, ACT_NONE, s);
  } else if (p.dtype == FSVD_BF16) {
    simt_attention_t<bf16>(p, B, M, x, ctx, trans, s);
  } else {
    simt_attention_t<float>(p, B, M, x, ctx, trans, s);
  }
}

void outproj_fwd(const Pack& p, int mode, size_t B, size_t M, const void* ctx, void* out,
                 void* trans, cudaStream_t s) {
  const int T = static_cast<int>(B * M), d = p.d;
  if (mode == FSVD_MODE_DENSE)
    fail(Kind::Config, "the dense output projection runs inside a layer (run_layer)");
  if (p.out_tc) {
    bf16* P = as<bf16>(trans);
    gemm_bf16(as<bf16>(ctx), d, as<bf16>(p.uo_t), d, P, p.prp, T, p.prp, d, nullptr, ACT_NONE, s);
    gemm_bf16(P, p.prp, as<bf16>(p.vo_t), p.prp, as<bf16>(out), d, T, d, p.prp, p.bo, ACT_NONE, s);
  } else if (p.x3) {
    bf16* P = as<bf16>(trans);
    const size_t tp = (size_t)T * p.prp;
    gemm_x3(pl(ctx, (size_t)T * d), d, wpl(p.uo_t, p.uo_t_lo), d, plo(P, tp), p.prp, T,
            p.prp, d, nullptr, ACT_NONE, s);
    gemm_x3(pl(P, tp), p.prp, wpl(p.vo_t, p.vo_t_lo), p.prp, plo(out, (size_t)T * d), d, T,
            d, p.prp, p.bo, ACT_NONE, s);
  } else if (p.dtype == FSVD_BF16) {
    simt_gemm<bf16>(as<bf16>(ctx), d, as<bf16>(p.uo), p.pr, as<bf16>(trans), p.pr, T, p.pr, d,
                    nullptr, ACT_NONE, s);
    simt_gemm<bf16>(as<bf16>(trans), p.pr, as<bf16>(p.vo), d, as<bf16>(out), d, T, d, p.pr, p.bo,
                    ACT_NONE, s);
  } else {
    simt_gemm<float>(as<float>(ctx), d, as<float>(p.uo), p.pr, as<float>(trans), p.pr, T, p.pr, d,
                     nullptr, ACT_NONE, s);
    simt_gemm<float>(as<float>(trans), p.pr, as<float>(p.vo), d, as<float>(out), d, T, d, p.pr,
                     p.bo, ACT_NONE, s);
  }
}

// attention + output projection of one layer: x -> branch.  On the tensor-
// core flash path the rank-space attention output feeds the folded
// out-projection directly (one GEMM, K = H*rp); `scratch` holds it.
void attention_block(const Pack& p, int mode, size_t B, size_t M, const void* x, void* scratch,
                     void* branch, void* trans, cudaStream_t s, const AttnMode& am = AttnMode{}) {
  const bool flash = mode == FSVD_MODE_FLASH_V1 || mode == FSVD_MODE_FLASH_V2;
  if (!flash) {
    const int T = static_cast<int>(B * M);
    bf16* o = tc_attention_dense(p, mode, B, M, x, trans, s);
    if (mode == FSVD_MODE_DENSE)  // dense_output_projection on the layer's W_o, b_o
      mm(p, o, p.H * p.dhp, p.do_t, p.do_lo, p.H * p.dhp, branch, p.d, T, p.d, p.H * p.dhp, p.dbo,
         ACT_NONE, s);
    else  // naive_projection (encoder.cpp:65-80): (ctx U_o) V_o + b_o
      outproj_fwd(p, FSVD_MODE_FLASH_V1, B, M, o, branch, trans, s);
    return;
  }
  if (flash && p.x3) {  // split planes: O after the projection planes in `trans`
    const int T = static_cast<int>(B * M), hr = p.H * p.rp;
    bf16* o = as<bf16>(trans) + kPlanes * (size_t)T * p.qkv_cols;
    x3_attention_rank(p, B, M, x, o, trans, s);
    gemm_x3(pl(o, (size_t)T * hr), hr, wpl(p.wov_t, p.wov_lo), hr,
            plo(branch, (size_t)T * p.d), p.d, T, p.d, hr, p.bov, ACT_NONE, s);
    return;
  }
  if (flash && p.attn_tc && p.out_tc) {
    const int T = static_cast<int>(B * M), hr = p.H * p.rp;
    tc_attention_rank(p, B, M, x, scratch, trans, s, am);
    gemm_bf16(as<bf16>(scratch), hr, as<bf16>(p.wov_t), hr, as<bf16>(branch), p.d, T, p.d, hr,
              p.bov, ACT_NONE, s);
    return;
  }
  attention_fwd(p, mode, B, M, x, scratch, trans, s);
  outproj_fwd(p, mode, B, M, scratch, branch, trans, s);
}

namespace {
template <typename T>
void simt_ffn_t(const Pack& p, int mode, size_t Tn, const void* x, void* out, void* trans,
                cudaStream_t s) {
  const int n = static_cast<int>(Tn), d = p.d, fr = p.fr, df = p.df;
  if (mode == FSVD_MODE_FLASH_V2) {
    simt_ffn_fused<T>(as<T>(x), as<T>(p.uup), as<T>(p.vup), p.bup, as<T>(p.udn), as<T>(p.vdn),
                      p.bdn, as<T>(out), n, d, fr, df, p.act, s);
    return;
  }
  T* P = as<T>(trans);
  T* Z = P + (size_t)n * fr;
  simt_gemm<T>(as<T>(x), d, as<T>(p.uup), fr, P, fr, n, fr, d, nullptr, ACT_NONE, s);
  FfnSimtArgs a{P, p.vup, p.bup, p.udn, Z, n, fr, df, p.act};
  simt_ffn_stream<T>(a, s);
  simt_gemm<T>(Z, fr, as<T>(p.vdn), d, as<T>(out), d, n, d, fr, p.bdn, ACT_NONE, s);
}
}  // namespace

// The CTA-pair FFN (ffn2_tc.cu) is opt-in (FSVD_FFN_PAIR=1): it is correct
// but measured slower than the single-CTA kernel on cfg2 (113 vs 85 us; see
// DESIGN.md), so the single-CTA kernel is the default.
// FSVD_PRE_LN_UNFUSED=1 keeps the pre-LN out-projection and LN2 as separate
// kernels (comparison runs).
bool pre_ln_unfused() {
  static const bool v = [] {
    const char* e = getenv("FSVD_PRE_LN_UNFUSED");
    return e && e[0] == '1';
  }();
  return v;
}

// V2 FFN on the CTA-pair kernel (ffn2_tc.cu): the default for the plain and
// the post-LN fused FFN (the pre-LN residual / chained-LN forms run k_ffn);
// FSVD_FFN_PAIR=0 selects the single-CTA kernel (developer A/B switch).
bool use_ffn_pair(const Pack& p, int T) {
  static const bool enabled = [] {
    const char* e = getenv("FSVD_FFN_PAIR");
    return !(e && e[0] == '0');
  }();
  return enabled && T >= 256 && ffn_pair_supported(p.d, p.df, p.frp);
}

void ffn_fwd(const Pack& p, int mode, size_t B, size_t M, const void* x, void* out, void* trans,
             cudaStream_t s) {
  const int T = static_cast<int>(B * M), d = p.d, df = p.df;
  if (mode == FSVD_MODE_DENSE || mode == FSVD_MODE_NAIVE_LOWRANK) {
    if (!p.dense) fail(Kind::Config, "dense / naive_lowrank modes need a pack built with dense=1");
    const size_t ew = p.x3 ? kPlanes : 1;
    if (mode == FSVD_MODE_DENSE) {  // ffn_dense (ffn.cpp:187-218) on the layer's dense weights
      const int ddf = p.ddf;
      bf16* hid = as<bf16>(trans);
      mm(p, x, d, p.din_t, p.din_lo, d, hid, ddf, T, ddf, d, p.dbin, p.dact, s);
      mm(p, hid, ddf, p.dout_t, p.dout_lo, ddf, out, d, T, d, ddf, p.dbout, ACT_NONE, s);
    } else {  // ffn_naive_lowrank (ffn.cpp:220-255): the hidden materialised
      if (!p.has_ffn) fail(Kind::Config, "naive_lowrank mode needs factorized FFN weights");
      const int frp = p.frp;
      bf16* P = as<bf16>(trans);
      bf16* hid = P + ew * (size_t)T * frp;
      bf16* Z = hid + ew * (size_t)T * df;
      mm(p, x, d, p.uup_t, p.uup_t_lo, d, P, frp, T, frp, d, nullptr, ACT_NONE, s);
      mm(p, P, frp, p.vup_t, p.vup_t_lo, frp, hid, df, T, df, frp, p.bup, p.act, s);
      mm(p, hid, df, p.udn_t, p.udn_t_lo, df, Z, frp, T, frp, df, nullptr, ACT_NONE, s);
      mm(p, Z, frp, p.vdn_t, p.vdn_t_lo, frp, out, d, T, d, frp, p.bdn, ACT_NONE, s);
    }
    return;
  }
  if (p.x3) {  // split planes: V1 chain for both FFN variants (ffn_v1 == ffn_v2)
    bf16* P = as<bf16>(trans);
    const size_t tf = (size_t)T * p.frp;
    bf16* Z = P + kPlanes * tf;
    gemm_x3(pl(x, (size_t)T * d), d, wpl(p.uup_t, p.uup_t_lo), d, plo(P, tf), p.frp, T,
            p.frp, d, nullptr, ACT_NONE, s);
    FfnTcArgs a{};
    a.T = T;
    a.d_model = d;
    a.d_ff = df;
    a.rank_pad = p.frp;
    a.up_v_t = as<bf16>(p.vup_t);
    a.up_b = p.bup;
    a.dn_u_t = as<bf16>(p.udn_t);
    a.dn_v_t = as<bf16>(p.vdn_t);
    a.dn_b = p.bdn;
    a.act = p.act;
    a.p_in = P;
    a.planes = true;
    a.z_out = Z;
    ffn_stream_bf16(a, s);
    gemm_x3(pl(Z, tf), p.frp, wpl(p.vdn_t, p.vdn_t_lo), p.frp, plo(out, (size_t)T * d), d,
            T, d, p.frp, p.bdn, ACT_NONE, s);
    return;
  }
  if (p.ffn_tc) {
    FfnTcArgs a{};
    a.T = T;
    a.d_model = d;
    a.d_ff = df;
    a.rank_pad = p.frp;
    a.x = as<bf16>(x);
    a.up_u_t = as<bf16>(p.uup_t);
    a.up_v_t = as<bf16>(p.vup_t);
    a.up_b = p.bup;
    a.dn_u_t = as<bf16>(p.udn_t);
    a.dn_v_t = as<bf16>(p.vdn_t);
    a.dn_b = p.bdn;
    a.act = p.act;
    a.out = as<bf16>(out);
    if (mode == FSVD_MODE_FLASH_V2 && !p.ffn_wide) {
      a.seq_tiles = seq_tiles_of(M);
      if (use_ffn_pair(p, T)) ffn_fused_pair_bf16(a, s);
      else ffn_fused_bf16(a, s);
    } else {
      bf16* P = as<bf16>(trans);
      bf16* Z = P + (size_t)T * p.frp;
      gemm_bf16(as<bf16>(x), d, a.up_u_t, d, P, p.frp, T, p.frp, d, nullptr, ACT_NONE, s);
      a.p_in = P;
      a.z_out = Z;
      ffn_stream_bf16(a, s);
      gemm_bf16(Z, p.frp, a.dn_v_t, p.frp, as<bf16>(out), d, T, d, p.frp, p.bdn, ACT_NONE, s);
    }
  } else if (p.dtype == FSVD_BF16) {
    simt_ffn_t<bf16>(p, mode, (size_t)T, x, out, trans, s);
  } else {
    simt_ffn_t<float>(p, mode, (size_t)T, x, out, trans, s);
  }
}

// out = resid + FFN(x) with the residual added in the FFN's last epilogue
// (pre-LN layers).  Returns false outside the tensor-core flash path.
bool ffn_resid_fwd(const Pack& p, int mode, size_t B, size_t M, const void* x, const void* resid,
                   void* out, void* trans, cudaStream_t s) {
  const int T = static_cast<int>(B * M), d = p.d;
  if (!p.ffn_tc || !(mode == FSVD_MODE_FLASH_V1 || mode == FSVD_MODE_FLASH_V2)) return false;
  FfnTcArgs a{};
  a.T = T;
  a.d_model = d;
  a.d_ff = p.df;
  a.rank_pad = p.frp;
  a.x = as<bf16>(x);
  a.up_u_t = as<bf16>(p.uup_t);
  a.up_v_t = as<bf16>(p.vup_t);
  a.up_b = p.bup;
  a.dn_u_t = as<bf16>(p.udn_t);
  a.dn_v_t = as<bf16>(p.vdn_t);
  a.dn_b = p.bdn;
  a.act = p.act;
  a.out = as<bf16>(out);
  if (mode == FSVD_MODE_FLASH_V2 && !p.ffn_wide) {
    a.resid = as<bf16>(resid);
    a.seq_tiles = seq_tiles_of(M);
    ffn_fused_bf16(a, s);
    return true;
  }
  bf16* P = as<bf16>(trans);
  bf16* Z = P + (size_t)T * p.frp;
  gemm_bf16(as<bf16>(x), d, a.up_u_t, d, P, p.frp, T, p.frp, d, nullptr, ACT_NONE, s);
  a.p_in = P;
  a.z_out = Z;
  ffn_stream_bf16(a, s);
  gemm_bf16(Z, p.frp, a.dn_v_t, p.frp, as<bf16>(out), d, T, d, p.frp, p.bdn, ACT_NONE, s,
            as<bf16>(resid), d);
  return true;
}

// out = LN2(x + FFN(x)) with the residual + LayerNorm fused into the FFN's
// last GEMM (V2: the fused kernel's epilogue; V1: the Z V_down GEMM).
// Returns false when the shape is outside the fused kernels' range.
bool ffn_ln_fwd(const Pack& p, int mode, size_t B, size_t M, const void* x, void* out,
                void* trans, cudaStream_t s) {
  const int T = static_cast<int>(B * M), d = p.d;
  if (!p.ffn_tc || p.d != p.dr || !gemm_ln_supported(d, p.frp)) return false;
  if (mode == FSVD_MODE_FLASH_V2 && !p.ffn_wide) {
    FfnTcArgs a{};
    a.T = T;
    a.d_model = d;
    a.d_ff = p.df;
    a.rank_pad = p.frp;
    a.x = as<bf16>(x);
    a.up_u_t = as<bf16>(p.uup_t);
    a.up_v_t = as<bf16>(p.vup_t);
    a.up_b = p.bup;
    a.dn_u_t = as<bf16>(p.udn_t);
    a.dn_v_t = as<bf16>(p.vdn_t);
    a.dn_b = p.bdn;
    a.act = p.act;
    a.out = as<bf16>(out);
    a.ln_g = p.ln2g;
    a.ln_b = p.ln2b;
    a.ln_eps = p.eps2;
    a.seq_tiles = seq_tiles_of(M);
    if (use_ffn_pair(p, T)) ffn_fused_pair_bf16(a, s);
    else ffn_fused_bf16(a, s);
    return true;
  }
  if (mode != FSVD_MODE_FLASH_V1 && mode != FSVD_MODE_FLASH_V2) return false;
  FfnTcArgs a{};
  a.T = T;
  a.d_model = d;
  a.d_ff = p.df;
  a.rank_pad = p.frp;
  a.up_v_t = as<bf16>(p.vup_t);
  a.up_b = p.bup;
  a.dn_u_t = as<bf16>(p.udn_t);
  a.dn_v_t = as<bf16>(p.vdn_t);
  a.dn_b = p.bdn;
  a.act = p.act;
  bf16* P = as<bf16>(trans);
  bf16* Z = P + (size_t)T * p.frp;
  gemm_bf16(as<bf16>(x), d, as<bf16>(p.uup_t), d, P, p.frp, T, p.frp, d, nullptr, ACT_NONE, s);
  a.p_in = P;
  a.z_out = Z;
  ffn_stream_bf16(a, s);
  gemm_ln_bf16(Z, p.frp, a.dn_v_t, p.frp, p.bdn, as<bf16>(x), p.ln2g, p.ln2b, p.eps2,
               as<bf16>(out), T, d, p.frp, s, nullptr, seq_tiles_of(M));
  return true;
}

namespace {
// Decode step (T = batch rows, one token each): A [T, max(H*rp, d)], B [T, d],
// transient = max(projection rows + split partials, FFN chain P | hidden | Z |
// branch).
struct DecodeLayout {
  size_t a, b, t;
  size_t total() const { return a + b + t + 256; }
};
DecodeLayout decode_layout(const Pack& p, size_t T, size_t len) {
  const size_t es = p.es;
  const size_t attn = align256(T * p.qkv_cols * es) +
                      align256(decode_partial_bytes(static_cast<int>(T), p.H, p.rp,
                                                    static_cast<int>(len)));
  // FFN chain: P | Z | branch (bf16) + the fp32 per-split partial Z
  const size_t nblk = (static_cast<size_t>(p.df) + 127) / 128;
  const size_t ffn = align256(T * (2 * (size_t)p.frp + p.d) * es) +
                     align256(nblk * T * p.frp * sizeof(float));
  return {align256(T * std::max<size_t>((size_t)p.H * p.rp, p.d) * es), align256(T * p.d * es),
          std::max(attn, ffn)};
}
// Skinny FFN branch for decode rows (one row tile): P = x U_up (64-wide GEMM
// tiles), the feature stream K3 with every 128-feature block on its own CTA
// (fp32 partial Z per block, summed in order), then Z V_down + b.
void ffn_branch_skinny(const Pack& p, int T, const void* x, void* branch, void* trans,
                       cudaStream_t s) {
  bf16* P = as<bf16>(trans);
  bf16* Z = P + (size_t)T * p.frp;
  bf16* br = as<bf16>(branch);
  float* part = reinterpret_cast<float*>(
      (reinterpret_cast<uintptr_t>(Z + (size_t)T * p.frp + (size_t)T * p.d) + 255) & ~uintptr_t(255));
  gemm_bf16(as<bf16>(x), p.d, as<bf16>(p.uup_t), p.d, P, p.frp, T, p.frp, p.d, nullptr, ACT_NONE, s);
  FfnTcArgs a{};
  a.T = T;
  a.d_model = p.d;
  a.d_ff = p.df;
  a.rank_pad = p.frp;
  a.up_v_t = as<bf16>(p.vup_t);
  a.up_b = p.bup;
  a.dn_u_t = as<bf16>(p.udn_t);
  a.dn_v_t = as<bf16>(p.vdn_t);
  a.dn_b = p.bdn;
  a.act = p.act;
  a.p_in = P;
  a.split_blocks = 1;
  a.z_part = part;
  ffn_stream_bf16(a, s);
  const int splits = (p.df + 127) / 128;
  z_partial_sum_bf16(part, splits, (int64_t)T * p.frp, Z, s);
  gemm_bf16(Z, p.frp, as<bf16>(p.vdn_t), p.frp, br, p.d, T, p.d, p.frp, p.bdn, ACT_NONE, s);
}
void layer_decode(const Pack& p, bool pre_ln, size_t B, const void* x, void* out, void* ws,
                  size_t ws_bytes, cudaStream_t s, const AttnMode& am) {
  const DecodeLayout lay = decode_layout(p, B, am.pos_dev ? am.max_seq : am.pos + 1);
  if (ws_bytes < lay.total())
    fail(Kind::Config, "workspace too small: need " + std::to_string(lay.total()) + " bytes, got " +
                           std::to_string(ws_bytes));
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  void* A = base;
  void* Bb = base + lay.a;
  void* trans = base + lay.a + lay.b;
  const int T = static_cast<int>(B), hr = p.H * p.rp;
  bf16* branch = as<bf16>(trans) + (size_t)T * 2 * p.frp;  // after the FFN chain's P | Z
  if (!pre_ln) {
    tc_attention_rank(p, B, 1, x, A, trans, s, am);                          // O_rank -> A
    gemm_bf16(as<bf16>(A), hr, as<bf16>(p.wov_t), hr, branch, p.d, T, p.d, hr, p.bov, ACT_NONE, s);
    ln(p, x, branch, p.ln1g, p.ln1b, p.eps1, Bb, T, s);                       // resid -> B
    ffn_branch_skinny(p, T, Bb, branch, trans, s);
    ln(p, Bb, branch, p.ln2g, p.ln2b, p.eps2, out, T, s);                     // out
  } else {
    ln(p, x, nullptr, p.ln1g, p.ln1b, p.eps1, Bb, T, s);                      // normed -> B
    tc_attention_rank(p, B, 1, Bb, A, trans, s, am);                          // O_rank -> A
    gemm_bf16(as<bf16>(A), hr, as<bf16>(p.wov_t), hr, branch, p.d, T, p.d, hr, p.bov, ACT_NONE, s);
    add(p, x, branch, Bb, (int64_t)T * p.d, s);                               // resid -> B
    ln(p, Bb, nullptr, p.ln2g, p.ln2b, p.eps2, A, T, s);                      // normed -> A
    ffn_branch_skinny(p, T, A, branch, trans, s);
    add(p, Bb, branch, out, (int64_t)T * p.d, s);                             // out
  }
}
}  // namespace

namespace {
// The fused pre-LN tensor-core schedule (layer_fwd) applies to this pack.
bool pre_ln_fused(const Pack& p, int mode, size_t T) {
  return p.attn_tc && p.out_tc && p.ffn_tc && p.dtype == FSVD_BF16 && p.d == p.dr &&
         (mode == FSVD_MODE_FLASH_V1 || mode == FSVD_MODE_FLASH_V2) && !p.ffn_wide &&
         gemm_ln_supported(p.d, p.H * p.rp) && !pre_ln_unfused();
}
// Layer p can apply q's LN1 in its FFN epilogue (ln_epi.cuh shape range).
bool pre_ln_linkable(const Pack& p, const Pack& q, int mode, size_t T) {
  return pre_ln_fused(p, mode, T) && pre_ln_fused(q, mode, T) && q.d == p.d &&
         gemm_ln_supported(p.d, p.frp);
}
}  // namespace

bool pre_ln_link_ok(const Pack& p, const Pack& q, int mode, size_t T) {
  return pre_ln_linkable(p, q, mode, T);
}

void model_layers_fwd(const Pack* const* packs, size_t n, int mode, bool pre_ln, size_t B, size_t M,
                      const void* x, void* out, void* ws, size_t ws_bytes, cudaStream_t s) {
  bool done = false;
  for (size_t i = 0; i < n; ++i) {
    LayerLink lk;
    lk.ln1_done = done;
    if (pre_ln && i + 1 < n && pre_ln_linkable(*packs[i], *packs[i + 1], mode, B * M))
      lk.next = packs[i + 1];
    layer_fwd(*packs[i], mode, pre_ln, B, M, i == 0 ? x : out, out, ws, ws_bytes, s, AttnMode{}, lk);
    done = lk.next != nullptr;
  }
}

void layer_fwd(const Pack& p, int mode, bool pre_ln, size_t B, size_t M, const void* x, void* out,
               void* ws, size_t ws_bytes, cudaStream_t s, const AttnMode& am,
               const LayerLink& link) {
  if (am.kind == AttnMode::Decode) {
    if (M != 1) fail(Kind::Config, "a decode step carries one token per sequence");
    if (!(p.attn_tc && p.out_tc && p.ffn_tc && p.dtype == FSVD_BF16))
      fail(Kind::Config, "decoder rows run on the bf16 tensor-core flash path");
    layer_decode(p, pre_ln, B, x, out, ws, ws_bytes, s, am);
    return;
  }
  const size_t T = B * M;
  if ((mode == FSVD_MODE_FLASH_V1 || mode == FSVD_MODE_FLASH_V2 ||
       mode == FSVD_MODE_NAIVE_LOWRANK) && !(p.has_attn && p.has_out && p.has_ffn))
    fail(Kind::Config, "this mode needs factorized weights on both sublayers");
  const WsLayout lay = ws_layout(p, B, M, mode, pre_ln, am.kind == AttnMode::Full);
  if (ws_bytes < lay.total())
    fail(Kind::Config, "workspace too small: need " + std::to_string(lay.total()) + " bytes, got " +
                           std::to_string(ws_bytes));
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  void* A = base;
  void* Bb = base + lay.a;
  void* trans = base + lay.a + lay.b;
  const int rows = static_cast<int>(T);
  if (am.kind != AttnMode::Full && !(p.attn_tc && p.out_tc &&
                                      (mode == FSVD_MODE_FLASH_V1 || mode == FSVD_MODE_FLASH_V2)))
    fail(Kind::Config, "decoder rows run on the bf16 tensor-core flash path");
  if (lay.chunks > 0) {
    // compact fused post-LN schedule (ws_layout): per chunk of sequences, K1
    // [Qt -> A | P_k P_v -> transient] and K2 (output over Qt in A); then
    // K6 (LN1 -> out, in place when out == x) and the FFN in place over out
    const int hr = p.H * p.rp, kvw = 2 * p.G * p.rp, n = p.qkv_cols;
    bf16* kv = as<bf16>(base + lay.a);
    const size_t cb = (B + lay.chunks - 1) / lay.chunks;
    for (size_t b0 = 0; b0 < B; b0 += cb) {
      const size_t nb = std::min(cb, B - b0);
      const int crows = static_cast<int>(nb * M);
      const size_t r0 = b0 * M;
      bf16* qa = as<bf16>(A) + r0 * hr;
      gemm_bf16_split(as<bf16>(x) + r0 * p.d, p.d, as<bf16>(p.wproj_t), p.d, qa, hr, hr, kv, kvw,
                      crows, n, p.d, p.bproj, s);
      AttnTcArgs a;
      a.qkv = qa;
      a.ldq = hr;
      a.qkv_cols = hr;
      a.q_off = 0;
      a.kv = kv;
      a.ldkv = kvw;
      a.kv_cols = kvw;
      a.k_off = 0;
      a.v_off = p.G * p.rp;
      a.batch = static_cast<int>(nb);
      a.seq = static_cast<int>(M);
      a.heads = p.H;
      a.groups = p.G;
      a.rank_pad = p.rp;
      a.out = qa;
      a.ldo = hr;
      attn_rankspace_bf16(a, s);
    }
    gemm_ln_bf16(as<bf16>(A), hr, as<bf16>(p.wov_t), hr, p.bov, as<bf16>(x), p.ln1g, p.ln1b,
                 p.eps1, as<bf16>(out), rows, p.d, hr, s, nullptr, seq_tiles_of(M));
    if (!ffn_ln_fwd(p, mode, B, M, out, out, A, s))
      fail(Kind::Config, "compact post-LN schedule without a fused FFN LayerNorm");
  } else if (lay.unfused_compact) {
    // K1 -> [Qt | P_k | P_v] (transient); K2 writes O over Qt; folded
    // out-projection -> A; K5 LN1(x + A) -> out; FFN(out) -> A; K5 LN2 -> out
    const int hr = p.H * p.rp, n = p.qkv_cols;
    bf16* qkv = as<bf16>(trans);
    gemm_bf16(as<bf16>(x), p.d, as<bf16>(p.wproj_t), p.d, qkv, n, rows, n, p.d, p.bproj, ACT_NONE,
              s);
    tc_attention(B, M, qkv, n, 0, hr, (p.H + p.G) * p.rp, p.H, p.G, p.rp, qkv, n, s);
    gemm_bf16(qkv, n, as<bf16>(p.wov_t), hr, as<bf16>(A), p.d, rows, p.d, hr, p.bov, ACT_NONE, s);
    ln(p, x, A, p.ln1g, p.ln1b, p.eps1, out, rows, s);
    ffn_fwd(p, mode, B, M, out, A, trans, s);
    ln(p, out, A, p.ln2g, p.ln2b, p.eps2, out, rows, s);
  } else if (!pre_ln && fused_post_ln(p, mode)) {
    // rank-space attention -> A; folded out-projection + residual + LN1 -> B
    tc_attention_rank(p, B, M, x, A, trans, s, am);
    gemm_ln_bf16(as<bf16>(A), p.H * p.rp, as<bf16>(p.wov_t), p.H * p.rp, p.bov, as<bf16>(x),
                 p.ln1g, p.ln1b, p.eps1, as<bf16>(Bb), rows, p.d, p.H * p.rp, s, nullptr, seq_tiles_of(M));
    if (!ffn_ln_fwd(p, mode, B, M, Bb, out, trans, s)) {              // out = LN2(B + ffn(B))
      ffn_fwd(p, mode, B, M, Bb, A, trans, s);
      ln(p, Bb, A, p.ln2g, p.ln2b, p.eps2, out, rows, s);
    }
  } else if (!pre_ln) {
    attention_block(p, mode, B, M, x, A, Bb, trans, s, am);           // branch -> B
    ln(p, x, Bb, p.ln1g, p.ln1b, p.eps1, Bb, rows, s);                // resid  -> B (in place)
    ffn_fwd(p, mode, B, M, Bb, A, trans, s);                          // ffn    -> A
    ln(p, Bb, A, p.ln2g, p.ln2b, p.eps2, out, rows, s);               // out
  } else if (pre_ln && pre_ln_fused(p, mode, T)) {
    // pre-LN, fused: the out-projection epilogue stores the residual stream
    // s = x + attn (into out) and LN2(s) (into A) in one pass; the FFN adds
    // its branch onto s in its own epilogue and, when chained, also applies
    // the next layer's LN1 (into A, where that layer's attention reads it)
    const int hr = p.H * p.rp;
    if (!link.ln1_done) ln(p, x, nullptr, p.ln1g, p.ln1b, p.eps1, A, rows, s);  // normed -> A
    tc_attention_rank(p, B, M, A, Bb, trans, s, am);                  // O_rank  -> B
    gemm_ln_bf16(as<bf16>(Bb), hr, as<bf16>(p.wov_t), hr, p.bov, as<bf16>(x), p.ln2g, p.ln2b,
                 p.eps2, as<bf16>(A), rows, p.d, hr, s, as<bf16>(out), seq_tiles_of(M));  // LN2 -> A, s -> out
    if (link.next && mode == FSVD_MODE_FLASH_V1) {
      // V1: P = A U_up, K3 stream -> Z, then Z V_down + b on the LN kernel:
      // s + ffn -> out and the next layer's LN1 -> A
      bf16* P = as<bf16>(trans);
      bf16* Z = P + (size_t)rows * p.frp;
      gemm_bf16(as<bf16>(A), p.d, as<bf16>(p.uup_t), p.d, P, p.frp, rows, p.frp, p.d, nullptr,
                ACT_NONE, s);
      FfnTcArgs a{};
      a.T = rows;
      a.d_model = p.d;
      a.d_ff = p.df;
      a.rank_pad = p.frp;
      a.up_v_t = as<bf16>(p.vup_t);
      a.up_b = p.bup;
      a.dn_u_t = as<bf16>(p.udn_t);
      a.dn_v_t = as<bf16>(p.vdn_t);
      a.dn_b = p.bdn;
      a.act = p.act;
      a.p_in = P;
      a.z_out = Z;
      ffn_stream_bf16(a, s);
      gemm_ln_bf16(Z, p.frp, as<bf16>(p.vdn_t), p.frp, p.bdn, as<bf16>(out), link.next->ln1g,
                   link.next->ln1b, link.next->eps1, as<bf16>(A), rows, p.d, p.frp, s,
                   as<bf16>(out), seq_tiles_of(M));
    } else if (link.next) {
      FfnTcArgs a{};
      a.T = rows;
      a.d_model = p.d;
      a.d_ff = p.df;
      a.rank_pad = p.frp;
      a.x = as<bf16>(A);
      a.up_u_t = as<bf16>(p.uup_t);
      a.up_v_t = as<bf16>(p.vup_t);
      a.up_b = p.bup;
      a.dn_u_t = as<bf16>(p.udn_t);
      a.dn_v_t = as<bf16>(p.vdn_t);
      a.dn_b = p.bdn;
      a.act = p.act;
      a.out = as<bf16>(A);                 // next layer's LN1(s + ffn)
      a.ln_g = link.next->ln1g;
      a.ln_b = link.next->ln1b;
      a.ln_eps = link.next->eps1;
      a.ln_resid = as<bf16>(out);          // s
      a.sum_out = as<bf16>(out);           // s + ffn: the residual stream
      a.seq_tiles = seq_tiles_of(M);
      if (use_ffn_pair(p, rows)) ffn_fused_pair_bf16(a, s);
      else ffn_fused_bf16(a, s);
    } else {
      ffn_resid_fwd(p, mode, B, M, A, out, out, trans, s);            // s + ffn -> out
    }
  } else if (p.attn_tc && p.out_tc && p.dtype == FSVD_BF16 &&
             (mode == FSVD_MODE_FLASH_V1 || mode == FSVD_MODE_FLASH_V2) &&
             p.ffn_tc) {
    // pre-LN, tensor-core path: both residual adds ride in GEMM epilogues
    const int hr = p.H * p.rp;
    ln(p, x, nullptr, p.ln1g, p.ln1b, p.eps1, A, rows, s);            // normed  -> A
    tc_attention_rank(p, B, M, A, Bb, trans, s, am);                  // O_rank  -> B
    gemm_bf16(as<bf16>(Bb), hr, as<bf16>(p.wov_t), hr, as<bf16>(A), p.d, rows, p.d, hr, p.bov,
              ACT_NONE, s, as<bf16>(x), p.d);                         // x + attn -> A
    ln(p, A, nullptr, p.ln2g, p.ln2b, p.eps2, Bb, rows, s);           // normed  -> B
    ffn_resid_fwd(p, mode, B, M, Bb, A, out, trans, s);               // A + ffn -> out
  } else {
    ln(p, x, nullptr, p.ln1g, p.ln1b, p.eps1, A, rows, s);            // normed -> A
    attention_block(p, mode, B, M, A, Bb, A, trans, s, am);           // branch -> A (via B)
    add(p, x, A, Bb, (int64_t)T * p.d, s);                            // resid  -> B
    ln(p, Bb, nullptr, p.ln2g, p.ln2b, p.eps2, A, rows, s);           // normed -> A
    ffn_fwd(p, mode, B, M, A, out, trans, s);                         // ffn    -> out
    add(p, Bb, out, out, (int64_t)T * p.d, s);                        // out = resid + ffn
  }
}

// Post-LN FFN sublayer: out = LN2(x + ffn(x)) (run_layer's second half,
// encoder.cpp:245-256); the fused kernel (K4 with its LayerNorm epilogue, or
// the V1 chain ending in K6) when the shape allows, else FFN then K5.
size_t ffn_block_workspace_bytes(const Pack& p, size_t B, size_t M, int mode) {
  const size_t T = B * M;
  return align256(T * p.d * p.es) + align256(T * op_transient_elems(p, 2, mode) * p.es) + 256;
}
void ffn_block_fwd(const Pack& p, int mode, size_t B, size_t M, const void* x, void* out,
                   void* ws, size_t ws_bytes, cudaStream_t s) {
  if (ws_bytes < ffn_block_workspace_bytes(p, B, M, mode))
    fail(Kind::Config, "workspace too small for the FFN block");
  const size_t T = B * M;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  void* A = base;
  void* trans = base + align256(T * p.d * p.es);
  if (ffn_ln_fwd(p, mode, B, M, x, out, trans, s)) return;
  ffn_fwd(p, mode, B, M, x, A, trans, s);
  ln(p, x, A, p.ln2g, p.ln2b, p.eps2, out, static_cast<int>(T), s);
}

void check_decoder_pack(const Pack& p) {
  if (!(p.attn_tc && p.out_tc && p.ffn_tc && p.dtype == FSVD_BF16 && p.d == p.dr))
    fail(Kind::Config, "decoder rows run on the bf16 tensor-core flash path (bf16 pack, "
                       "rank padding 16/32/64)");
}

size_t kv_cache_bytes(const Pack& p, size_t B, size_t max_seq) {
  return B * max_seq * 2 * p.G * p.rp * p.es;
}

size_t decoder_workspace_bytes(const Pack& p, size_t B, size_t max_seq, bool pre_ln) {
  const size_t prefill = prefill_workspace_bytes(p, B, max_seq, pre_ln);
  return std::max(prefill, decode_layout(p, B, max_seq).total());
}

}  // namespace fsvd
